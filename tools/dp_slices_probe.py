"""Data-parallel step on one GPU (NCCL world size 1) with layer 0's dW in
1 or 4 row slices (SGB200_DP_L0_SLICES): the GEMM-side cost of slicing, which
at 8 GPUs buys an overlapped last all-reduce bucket.  Shape: c4's per-GPU
shard at 8 GPUs (4 x 4096, batch 8192) unless given WIDTH DEPTH BATCH."""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist

from paper_1811_01457_b200.dense import Chain, Dense
from paper_1811_01457_b200.train import Trainer

width, depth, batch = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4, 8192)))
s = socket.socket()
s.bind(("127.0.0.1", 0))
port = s.getsockname()[1]
s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
sizes = (width,) * (depth + 1)
acts = ("tanh",) * (depth - 1) + ("identity",)
X = torch.rand((batch, width), device="cuda")
Y = torch.rand((batch, width), device="cuda") * 2 - 1
for sl in ("1", "4"):
    os.environ["SGB200_DP_L0_SLICES"] = sl
    chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(depth)]).init_params(np.random.default_rng(0))
    tr = Trainer(chain, batch, loss="mse", lr=1e-4, precision="bf16", dp=True, graph=True)
    for _ in range(5):
        tr.step(X, Y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        tr.step(X, Y)
    b.record()
    torch.cuda.synchronize()
    print(f"slices={sl} (buckets {len(tr.engine.bucket_bounds)}): {a.elapsed_time(b) / 20:.4f} ms/step")
    torch.cuda.synchronize()
    tr.dp.close()
dist.destroy_process_group()
