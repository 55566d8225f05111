"""Time one Dense-chain training step at a given batch (e.g. the per-GPU shard of c5 at 8 GPUs)."""
import sys

import numpy as np
import torch

from paper_1811_01457_b200.dense import Chain, Dense
from paper_1811_01457_b200.train import Trainer

width, depth, batch = (int(v) for v in sys.argv[1:4])
graph = len(sys.argv) < 5 or sys.argv[4] != "nograph"
sizes = (width,) * (depth + 1)
acts = ("tanh",) * (depth - 1) + ("identity",)
chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(depth)]).init_params(np.random.default_rng(0))
tr = Trainer(chain, batch, loss="mse", lr=1e-4, precision="bf16", graph=graph)
X = torch.rand((batch, width), device="cuda")
Y = torch.rand((batch, width), device="cuda") * 2 - 1
for _ in range(5):
    tr.step(X, Y)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    tr.step(X, Y)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
fl = tr.engine.flops_per_step()
print(f"width {width} depth {depth} batch {batch} graph={graph}: {ms:.4f} ms/step, {batch / ms * 1e3:.0f} samples/s, "
      f"{fl / ms / 1e9:.1f} TFLOP/s")
