"""First light of the persistent GEMM chain (tools only): a 3-layer chain vs the
per-layer path, bitwise, then timings of the c5 step (chain vs per layer)."""
import os
import sys
import time

import numpy as np
import torch

from paper_1811_01457_b200.dense import Chain, ChainEngine, Dense

which = sys.argv[1] if len(sys.argv) > 1 else "small"
if which == "small":
    sizes, acts, B = (512, 512, 384, 300), ("tanh", "sigmoid", "identity"), 1024
else:
    W, L, B = (int(v) for v in sys.argv[2:5])
    sizes, acts = (W,) * (L + 1), ("tanh",) * (L - 1) + ("identity",)
rng = np.random.default_rng(0)
chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(len(acts))]).init_params(rng)
X = torch.rand((B, sizes[0]), device="cuda")
Y = torch.rand((B, sizes[-1]), device="cuda") * 2 - 1
res = {}
for use in (False, "full", "pairwise"):
    e = ChainEngine(chain, B, "mse", "bf16", small=False, gemm_chain=use)

    def step():
        e.load_batch(X, Y)
        e.forward()
        e.loss_and_seed()
        e.pullback()

    t0 = time.time()
    step()
    torch.cuda.synchronize()
    print("use_chain", use, "first step ok", round(time.time() - t0, 2), "s", flush=True)
    if use == "full":
        print("  fwd units", e.chains[0].units, "est", round(e.chains[0].est_us, 1), "us; bwd units",
              e.chains[1].units, "est", round(e.chains[1].est_us, 1), "us", flush=True)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        step()
    t.record()
    torch.cuda.synchronize()
    print("  ms/step (fwd+loss+pullback, eager issue)", round(s.elapsed_time(t) / 10, 4), flush=True)
    res[use] = (e.loss.clone(), e.G.clone(), e.Zt.clone())
for mode in ("full", "pairwise"):
    print(mode, "bit-identical loss/G/Zt:", [torch.equal(a, b) for a, b in zip(res[False], res[mode])])
