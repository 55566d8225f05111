"""c1 (MLP 784-32-10, batch 128) step: device time of the one-launch kernel
(CUPTI via torch.profiler), host-issue-bound step time, and the step time
with 20 steps captured in one CUDA graph (no host launch overhead)."""
import numpy as np
import torch

from paper_1811_01457_b200.dense import Chain, Dense
from paper_1811_01457_b200.train import Trainer

B = 128
rng = np.random.default_rng(0)
chain = Chain(Dense(784, 32, "sigmoid"), Dense(32, 10, "identity")).init_params(rng)
X = torch.rand((B, 784), device="cuda")
Y = torch.zeros((B, 10), device="cuda")
Y[torch.arange(B), torch.randint(0, 10, (B,), device="cuda")] = 1
for small in (True, False):
    tr = Trainer(chain, B, loss="softmax_xent", lr=0.05, small=small, graph=not small)
    for _ in range(5):
        tr.step(X, Y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(200):
        tr.step(X, Y)
    e.record()
    torch.cuda.synchronize()
    eager = s.elapsed_time(e) / 200
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(20):
            tr.step(X, Y)
        torch.cuda.synchronize()
    kern = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            k = kern.setdefault(ev.name[:60], [0, 0.0])
            k[0] += 1
            k[1] += ev.device_time
    line = f"small={small}: {eager * 1e3:.1f} us/step issued from Python"
    if small:
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            with torch.cuda.graph(g):
                for _ in range(20):
                    tr.step(X, Y)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        s.record()
        for _ in range(10):
            g.replay()
        e.record()
        torch.cuda.synchronize()
        line += f"; {s.elapsed_time(e) / 200 * 1e3:.1f} us/step with 20 steps per graph"
    print(line)
    for k, (n, t) in sorted(kern.items(), key=lambda kv: -kv[1][1]):
        print(f"   {k:60s} n={n:4d} avg {t / n:8.2f} us")
