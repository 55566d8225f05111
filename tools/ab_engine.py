"""Interleaved same-process A/B of the Dense training step: two Trainers on
the same chain and batch, B with one engine attribute flipped (e.g.
fused_mse=0), timed in alternating rounds of CUDA-event-timed steps so clock
and power drift hit both arms alike.

    python tools/ab_engine.py c5 fused_mse 0 [rounds] [steps]
"""
import statistics
import sys

import numpy as np
import torch

from paper_1811_01457_b200.dense import Chain, Dense
from paper_1811_01457_b200.train import Trainer

WORKLOADS = {
    "c4": ((4096,) * 5, ("tanh",) * 3 + ("identity",), 65536),
    "c5": ((1024,) * 17, ("tanh",) * 15 + ("identity",), 32768),
}


def main():
    name, attr, val = sys.argv[1], sys.argv[2], sys.argv[3]
    rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 8
    steps = int(sys.argv[5]) if len(sys.argv) > 5 else 10
    sizes, acts, batch = WORKLOADS[name]
    chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(len(acts))]).init_params(
        np.random.default_rng(11))
    g = torch.Generator(device="cuda").manual_seed(100)
    X = torch.rand((batch, sizes[0]), generator=g, device="cuda")
    Y = torch.rand((batch, sizes[-1]), generator=g, device="cuda") * 2 - 1
    arms = {}
    for arm in ("A", "B"):
        tr = Trainer(chain, batch, loss="mse", lr=1e-4, precision="bf16", graph=True)
        if arm == "B":
            old = getattr(tr.engine, attr)
            setattr(tr.engine, attr, type(old)(int(val)) if isinstance(old, (bool, int)) else val)
        for _ in range(3):
            tr.step(X, Y)
        arms[arm] = tr
    torch.cuda.synchronize()
    times = {"A": [], "B": []}
    for r in range(rounds):
        for arm in (("A", "B") if r % 2 == 0 else ("B", "A")):
            tr = arms[arm]
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            for _ in range(steps):
                tr.step(X, Y)
            e.record()
            torch.cuda.synchronize()
            times[arm].append(s.elapsed_time(e) / steps)
    for arm in ("A", "B"):
        t = times[arm]
        print(f"{name} {arm}{'' if arm == 'A' else f' ({attr}={val})'}: median {statistics.median(t):.4f} ms "
              f"min {min(t):.4f} max {max(t):.4f}  loss {float(arms[arm].engine.loss.item()):.6g}")
    d = [b - a for a, b in zip(times["A"], times["B"])]
    se = statistics.stdev(d) / len(d) ** 0.5 if len(d) > 1 else float("nan")
    print(f"{name} B-A per round: median {statistics.median(d):+.4f} ms  mean {statistics.mean(d):+.4f} "
          f"+- {se:.4f} (stderr, {len(d)} rounds)")


if __name__ == "__main__":
    main()
