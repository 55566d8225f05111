"""Why the bench's c2 K2 runs slower than tools/ew_probe.py's (tools only):
the headline data and allocation order, timed (1) K2 back to back, (2) K1/K2
alternating (the bench's step), (3) alternating with events between them."""
import sys

import torch

from paper_1811_01457_b200 import fused as F
from paper_1811_01457_b200.irtext import parse_ir

sys.path.insert(0, ".")
from bench import AFFSIG  # noqa: E402

m = parse_ir(AFFSIG)
R, C = 1 << 16, 1 << 12
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1234
g = torch.Generator(device="cuda").manual_seed(seed)
x = torch.rand((R, C), generator=g, device="cuda") * 4 - 2
a = torch.rand((C,), generator=g, device="cuda") * 4 - 2
b = torch.rand((C,), generator=g, device="cuda") * 4 - 2
yb = torch.rand((R, C), generator=g, device="cuda") * 2 - 1
y, xbar = torch.empty_like(x), torch.empty_like(x)
abar, bbar = torch.empty_like(a), torch.empty_like(b)
n = R * C


def k1():
    F.fused_map(m, "affsig", [a, x, b], out=y, check=False)


def k2():
    F.fused_map_grad(m, "affsig", [a, x, b], yb, check=False, outs=[abar, xbar, bbar])


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


print(f"seed {seed}: K1 alone {timeit(k1):.4f} ms, K2 alone {timeit(k2):.4f} ms, "
      f"K1+K2 step {timeit(lambda: (k1(), k2())):.4f} ms")
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(20)]
for i in range(20):
    ev[i][0].record()
    k1()
    ev[i][1].record()
    k2()
    ev[i][2].record()
torch.cuda.synchronize()
print(f"  event-split: K1 {sum(e[0].elapsed_time(e[1]) for e in ev) / 20:.4f} ms, "
      f"K2 {sum(e[1].elapsed_time(e[2]) for e in ev) / 20:.4f} ms")

# what precedes K2: another K2, K1, a read-only kernel, a write-heavy copy (event-split)
scratch = torch.empty_like(x)
for label, pre in (("K2", k2), ("K1", k1), ("sum(x) read-only", lambda: x.sum()),
                   ("copy x->scratch", lambda: scratch.copy_(x)), ("fill scratch", lambda: scratch.fill_(1.0))):
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(10)]
    for _ in range(3):
        pre()
        k2()
    for i in range(10):
        pre()
        ev[i][0].record()
        k2()
        ev[i][1].record()
    torch.cuda.synchronize()
    print(f"  K2 after {label:18s} {sum(e[0].elapsed_time(e[1]) for e in ev) / 10:.4f} ms")
