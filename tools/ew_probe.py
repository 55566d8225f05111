"""Probe the fused-kernel skeleton at the c2 size: sigmoid(a*x+b) vs plain a*x+b
(same memory traffic, less math) vs torch's own 1R1W / 2R1W kernels."""
import sys

import torch

from paper_1811_01457_b200 import fused as F
from paper_1811_01457_b200.irtext import parse_ir

SRC = """
func @affsig(%a: f64, %x: f64, %b: f64) -> f64 {
^entry:
  %m = mul %a, %x
  %s = add %m, %b
  %y = sigmoid %s
  ret %y
}
func @aff(%a: f64, %x: f64, %b: f64) -> f64 {
^entry:
  %m = mul %a, %x
  %s = add %m, %b
  ret %s
}
func @ident(%a: f64, %x: f64, %b: f64) -> f64 {
^entry:
  ret %x
}
"""


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


m = parse_ir(SRC)
R, C = 1 << 16, 1 << 12
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand((R, C), generator=g, device="cuda") * 4 - 2
yb = torch.rand((R, C), generator=g, device="cuda") * 2 - 1
a = torch.rand(C, generator=g, device="cuda") * 4 - 2
b = torch.rand(C, generator=g, device="cuda") * 4 - 2
y = torch.empty_like(x)
xbar = torch.empty_like(x)
abar = torch.empty_like(a)
bbar = torch.empty_like(b)
n = R * C
for name in ("affsig", "aff", "ident"):
    f = timeit(lambda: F.fused_map(m, name, [a, x, b], out=y, check=False))
    gr = timeit(lambda: F.fused_map_grad(m, name, [a, x, b], yb, check=False, outs=[abar, xbar, bbar]))
    print(f"{name:7s} K1 {f:.4f} ms {8 * n / f / 1e6:7.1f} GB/s | K2 {gr:.4f} ms {12 * n / gr / 1e6:7.1f} GB/s")
f = timeit(lambda: torch.mul(x, 2.0, out=y))
print(f"torch mul 1R1W {f:.4f} ms {8 * n / f / 1e6:.1f} GB/s")
f = timeit(lambda: torch.mul(x, yb, out=y))
print(f"torch mul 2R1W {f:.4f} ms {12 * n / f / 1e6:.1f} GB/s")

# c2 variants of SURVEY §8(d): scalar a, b (full-reduction gradients) and (R,1) a, b (row reductions)
ac = torch.rand((R, 1), generator=g, device="cuda") * 4 - 2
bc = torch.rand((R, 1), generator=g, device="cuda") * 4 - 2
abar_c, bbar_c = torch.empty_like(ac), torch.empty_like(bc)
a1, b1 = torch.rand(1, generator=g, device="cuda") * 4 - 2, torch.rand(1, generator=g, device="cuda") * 4 - 2
abar_1, bbar_1 = torch.empty_like(a1), torch.empty_like(b1)
for label, args, outs in (("(R,1) a,b", [ac, x, bc], [abar_c, xbar, bbar_c]),
                          ("1-elem a,b", [a1, x, b1], [abar_1, xbar, bbar_1])):
    f = timeit(lambda: F.fused_map(m, "affsig", args, out=y, check=False))
    gr = timeit(lambda: F.fused_map_grad(m, "affsig", args, yb, check=False, outs=outs))
    print(f"{label:10s} K1 {f:.4f} ms {8 * n / f / 1e6:7.1f} GB/s | K2 {gr:.4f} ms {12 * n / gr / 1e6:7.1f} GB/s")
f = timeit(lambda: F.fused_map(m, "affsig", [0.7, x, -0.3], out=y, check=False))
gr = timeit(lambda: F.fused_map_grad(m, "affsig", [0.7, x, -0.3], yb, check=False))
print(f"{'f64 a,b':10s} K1 {f:.4f} ms {8 * n / f / 1e6:7.1f} GB/s | K2 {gr:.4f} ms {12 * n / gr / 1e6:7.1f} GB/s")
