"""One c5-shaped Dense GEMM of a chosen kind, for ncu captures (tools only).

  python tools/gemm_one.py fwd|dx|dxplain|dw [M N K] [reps]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1811_01457_b200.gemm import gemm  # noqa: E402

kind = sys.argv[1]
M, N, K = (int(v) for v in (sys.argv[2:5] if len(sys.argv) > 4 else (32768, 1024, 1024)))
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
bf = torch.bfloat16
X = (torch.rand((M, K), device="cuda") * 2 - 1).to(bf)
W = ((torch.rand((N, K), device="cuda") * 2 - 1) * 0.03).to(bf)
dZ = ((torch.rand((M, N), device="cuda") * 2 - 1) * 1e-3).to(bf)
H = (torch.rand((M, K), device="cuda") * 2 - 1).to(bf)
bias = torch.zeros(N, device="cuda")
Hout = torch.empty((M, N), dtype=bf, device="cuda")
dX = torch.empty((M, K), dtype=bf, device="cuda")
dW = torch.empty((N, K), device="cuda")
cs = torch.empty(((M + 31) // 32, max(N, K)), device="cuda")
X32, dZ32 = X.float(), dZ.float()
fn = {
    "fwd": lambda: gemm(X, W, epilogue="bias_act", act="tanh", bias=bias, out_lp=Hout),
    "dx": lambda: gemm(dZ, W, b_mn=True, epilogue="act_grad", act="tanh", aux=H, out_lp=dX, colsum=cs),
    "dxplain": lambda: gemm(dZ, W, b_mn=True, out_lp=dX),
    "dw": lambda: gemm(dZ, X, a_mn=True, b_mn=True, out=dW),
    "dw32": lambda: gemm(dZ32, X32, a_mn=True, b_mn=True, precision="tf32", out=dW),
    "dx32": lambda: gemm(dZ32, W.float(), b_mn=True, precision="tf32", out=torch.empty((M, K), device="cuda")),
}[kind]
for _ in range(min(reps, 3)):
    fn()
torch.cuda.synchronize()
if reps > 3:
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / reps * 1e3
    K2 = M if kind.startswith("dw") else K
    print(f"{kind} {M}x{N}x{K}: {us:.1f} us, {2 * M * N * K / us / 1e6:.1f} TF/s")
