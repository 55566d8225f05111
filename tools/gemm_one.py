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
fn = {
    "fwd": lambda: gemm(X, W, epilogue="bias_act", act="tanh", bias=bias, out_lp=Hout),
    "dx": lambda: gemm(dZ, W, b_mn=True, epilogue="act_grad", act="tanh", aux=H, out_lp=dX, colsum=cs),
    "dxplain": lambda: gemm(dZ, W, b_mn=True, out_lp=dX),
    "dw": lambda: gemm(dZ, X, a_mn=True, b_mn=True, out=dW),
}[kind]
for _ in range(reps):
    fn()
torch.cuda.synchronize()
