"""cuBLAS (torch.matmul, bf16) beside our tcgen05 GEMMs on the three Dense-layer
products of a width-W layer at batch B (default: c5, W=1024, B=32768)."""
import sys

import torch

from paper_1811_01457_b200.gemm import gemm

W, B = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (1024, 32768)))


def t(fn, reps=50):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


X = torch.randn((B, W), device="cuda").to(torch.bfloat16)
Wt = torch.randn((W, W), device="cuda").to(torch.bfloat16)
dZ = torch.randn((B, W), device="cuda").to(torch.bfloat16)
H = torch.rand((B, W), device="cuda").to(torch.bfloat16)
bias = torch.randn(W, device="cuda")
o_lp = torch.empty((B, W), dtype=torch.bfloat16, device="cuda")
o_w = torch.empty((W, W), device="cuda")
o_wlp = torch.empty((W, W), dtype=torch.bfloat16, device="cuda")
cs = torch.empty(((B + 31) // 32, W), device="cuda")
fl = 2 * B * W * W
rows = {
    "fwd  Z=X.W^T": (lambda: torch.matmul(X, Wt.t(), out=o_lp),
                     lambda: gemm(X, Wt, epilogue="bias_act", act="tanh", bias=bias, out_lp=o_lp)),
    "dX   dZ.W": (lambda: torch.matmul(dZ, Wt, out=o_lp),
                  lambda: gemm(dZ, Wt, b_mn=True, epilogue="act_grad", act="tanh", aux=H, out_lp=o_lp, colsum=cs)),
    "dW   dZ^T.X": (lambda: torch.matmul(dZ.t(), X, out=o_wlp),
                    lambda: gemm(dZ, X, a_mn=True, b_mn=True, out=o_w)),
}
for name, (cub, ours) in rows.items():
    tc, to = t(cub), t(ours)
    print(f"{name:14s} B={B} W={W}: cuBLAS {tc:7.1f} us {fl / tc / 1e6:7.1f} TF/s | ours (fused epilogue) {to:7.1f} us "
          f"{fl / to / 1e6:7.1f} TF/s")
