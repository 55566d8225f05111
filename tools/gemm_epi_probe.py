"""c5-shaped GEMM (32768 x 1024 x 1024, bf16) with different epilogues: how much of
the tile time the epilogue costs when K is short."""
import sys

import torch

from paper_1811_01457_b200.gemm import gemm

M, N, K = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (32768, 1024, 1024)))
A = torch.randn((M, K), device="cuda").to(torch.bfloat16)
W = torch.randn((N, K), device="cuda").to(torch.bfloat16)
bias = torch.randn(N, device="cuda")
out32 = torch.empty((M, N), device="cuda")
outlp = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
aux = torch.rand((M, N), device="cuda").to(torch.bfloat16)
cs = torch.empty(((M + 31) // 32, N), device="cuda")
cases = {
    "store_f32": lambda: gemm(A, W, out=out32),
    "store_bf16": lambda: gemm(A, W, out_lp=outlp),
    "bias_tanh_bf16": lambda: gemm(A, W, epilogue="bias_act", act="tanh", bias=bias, out_lp=outlp),
    "act_grad_bf16_colsum": lambda: gemm(A, W, epilogue="act_grad", act="tanh", aux=aux, out_lp=outlp, colsum=cs),
}
for name, fn in cases.items():
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 50
    print(f"{name:22s} {ms * 1e3:7.1f} us  {2 * M * N * K / ms / 1e9:7.1f} TF/s")
