import torch
from paper_1811_01457_b200.gemm import gemm
M, N, K = 8192, 4096, 4096
A = torch.randn((M, K), device="cuda").to(torch.bfloat16)
W = (torch.randn((N, K), device="cuda") * 0.02).to(torch.bfloat16)
bias = torch.randn(N, device="cuda")
seed = torch.randn((M, N), device="cuda")
h = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
dz = torch.empty_like(h)
cs = torch.empty(((M + 31) // 32, N), device="cuda")
cases = {
  "bias_act": lambda: gemm(A, W, epilogue="bias_act", act="sigmoid", bias=bias, out_lp=h),
  "bias_act+colsum": lambda: gemm(A, W, epilogue="bias_act", act="sigmoid", bias=bias, out_lp=h, colsum=cs),
  "seed": lambda: gemm(A, W, epilogue="bias_act_seed", act="sigmoid", bias=bias, seed=seed, out_lp=h, out2_lp=dz, colsum=cs),
  "seed_nocolsum": lambda: gemm(A, W, epilogue="bias_act_seed", act="sigmoid", bias=bias, seed=seed, out_lp=h, out2_lp=dz),
}
for rep in range(2):
  for name, fn in cases.items():
    for _ in range(3): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): fn()
    e.record(); torch.cuda.synchronize()
    us = s.elapsed_time(e) / 20 * 1e3
    print(f"{name:18s} {us:7.1f} us {2*M*N*K/us/1e6:7.1f} TF/s")
