"""Epilogue stage profile of one GEMM (trace build, SGB200_LIB=.../libsgb200_trace.so):
cycles per stage summed over the lane-0 threads of the first 8 CTAs.

    SGB200_LIB=paper_1811_01457_b200/_lib/libsgb200_trace.so python tools/epi_cprof.py M N K mode
mode: bias_act_f32 | bias_act_bf16 | bias_mse
"""
import ctypes
import sys

import torch

from paper_1811_01457_b200 import runtime as rt
from paper_1811_01457_b200.gemm import gemm

STAGES = ["tmem_ld", "aux/targets wait", "bias+act math", "stores issued", "column sums", "mse targets+dz", "bias load+add (or mse next issue)", "mse loss reduce+store"]


def main():
    M, N, K = (int(v) for v in sys.argv[1:4])
    mode = sys.argv[4]
    lib = rt.load_library()
    lib.sg_gemm_cprof.argtypes = [ctypes.c_int, ctypes.c_void_p]
    g = torch.Generator(device="cuda").manual_seed(0)
    H = (torch.rand((M, K), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    W = ((torch.rand((N, K), generator=g, device="cuda") * 2 - 1) * K ** -0.5).to(torch.bfloat16)
    b = torch.rand(N, generator=g, device="cuda") * 0.1
    Y = torch.rand((M, N), generator=g, device="cuda") * 2 - 1
    Z = torch.empty((M, N), device="cuda")
    dz = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    cs = torch.empty(((M + 31) // 32, N), device="cuda")
    part = torch.zeros(((M + 31) // 32) * ((N + 31) // 32), dtype=torch.float64, device="cuda")

    def run():
        if mode == "bias_act_f32":
            gemm(H, W, epilogue="bias_act", bias=b, out=Z)
        elif mode == "bias_act_bf16":
            gemm(H, W, epilogue="bias_act", bias=b, out_lp=dz, colsum=cs)
        else:
            gemm(H, W, epilogue="bias_mse", bias=b, seed=Y, out2_lp=dz, colsum=cs, loss_part=part, loss_scale=1.0 / M)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    rt.check(lib.sg_gemm_cprof(1, None))
    run()
    torch.cuda.synchronize()
    out = (ctypes.c_ulonglong * 8)()
    rt.check(lib.sg_gemm_cprof(0, out))
    tot = sum(out)
    print(f"{M}x{N}x{K} {mode}: " + "  ".join(f"{STAGES[k]} {out[k] / max(tot, 1) * 100:.1f}% ({out[k] / 1e6:.2f} Mcyc)"
                                              for k in range(8) if out[k]))


if __name__ == "__main__":
    main()
