"""Top-layer forward GEMM + MSE loss, separate (bias_act into fp32 z, then
sg_loss) vs fused (bias_mse epilogue): CUDA-event times per piece, interleaved.

    python tools/mse_epi_probe.py M N K [reps]
"""
import statistics
import sys

import torch

from paper_1811_01457_b200 import runtime as rt
from paper_1811_01457_b200.dense import LOSSES, _dt, _lib, _p
from paper_1811_01457_b200.gemm import gemm


def main():
    M, N, K = (int(v) for v in sys.argv[1:4])
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    g = torch.Generator(device="cuda").manual_seed(0)
    H = (torch.rand((M, K), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    W = ((torch.rand((N, K), generator=g, device="cuda") * 2 - 1) * K ** -0.5).to(torch.bfloat16)
    b = torch.rand(N, generator=g, device="cuda") * 0.1
    Y = torch.rand((M, N), generator=g, device="cuda") * 2 - 1
    Z = torch.empty((M, N), device="cuda")
    dz = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    cs = torch.empty(((M + 31) // 32, N), device="cuda")
    part = torch.zeros(max(((M + 31) // 32) * ((N + 31) // 32), (M + 31) // 32 * ((N + 511) // 512)),
                       dtype=torch.float64, device="cuda")
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    lib = _lib()
    scale = 1.0 / M

    def sep_gemm():
        gemm(H, W, epilogue="bias_act", bias=b, out=Z)

    def sep_loss():
        rt.check(lib.sg_loss(rt.context(), LOSSES["mse"], _p(Z), _dt(Z), Z.stride(0), _p(Y), Y.stride(0), M, N,
                             scale, _p(loss), _p(part), part.numel(), _p(dz), _dt(dz), dz.stride(0), None, 0, 0,
                             _p(cs), cs.stride(0), rt.stream_ptr()), "sg_loss")

    def fused():
        gemm(H, W, epilogue="bias_mse", bias=b, seed=Y, out2_lp=dz, colsum=cs, loss_part=part, loss_scale=scale)

    def plain_store_bf16():
        gemm(H, W, epilogue="bias_act", bias=b, out_lp=dz)

    def store_bf16_colsum():
        gemm(H, W, epilogue="bias_act", bias=b, out_lp=dz, colsum=cs)

    def fused_nocs():
        gemm(H, W, epilogue="bias_mse", bias=b, seed=Y, out2_lp=dz, loss_part=part, loss_scale=scale)

    fns = {"gemm bias_act fp32 z": sep_gemm, "sg_loss (mse)": sep_loss, "gemm bias_mse (fused)": fused,
           "gemm bias_act bf16 out (floor)": plain_store_bf16, "gemm bias_act bf16 + colsum": store_bf16_colsum,
           "gemm bias_mse without colsum": fused_nocs}
    for f in fns.values():
        for _ in range(3):
            f()
    t = {k: [] for k in fns}
    for r in range(reps):
        for k, f in fns.items():
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            f()
            e.record()
            torch.cuda.synchronize()
            t[k].append(s.elapsed_time(e))
    tf = 2.0 * M * N * K / 1e12
    for k, v in t.items():
        m = statistics.median(v)
        print(f"{M}x{N}x{K} {k:34s} median {m * 1e3:8.1f} us  ({tf / (m * 1e-3):7.1f} TF/s-equiv)")
    print(f"separate total {sum(statistics.median(t[k]) for k in list(fns)[:2]) * 1e3:.1f} us")


if __name__ == "__main__":
    main()
