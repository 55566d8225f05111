"""Time one tcgen05 GEMM shape per precision/layout (CUDA events, 20 reps)."""
import sys

import torch

from paper_1811_01457_b200.gemm import gemm


def main():
    M, N, K = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 4096, 4096)))
    for prec, dt in (("bf16", torch.bfloat16), ("tf32", torch.float32)):
        for a_mn, b_mn in ((False, False), (False, True), (True, True)):
            A = torch.randn((K, M) if a_mn else (M, K), device="cuda").to(dt)
            B = torch.randn((K, N) if b_mn else (N, K), device="cuda").to(dt)
            out = torch.empty((M, N), device="cuda")
            for _ in range(3):
                gemm(A, B, a_mn=a_mn, b_mn=b_mn, precision=prec, out=out)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(20):
                gemm(A, B, a_mn=a_mn, b_mn=b_mn, precision=prec, out=out)
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / 20
            print(f"{prec} a_mn={a_mn} b_mn={b_mn} {M}x{N}x{K}: {ms:.4f} ms {2*M*N*K/ms/1e9:.1f} TF/s")


if __name__ == "__main__":
    main()
