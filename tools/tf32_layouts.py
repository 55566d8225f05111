"""TF32 tcgen05 GEMM per operand layout beside cuBLAS TF32 on the same products
(the three Dense-layer products of c3: fwd X.W^T, dX dZ.W, dW dZ^T.X)."""
import torch

from paper_1811_01457_b200.gemm import gemm

torch.backends.cuda.matmul.allow_tf32 = True


def t(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


B, D = 8192, 4096
X = torch.randn(B, D, device="cuda")
W = torch.randn(D, D, device="cuda")
dZ = torch.randn(B, D, device="cuda")
o = torch.empty(B, D, device="cuda")
ow = torch.empty(D, D, device="cuda")
fl = 2 * B * D * D
for name, ours, cub in (
    ("fwd X.W^T   (K-major, K-major)", lambda: gemm(X, W, precision="tf32", out=o), lambda: torch.matmul(X, W.t(), out=o)),
    ("dX  dZ.W    (K-major, MN-major)", lambda: gemm(dZ, W, b_mn=True, precision="tf32", out=o),
     lambda: torch.matmul(dZ, W, out=o)),
    ("dW  dZ^T.X  (MN-major, MN-major)", lambda: gemm(dZ, X, a_mn=True, b_mn=True, precision="tf32", out=ow),
     lambda: torch.matmul(dZ.t(), X, out=ow)),
):
    a, c = t(ours), t(cub)
    print(f"{name}: ours {fl / a / 1e9:7.1f} TF/s | cuBLAS {fl / c / 1e9:7.1f} TF/s")
