"""One GEMM through a single-problem persistent chain vs the standalone
CTA-pair kernel (tools only): the chain kernel's per-unit cost."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1811_01457_b200.dense import _pair_splits  # noqa: E402
from paper_1811_01457_b200.gemm import GemmChain, gemm, gemm_desc  # noqa: E402

M, N, K = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (32768, 1024, 1024)))
bf = torch.bfloat16
X = (torch.rand((M, K), device="cuda") * 2 - 1).to(bf)
W = ((torch.rand((N, K), device="cuda") * 2 - 1) * 0.03).to(bf)
dZ = ((torch.rand((M, N), device="cuda") * 2 - 1) * 1e-3).to(bf)
H = (torch.rand((M, K), device="cuda") * 2 - 1).to(bf)
bias = torch.zeros(N, device="cuda")
Hout = torch.empty((M, N), dtype=bf, device="cuda")
dX = torch.empty((M, K), dtype=bf, device="cuda")
dW = torch.empty((N, K), device="cuda")
cs = torch.empty(((M + 31) // 32, K), device="cuda")
kinds = {
    "fwd": dict(A=X, B=W, epilogue="bias_act", act="tanh", bias=bias, out_lp=Hout),
    "dx": dict(A=dZ, B=W, b_mn=True, epilogue="act_grad", act="tanh", aux=H, out_lp=dX, colsum=cs),
    "dw": dict(A=dZ, B=X, a_mn=True, b_mn=True, out=dW),
}


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


for name, kw in kinds.items():
    kw = dict(kw)
    A, B = kw.pop("A"), kw.pop("B")
    t_std = timeit(lambda: gemm(A, B, **kw))
    splits = _pair_splits(N, K, M, 74) if name == "dw" else 1
    ch = GemmChain([(gemm_desc(A, B, **kw), splits, [])])
    t_ch = timeit(ch.run)
    print(f"{name:4s} {M}x{N}x{K}: standalone {t_std:7.1f} us, one-problem chain {t_ch:7.1f} us "
          f"({t_ch / t_std:.2f}x), chain units {ch.units}")
    ch.close()
