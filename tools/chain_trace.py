"""Timeline of the persistent GEMM chains of one Dense-chain step (tools only).

Uses the instrumented library (make -C paper_1811_01457_b200/csrc trace).
Per chain launch (forward, backward): span, per-unit period (accumulator
complete -> next accumulator complete of the same pair), epilogue length,
and how long producers waited for dependencies.

  python tools/chain_trace.py W L B
"""
import ctypes
import os
import statistics
import sys

os.environ["SGB200_LIB"] = "libsgb200_trace.so"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_01457_b200 import runtime as rt  # noqa: E402
from paper_1811_01457_b200.dense import Chain, ChainEngine, Dense  # noqa: E402

W, L, B = (int(v) for v in sys.argv[1:4])
ITERS = 512
lib = rt.load_library()
lib.sg_chain_trace_buffer.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
lib.sg_chain_cprof.argtypes = [ctypes.c_int, ctypes.c_void_p]
acts = ("tanh",) * (L - 1) + ("identity",)
chain = Chain(*[Dense(W, W, a) for a in acts]).init_params(np.random.default_rng(0))
e = ChainEngine(chain, B, "mse", "bf16", small=False, gemm_chain=True)
X = torch.rand((B, W), device="cuda")
Y = torch.rand((B, W), device="cuda") * 2 - 1


def step():
    e.load_batch(X, Y)
    e.forward()
    e.loss_and_seed()
    e.pullback()


for _ in range(3):
    step()
torch.cuda.synchronize()
buf = torch.zeros(2 * 148 * ITERS * 4, dtype=torch.int64, device="cuda")
rt.check(lib.sg_chain_trace_buffer(buf.data_ptr(), ITERS, 2))
step()
torch.cuda.synchronize()
rt.check(lib.sg_chain_trace_buffer(None, 0, 0))
t = buf.view(2, 148, ITERS, 4).cpu().numpy().astype("float64")
for k, name in enumerate(("forward chain", "backward chain")):
    tk = t[k]
    t0 = tk[tk > 0].min()
    period, epi, chunks, sig, gap_next, busy = [], [], [], [], [], 0.0
    nunits = 0
    for c in range(0, 148, 2):
        prev_af = None
        for i in range(ITERS):
            ms_, af, cd, ee = tk[c, i]
            if af == 0:
                break
            nunits += 1
            epi.append(ee - af)
            chunks.append(cd - af)
            sig.append(ee - cd)
            if i + 1 < ITERS and tk[c, i + 1, 1] > 0:
                gap_next.append(tk[c, i + 1, 1] - ee)  # epilogue idle: waiting for the next accumulator
            if prev_af is not None:
                period.append(af - prev_af)
            busy += af - max(ms_, prev_af if prev_af is not None else ms_)
            prev_af = af
    end = tk[:, :, 3].max()
    span = end - t0
    med = lambda v: statistics.median(v) / 1e3 if v else float("nan")  # noqa: E731
    pct = lambda v, q: float(np.percentile(v, q)) / 1e3 if v else float("nan")  # noqa: E731
    print(f"{name}: {nunits} units, span {span / 1e3:.1f} us, unit period median {med(period):.2f} "
          f"(p90 {pct(period, 90):.2f}) us, epilogue median {med(epi):.2f} us, "
          f"(chunks {med(chunks):.2f}, signal/fix-up {med(sig):.2f}, then idle {med(gap_next):.2f}), "
          f"MMA busy {busy / 74 / span * 100:.1f} % of span per pair")

# epilogue stage profile of the chained step (lane 0 of every warp of CTAs 0-7)
prof = (ctypes.c_ulonglong * 8)()
rt.check(lib.sg_chain_cprof(1, None))
step()
torch.cuda.synchronize()
rt.check(lib.sg_chain_cprof(0, prof))
tot = sum(prof[:5]) or 1
names = ["TMEM load", "aux wait", "math", "stores", "colsum"]
print("epilogue cycles per stage (share):", ", ".join(f"{n} {prof[k] / tot * 100:.0f}%" for k, n in enumerate(names)),
      f"total {tot / 1e6:.1f} Mcycles")

