"""Tile timelines of the CTA-pair GEMM (tools only).

Loads the instrumented library (make -C paper_1811_01457_b200/csrc trace ->
_lib/libsgb200_trace.so: %globaltimer stamps compiled in, launches numbered
on the device).

  python tools/gemm_trace.py gemm [M N K]    single GEMMs of a Dense layer's three products
  python tools/gemm_trace.py step W L B      one Trainer step (CUDA graph) of an L x W MLP at batch B

gemm: per-tile medians over all CTAs --
  period   = accumulator complete -> next accumulator complete (per-tile throughput)
  epilogue = accumulator complete -> last epilogue warp done
  span     = first MMA start -> last epilogue end of the launch (vs the CUDA-event time)
step: per GEMM launch of the step, in stream order: span, and the gap from
  the previous GEMM's last epilogue end to this one's first MMA start (the
  launch / prologue / pipeline-fill cost that a persistent chain would hide).
"""
import ctypes
import os
import statistics
import sys

os.environ["SGB200_LIB"] = "libsgb200_trace.so"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_01457_b200 import runtime as rt  # noqa: E402
from paper_1811_01457_b200.gemm import gemm  # noqa: E402

ITERS = 64
lib = rt.load_library()
lib.sg_gemm_trace_buffer.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]


def traced(fn, launches):
    buf = torch.zeros(launches * 148 * ITERS * 4, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    rt.check(lib.sg_gemm_trace_buffer(buf.data_ptr(), ITERS, launches))
    fn()
    torch.cuda.synchronize()
    rt.check(lib.sg_gemm_trace_buffer(None, 0, 0))
    return buf.view(launches, 148, ITERS, 4).cpu().numpy().astype("float64")


def launch_stats(t):
    """(first MMA start, last epilogue end, per-tile periods, epilogues) of one launch."""
    main, epi, period = [], [], []
    for c in range(0, 148, 2):
        for i in range(ITERS):
            ms_, af = t[c, i, 0], t[c, i, 1]
            if ms_ == 0 or af == 0:
                break
            main.append(af - ms_)
            epi.append(max(t[c, i, 3], t[c + 1, i, 3]) - af)
            if i > 0 and t[c, i - 1, 1] > 0:
                period.append(af - t[c, i - 1, 1])
    starts = t[:, :, 0][t[:, :, 0] > 0]
    ends = t[:, :, 3][t[:, :, 3] > 0]
    if not len(starts):
        return None
    return starts.min(), ends.max(), period, epi, main


def med(v):
    return statistics.median(v) / 1e3 if v else float("nan")


def gemm_mode(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(0)
    bf = torch.bfloat16
    X = (torch.rand((M, K), generator=g, device="cuda") * 2 - 1).to(bf)
    W = ((torch.rand((N, K), generator=g, device="cuda") * 2 - 1) * 0.03).to(bf)
    dZ = ((torch.rand((M, N), generator=g, device="cuda") * 2 - 1) * 1e-3).to(bf)
    Hprev = (torch.rand((M, K), generator=g, device="cuda") * 2 - 1).to(bf)
    bias = torch.zeros(N, device="cuda")
    Hout = torch.empty((M, N), dtype=bf, device="cuda")
    dX = torch.empty((M, K), dtype=bf, device="cuda")
    dW = torch.empty((N, K), device="cuda")
    cs = torch.empty(((M + 31) // 32, max(N, K)), device="cuda")
    cases = {
        "fwd  bias+tanh -> bf16": lambda: gemm(X, W, epilogue="bias_act", act="tanh", bias=bias, out_lp=Hout),
        "dX   act'(tanh)+colsum -> bf16": lambda: gemm(dZ, W, b_mn=True, epilogue="act_grad", act="tanh",
                                                     aux=Hprev, out_lp=dX, colsum=cs),
        "dX   act'(tanh) -> bf16": lambda: gemm(dZ, W, b_mn=True, epilogue="act_grad", act="tanh", aux=Hprev,
                                              out_lp=dX),
        "dX   plain -> bf16": lambda: gemm(dZ, W, b_mn=True, out_lp=dX),
        "dW   -> f32": lambda: gemm(dZ, X, a_mn=True, b_mn=True, out=dW),
    }
    for name, fn in cases.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            fn()
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) / 20 * 1e3
        t = traced(lambda: [fn() for _ in range(8)], 8)
        spans, gaps = [], []
        prev_end = None
        allp, alle = [], []
        for k in range(8):
            st = launch_stats(t[k])
            if st is None:
                continue
            a, b, period, epi, _ = st
            spans.append(b - a)
            if prev_end is not None:
                gaps.append(a - prev_end)
            prev_end = b
            allp += period
            alle += epi
        print(f"{name:32s} {us:7.1f} us/launch ({2 * M * N * K / us / 1e6:6.1f} TF/s): tile period {med(allp):5.2f} us, "
              f"epilogue {med(alle):5.2f}, span {med(spans):6.1f} us, gap to the next launch {med(gaps):5.2f} us")


def step_mode(W, L, B):
    from paper_1811_01457_b200.dense import Chain, Dense
    from paper_1811_01457_b200.train import Trainer

    acts = ("tanh",) * (L - 1) + ("identity",)
    chain = Chain(*[Dense(W, W, a) for a in acts]).init_params(np.random.default_rng(0))
    tr = Trainer(chain, B, loss="mse", lr=1e-4, precision="bf16", graph=True)
    X = torch.rand((B, W), device="cuda")
    Y = torch.rand((B, W), device="cuda") * 2 - 1
    for _ in range(5):
        tr.step(X, Y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        tr.step(X, Y)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    n = 3 * L
    t = traced(lambda: tr.step(X, Y), n)
    rows = []
    for k in range(n):
        st = launch_stats(t[k])
        if st is None:
            break
        rows.append(st)
    t0 = rows[0][0]
    tot_gap = 0.0
    print(f"step {L}x{W} batch {B}: {ms * 1e3:.1f} us/step (graph), {len(rows)} pair-GEMM launches traced")
    for k, (a, b, period, epi, main) in enumerate(rows):
        gap = (a - rows[k - 1][1]) if k else 0.0
        tot_gap += gap
        print(f"  #{k:2d} start +{(a - t0) / 1e3:8.1f} span {(b - a) / 1e3:6.1f} gap {gap / 1e3:5.1f} "
              f"period {med(period):5.2f} epi {med(epi):5.2f} main {med(main):5.2f}")
    print(f"  total span {(rows[-1][1] - t0) / 1e3:.1f} us, sum of gaps {tot_gap / 1e3:.1f} us")


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "gemm"
    if mode == "step":
        step_mode(*(int(v) for v in sys.argv[2:5]))
    else:
        gemm_mode(*(int(v) for v in (sys.argv[2:5] if len(sys.argv) > 4 else (32768, 1024, 1024))))
