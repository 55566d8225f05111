"""Tile timeline of the CTA-pair GEMM (tools only).

Loads the instrumented library (make -C paper_1811_01457_b200/csrc trace ->
_lib/libsgb200_trace.so, %globaltimer stamps compiled in) and, for the
Dense-layer products of a shape, prints per-tile medians over all CTAs:
  mainloop = MMA start -> accumulator complete (epilogue wake-up)
  epilogue = accumulator complete -> last epilogue warp done
  period   = accumulator complete -> next accumulator complete (per-tile throughput;
             the ideal is the tile's MMA time at the measured 1664 TF/s burst peak)
  mma_wait = MMA start of a tile - the previous tile's accumulator complete
             (negative: issued ahead; positive: the tensor pipe idled)
and the kernel span (first MMA start -> last epilogue end).

  python tools/gemm_trace.py [M N K]      (default: the c5 layer 32768 1024 1024)
"""
import ctypes
import os
import statistics
import sys

os.environ["SGB200_LIB"] = "libsgb200_trace.so"
import torch  # noqa: E402

from paper_1811_01457_b200 import runtime as rt  # noqa: E402
from paper_1811_01457_b200.gemm import gemm  # noqa: E402

M, N, K = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (32768, 1024, 1024)))
ITERS = 64
lib = rt.load_library()
lib.sg_gemm_trace_buffer.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = torch.zeros(148 * ITERS * 4, dtype=torch.int64, device="cuda")
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
    "dX   act'(tanh)+colsum -> bf16": lambda: gemm(dZ, W, b_mn=True, epilogue="act_grad", act="tanh", aux=Hprev,
                                                 out_lp=dX, colsum=cs),
    "dX   plain -> bf16": lambda: gemm(dZ, W, b_mn=True, out_lp=dX),
    "dW   (split-K) -> f32": lambda: gemm(dZ, X, a_mn=True, b_mn=True, out=dW),
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
    buf.zero_()
    rt.check(lib.sg_gemm_trace_buffer(buf.data_ptr(), ITERS))
    fn()
    torch.cuda.synchronize()
    rt.check(lib.sg_gemm_trace_buffer(None, 0))
    t = buf.view(148, ITERS, 4).cpu().numpy().astype("float64")
    main, epi, wait, epi0, period = [], [], [], [], []
    t0 = t[t > 0].min()
    span_end = t[:, :, 3].max()
    starts = []
    for c in range(0, 148, 2):  # leader CTAs hold the MMA stamps
        for i in range(ITERS):
            ms_, af, e0, e7 = t[c, i]
            if ms_ == 0 or af == 0:
                break
            starts.append(ms_)
            main.append(af - ms_)
            epi.append(max(e7, t[c + 1, i, 3]) - af)
            epi0.append(e0 - af)
            if i > 0 and t[c, i - 1, 1] > 0:
                wait.append(ms_ - t[c, i - 1, 1])
                period.append(af - t[c, i - 1, 1])
    med = lambda v: statistics.median(v) / 1e3 if v else float("nan")  # noqa: E731
    print(f"{name:32s} {us:7.1f} us ({2 * M * N * K / us / 1e6:6.1f} TF/s) tiles/CTA-pair {len(main) / 74:4.1f}: "
          f"period {med(period):5.2f} us (ideal {2 * 256 * 256 * K / 22.5e6:4.2f}), mainloop {med(main):5.2f}, epilogue {med(epi):5.2f} (warp0 {med(epi0):5.2f}), "
          f"mma idle after prev acc {med(wait):5.2f}, first MMA at +{(min(starts) - t0) / 1e3:5.2f}, "
          f"span {(span_end - t0) / 1e3:6.1f} us")
