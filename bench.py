"""Benchmark of the sgb200 hot path (contract: one JSON line on rank 0).

Headline workload (BASELINE.json configs[1]): fused broadcast of the user
function sigma.(a .* x .+ b) and its gradient over 2^28 fp32 elements,
x of shape (65536, 4096), a and b of shape (4096,).  One *step* = the
forward kernel K1 (y = f.(a, x, b)) + the fused adjoint K2 (xbar, abar,
bbar from ybar).  Algorithmic traffic is 20 B/element (fwd: read x, write
y; grad: read x and ybar, write xbar), 5.37 GB per step.
Inputs are 1 GiB each, larger than L2 (126 MB), so no L2 flush is needed.

Multi-GPU: the fused broadcast does not shard: N ranks run
N independent replicas ("scaling": "weak"), timed as the max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

AFFSIG = """
func @affsig(%a: f64, %x: f64, %b: f64) -> f64 {
^entry:
  %m = mul %a, %x
  %s = add %m, %b
  %y = sigmoid %s
  ret %y
}
"""
R_ROWS, C_COLS = 65536, 4096          # 2^28 elements
BYTES_PER_ELEM = 20                    # fwd 8 + grad 12
METRIC = "fused-broadcast GB/s vs HBM peak"


def traffic_of(kernel: str, applicable: bool):
    """DRAM bytes per launch of `kernel` from the committed ncu capture (profiles/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not applicable or not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(kernel, {}).get("bytes")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "bf16_tflops": d.get("bf16_tflops", 1590.0),
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", 1400.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback"}


# ------------------------------------------------------------ dist plumbing
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world, local):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist if world > 1 else None


def barrier(dist):
    import torch

    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(dist, v: float) -> float:
    import torch

    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, device_index: int, period_s: float = float(os.environ.get("SGB200_CLOCK_PERIOD", "0.002"))):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self.period = period_s
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self.nv = None
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join()

    def summary(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "nvml unavailable"}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------- broadcast (c2)
def c2_config(R, C, world):
    """The headline workload's config, shared by both arms (the reference arm
    measures the same workload on a bounded CPU sample, see cpu_baseline.sample)."""
    return {"workload": "c2 fused broadcast sigma.(a.*x.+b) + gradient, 2^28 fp32 elements",
            "shape": [R, C], "broadcast": "a,b of shape (4096,)",
            "bytes_per_elem": BYTES_PER_ELEM, "l2": "inputs 1 GiB each > 126 MB L2, no flush",
            "parallelism": f"replicas x{world}"}


def broadcast_bench(args, world, rank, local, dist):
    import torch

    from paper_1811_01457_b200 import fused as F
    from paper_1811_01457_b200.irtext import parse_ir

    module = parse_ir(AFFSIG)
    R, C = args.rows, C_COLS
    n = R * C
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    x = torch.rand((R, C), generator=g, device="cuda") * 4 - 2          # U[-2,2] (progen range)
    a = torch.rand((C,), generator=g, device="cuda") * 4 - 2
    b = torch.rand((C,), generator=g, device="cuda") * 4 - 2
    yb = torch.rand((R, C), generator=g, device="cuda") * 2 - 1         # seed ybar ~ U[-1,1]
    y = torch.empty_like(x)
    xbar = torch.empty_like(x)
    abar = torch.empty_like(a)
    bbar = torch.empty_like(b)
    stream = torch.cuda.current_stream()

    def step():
        F.fused_map(module, "affsig", [a, x, b], out=y, check=False)
        F.fused_map_grad(module, "affsig", [a, x, b], yb, check=False, outs=[abar, xbar, bbar])

    for _ in range(args.warmup):
        step()
    F.check_errors(module, "affsig")
    barrier(dist)
    # the timed region: exactly the steps, nothing recorded between the kernels
    # (the fused kernels are launched with programmatic dependent launch)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record(stream)
        for i in range(args.steps):
            step()
        stop.record(stream)
        torch.cuda.synchronize()
    barrier(dist)
    ms_total = start.elapsed_time(stop)
    ms_total = max_over_ranks(dist, ms_total)
    # per-kernel split (K1 | K2 + finalize).  K1 is timed alone, back to back
    # with events only around the loop, and K2 + finalize is the step minus
    # that: events recorded BETWEEN the kernels stretch K2 by 35-50 us (the
    # event split below adds up to more than the measured step;
    # tools/c2_context_probe.py), so they only go into "event_split".
    n_ev = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n_ev):
        F.fused_map(module, "affsig", [a, x, b], out=y, check=False)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_step = ms_total / args.steps
    fwd_ms = e0.elapsed_time(e1) / n_ev
    grad_ms = ms_step - fwd_ms
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_ev)]
    for i in range(n_ev):
        ev[i][0].record(stream)
        F.fused_map(module, "affsig", [a, x, b], out=y, check=False)
        ev[i][1].record(stream)
        F.fused_map_grad(module, "affsig", [a, x, b], yb, check=False, outs=[abar, xbar, bbar])
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    event_split = {"fwd_K1": round(statistics.mean(e[0].elapsed_time(e[1]) for e in ev), 4),
                   "grad_K2_plus_finalize": round(statistics.mean(e[1].elapsed_time(e[2]) for e in ev), 4)}
    F.check_errors(module, "affsig")
    value = world * n * BYTES_PER_ELEM / (ms_step * 1e-3) / 1e9

    # e2e through the public API with pinned host buffers (H2D x, ybar; D2H y, xbar, abar, bbar)
    hx = torch.empty((R, C), dtype=torch.float32, pin_memory=True)
    hyb = torch.empty_like(hx, pin_memory=True)
    hy = torch.empty_like(hx, pin_memory=True)
    hxb = torch.empty_like(hx, pin_memory=True)
    ha, hb = torch.empty((C,), pin_memory=True), torch.empty((C,), pin_memory=True)
    hx.copy_(x, non_blocking=False)
    hyb.copy_(yb, non_blocking=False)
    dx_in, dyb_in = torch.empty_like(x), torch.empty_like(yb)
    e2e_steps = max(3, min(args.steps, 10))

    def e2e_step():
        dx_in.copy_(hx, non_blocking=True)
        dyb_in.copy_(hyb, non_blocking=True)
        F.fused_map(module, "affsig", [a, dx_in, b], out=y, check=False)
        F.fused_map_grad(module, "affsig", [a, dx_in, b], dyb_in, check=False, outs=[abar, xbar, bbar])
        hy.copy_(y, non_blocking=True)
        hxb.copy_(xbar, non_blocking=True)
        ha.copy_(abar, non_blocking=True)
        hb.copy_(bbar, non_blocking=True)

    e2e_step()
    barrier(dist)
    s2, t2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    t2.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(dist, s2.elapsed_time(t2)) / e2e_steps
    F.check_errors(module, "affsig")
    h2d = 2 * n * 4
    d2h = 2 * n * 4 + 2 * C * 4
    e2e_serial_ms = e2e_ms

    # pipelined e2e: row chunks on three streams so H2D of chunk i+1, the
    # kernels of chunk i and D2H of chunk i-1 overlap (PCIe is full duplex);
    # the broadcast-axis cotangents are summed over chunks with reduce_to.
    # Consecutive steps overlap too: a chunk's buffers are reused as soon as
    # the previous step is done with them (per-chunk events guard the
    # write-after-read hazards), so the pipeline fills once per timed run.
    nch = next(c for c in (int(os.environ.get("SGB200_E2E_CHUNKS", "16")), 16, 8, 1) if R % c == 0)
    rc = R // nch
    s_in, s_cp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    apart = torch.empty((nch, C), device="cuda")
    bpart = torch.empty((nch, C), device="cuda")
    read_done = [None] * nch   # kernels of the previous step finished reading dx_in/dyb_in[chunk]
    out_done = [None] * nch    # D2H of the previous step finished reading y/xbar[chunk]
    red_done = [None]          # previous step's abar/bbar copied out

    def e2e_pipelined():
        start_ev = torch.cuda.Event()
        start_ev.record(stream)
        for st in (s_in, s_cp, s_out):
            st.wait_event(start_ev)
        for i in range(nch):
            sl = slice(i * rc, (i + 1) * rc)
            with torch.cuda.stream(s_in):
                if read_done[i] is not None:
                    s_in.wait_event(read_done[i])
                dx_in[sl].copy_(hx[sl], non_blocking=True)
                dyb_in[sl].copy_(hyb[sl], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            s_cp.wait_event(ev_in)
            if out_done[i] is not None:
                s_cp.wait_event(out_done[i])
            with torch.cuda.stream(s_cp):
                F.fused_map(module, "affsig", [a, dx_in[sl], b], out=y[sl], check=False, stream=s_cp)
                F.fused_map_grad(module, "affsig", [a, dx_in[sl], b], dyb_in[sl], check=False, stream=s_cp,
                                 outs=[apart[i], xbar[sl], bpart[i]])
                ev_c = torch.cuda.Event()
                ev_c.record(s_cp)
            read_done[i] = ev_c
            s_out.wait_event(ev_c)
            with torch.cuda.stream(s_out):
                hy[sl].copy_(y[sl], non_blocking=True)
                hxb[sl].copy_(xbar[sl], non_blocking=True)
                ev_o = torch.cuda.Event()
                ev_o.record(s_out)
            out_done[i] = ev_o
        with torch.cuda.stream(s_cp):
            if red_done[0] is not None:
                s_cp.wait_event(red_done[0])
            F.reduce_to(apart, (C,), out=abar, stream=s_cp)
            F.reduce_to(bpart, (C,), out=bbar, stream=s_cp)
            ev_r = torch.cuda.Event()
            ev_r.record(s_cp)
        s_out.wait_event(ev_r)
        with torch.cuda.stream(s_out):
            ha.copy_(abar, non_blocking=True)
            hb.copy_(bbar, non_blocking=True)
            ev_ro = torch.cuda.Event()
            ev_ro.record(s_out)
        red_done[0] = ev_ro

    def join_all():
        for st in (s_in, s_cp, s_out):
            stream.wait_stream(st)

    e2e_pipelined()
    join_all()
    torch.cuda.synchronize()
    barrier(dist)
    s3, t3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s3.record(stream)
    for _ in range(e2e_steps):
        e2e_pipelined()
    join_all()
    t3.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(dist, s3.elapsed_time(t3)) / e2e_steps
    F.check_errors(module, "affsig")

    # the host link the e2e number is bound by: concurrent H2D + D2H of 256 MB chunks
    # of the same pinned buffers (PCIe is full duplex)
    pc = min(n, 64 << 20)
    pcie_in, pcie_out = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        sp, tp = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sp.record(stream)
        pcie_in.wait_event(sp)
        pcie_out.wait_event(sp)
        with torch.cuda.stream(pcie_in):
            for k in range(4):
                dx_in.view(-1)[:pc].copy_(hx.view(-1)[:pc], non_blocking=True)
        with torch.cuda.stream(pcie_out):
            for k in range(4):
                hy.view(-1)[:pc].copy_(y.view(-1)[:pc], non_blocking=True)
        stream.wait_stream(pcie_in)
        stream.wait_stream(pcie_out)
        tp.record(stream)
        torch.cuda.synchronize()
    pcie_gbps = 4 * pc * 4 / (sp.elapsed_time(tp) * 1e-3) / 1e9  # per direction, both running

    peaks = load_peaks()
    grad_bytes = 12 * n
    achieved = grad_bytes / (grad_ms * 1e-3) / 1e9
    rec = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded U[-2,2] inputs, U[-1,1] seed ybar)",
        "config": c2_config(R, C, world),
        "kernels_ms": {"fwd_K1": round(fwd_ms, 4), "grad_K2_plus_finalize": round(grad_ms, 4),
                       "fwd_GBps": round(8 * n / (fwd_ms * 1e-3) / 1e9, 1),
                       "grad_GBps": round(achieved, 1),
                       "split": "K1 timed alone back to back (events around the loop only); "
                                "K2 + finalize = the timed step minus K1",
                       "event_split": event_split},
        "roofline": {"bound": "hbm", "kernel": "sg_ew_grad (K2, incl. 2 partial-sum finalizers)",
                     "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / peaks["hbm_gbs"], 4),
                     "traffic": traffic_of("sg_ew_grad", R * C == R_ROWS * C_COLS),
                     "peak_source": peaks["source"],
                     "step_frac": round(value / world / peaks["hbm_gbs"], 4)},
        "e2e": {"value": round(world * n * BYTES_PER_ELEM / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": f"fused_map + fused_map_grad public API on {nch} row chunks, pinned host buffers, "
                        "H2D / kernels / D2H overlapped on three streams (also across steps)",
                "pcie_GBps_per_direction_measured": round(pcie_gbps, 1),
                "pcie_bound_ms": round(max(h2d, d2h) / (pcie_gbps * 1e9) * 1e3, 2),
                "serial_ms_per_step": round(e2e_serial_ms, 3),
                "serial_value": round(world * n * BYTES_PER_ELEM / (e2e_serial_ms * 1e-3) / 1e9, 2)},
        "gpu_launches": (count_launches(step) or 4) * args.steps,
        "clocks": clocks.summary(),
    }
    return rec


def cpu_baseline_broadcast(rows=64):
    """Oracle port (per-element interpreter = the reference's algorithm) on a bounded sample."""
    from oracle import scalar as OS
    from paper_1811_01457_b200.irtext import parse_ir

    m = parse_ir(AFFSIG)
    rng = np.random.default_rng(0)
    C = C_COLS
    x = rng.uniform(-2, 2, (rows, C)).astype(np.float32).astype(np.float64)
    a = rng.uniform(-2, 2, C).astype(np.float32).astype(np.float64)
    b = rng.uniform(-2, 2, C).astype(np.float32).astype(np.float64)
    yb = rng.uniform(-1, 1, (rows, C)).astype(np.float32).astype(np.float64)
    n = rows * C
    t0 = time.perf_counter()
    budget = [1 << 60]
    flat_x = x.reshape(-1)
    ys = [OS.eval_scalar(m, "affsig", (a[i % C], flat_x[i], b[i % C]), budget) for i in range(n)]
    t1 = time.perf_counter()
    cols = [OS.eval_dual(m, "affsig", (a[i % C], flat_x[i], b[i % C]), budget) for i in range(n)]
    parts = np.array(cols).T[1:].reshape(3, rows, C)
    OS.fused_map_pullback(list(parts), [(C,), (rows, C), (C,)], yb)
    t2 = time.perf_counter()
    del ys
    # numpy-vectorised restatement ("best CPU" line, multi-threaded ufuncs)
    t3 = time.perf_counter()
    p, pr = OS.vec_eval(m, "affsig", [a, x, b])
    OS.fused_map_pullback(pr, [(C,), (rows, C), (C,)], yb)
    t4 = time.perf_counter()
    sec = t2 - t0
    return {
        "value": round(n * BYTES_PER_ELEM / sec / 1e9, 6),
        "unit": "GB/s",
        "cores": 1,
        "kind": "port",
        "sample": f"{rows}x{C} = {n} elements, fwd (interp.py:322-332) + fused_pack/pullback "
                  f"(forward_ad.py:194-235) via the oracle's per-element interpreter",
        "us_per_elem_fwd": round((t1 - t0) / n * 1e6, 3),
        "us_per_elem_pack": round((t2 - t1) / n * 1e6, 3),
        "extrapolated_s_at_2^28": round(sec / n * (1 << 28), 1),
        "numpy_vectorised_GBps": round(n * BYTES_PER_ELEM / (t4 - t3) / 1e9, 4),
        "host_cores_available": len(os.sched_getaffinity(0)),
    }


# ------------------------------------------------------- dense workloads
def _timed(fn, steps, warmup, dist, stream, per_step_events=None):
    """CUDA-event time of `steps` calls (max over ranks), after `warmup` calls.
    The timed loop records no events between kernels (they break the
    programmatic-dependent-launch overlap and stretch the kernel after them);
    with `per_step_events`, a SEPARATE run of `steps` calls records them for
    the per-kernel split."""
    import torch

    for _ in range(warmup):
        fn(None)
    barrier(dist)
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for i in range(steps):
        fn(None)
    t.record(stream)
    torch.cuda.synchronize()
    barrier(dist)
    ms = max_over_ranks(dist, s.elapsed_time(t)) / steps
    evs = []
    if per_step_events:
        for i in range(steps):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(per_step_events)]
            evs.append(ev)
            fn(ev)
        torch.cuda.synchronize()
    return ms, evs


def broadcast_variant_bench(args, dist, peaks, variant):
    """SURVEY §8(d) c2 variants at the full 2^28 size: scalar a, b (f64 by value;
    full-reduction cotangents), (R,1) a, b (row reductions), or the main
    (C,) a, b case in f64 -- the reference's own dtype, where + - * / round
    exactly like the reference's Python floats (only libm ulps differ)."""
    import statistics

    import torch

    from paper_1811_01457_b200 import fused as F
    from paper_1811_01457_b200.irtext import parse_ir

    module = parse_ir(AFFSIG)
    R, C = args.rows, C_COLS
    n = R * C
    g = torch.Generator(device="cuda").manual_seed(4321)
    dt = torch.float64 if variant == "f64" else torch.float32
    esz = 8 if variant == "f64" else 4
    x = torch.rand((R, C), generator=g, device="cuda", dtype=dt) * 4 - 2
    yb = torch.rand((R, C), generator=g, device="cuda", dtype=dt) * 2 - 1
    y, xbar = torch.empty_like(x), torch.empty_like(x)
    if variant == "f64":
        a = torch.rand(C, generator=g, device="cuda", dtype=dt) * 4 - 2
        b = torch.rand(C, generator=g, device="cuda", dtype=dt) * 4 - 2
        abar, bbar = torch.empty_like(a), torch.empty_like(b)
        desc = "f64 (the reference's dtype), a, b of shape (C,)"
    elif variant == "scalar":
        a, b = 0.7, -0.3
        abar, bbar = torch.empty(1, device="cuda"), torch.empty(1, device="cuda")
        desc = "a, b f64 scalars (full-reduction cotangents)"
    else:
        a = torch.rand((R, 1), generator=g, device="cuda") * 4 - 2
        b = torch.rand((R, 1), generator=g, device="cuda") * 4 - 2
        abar, bbar = torch.empty_like(a), torch.empty_like(b)
        desc = "a, b of shape (R,1) (row-reduction cotangents)"
    stream = torch.cuda.current_stream()

    def step(ev):
        if ev: ev[0].record(stream)
        F.fused_map(module, "affsig", [a, x, b], out=y, check=False)
        if ev: ev[1].record(stream)
        F.fused_map_grad(module, "affsig", [a, x, b], yb, check=False, outs=[abar, xbar, bbar])
        if ev: ev[2].record(stream)

    ms, evs = _timed(step, max(5, args.dense_steps), args.warmup, dist, stream, per_step_events=3)
    F.check_errors(module, "affsig")
    fwd = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    grad = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    bpe = BYTES_PER_ELEM * esz // 4  # 20 B/elem in fp32, 40 in f64
    return {
        "workload": f"c2 variant: sigma.(a.*x.+b) + gradient, 2^28 {'f64' if esz == 8 else 'fp32'}, {desc}",
        "key": {"scalar": "c2 scalar a,b", "col": "c2 (R,1) a,b", "f64": "c2 f64"}[variant],
        "value": round(n * bpe / (ms * 1e-3) / 1e9, 1), "unit": "GB/s", "ms_per_step": round(ms, 4),
        "bytes_per_elem": bpe,
        "kernels_ms": {"fwd_K1": round(fwd, 4), "grad_K2_plus_finalize": round(grad, 4),
                       "fwd_GBps": round(2 * esz * n / (fwd * 1e-3) / 1e9, 1),
                       "grad_GBps": round(3 * esz * n / (grad * 1e-3) / 1e9, 1)},
        "roofline": {"bound": "hbm", "kernel": "sg_ew_grad", "achieved": round(3 * esz * n / (grad * 1e-3) / 1e9, 1),
                     "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(3 * esz * n / (grad * 1e-3) / 1e9 / peaks["hbm_gbs"], 4)},
        "gpu_launches_per_step": 3 if variant == "scalar" else 3,
    }


TF32_PEAK_TFLOPS = 1100.0  # B200_PROFILING.md dense TF32 figure (the fallback when no measurement runs)
_TF32_PEAK = None


def measured_tf32_peak(stream):
    """Dense TF32 peak measured on this box the way MEASURED_PEAKS.json measures
    bf16: cuBLAS (torch.matmul, allow_tf32) fp32 8192^3, best of 10 (burst)."""
    global _TF32_PEAK
    if _TF32_PEAK is None:
        import torch

        torch.backends.cuda.matmul.allow_tf32 = True
        n = 8192
        a = torch.rand((n, n), device="cuda")
        b = torch.rand((n, n), device="cuda")
        for _ in range(3):
            a @ b
        best = float("inf")
        for _ in range(10):
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            a @ b
            s1.record(stream)
            torch.cuda.synchronize()
            best = min(best, s0.elapsed_time(s1))
        _TF32_PEAK = round(2.0 * n ** 3 / (best * 1e-3) / 1e12, 1)
        del a, b
    return _TF32_PEAK


def dense_c3_bench(args, dist, peaks, precision="bf16"):
    """c3: one Dense 4096->4096 (sigmoid) fwd + pullback, batch 8192, bf16 or TF32 tensor cores."""
    import torch

    from paper_1811_01457_b200 import runtime as rt
    from paper_1811_01457_b200.dense import ACT, DenseLayer, _dt, _lib, _p
    from paper_1811_01457_b200.gemm import gemm

    M, D = 8192, 4096
    g = torch.Generator(device="cuda").manual_seed(3)
    layer = DenseLayer(M, D, D, "sigmoid", precision=precision)
    r = (6.0 / (2 * D)) ** 0.5
    layer.W.copy_((torch.rand((D, D), generator=g, device="cuda") * 2 - 1) * r)
    if layer.Wb is not layer.W:
        layer.Wb.copy_(layer.W.to(torch.bfloat16))
    layer.b.copy_((torch.rand(D, generator=g, device="cuda") * 2 - 1) * 0.01)
    layer.X.copy_((torch.rand((M, D), generator=g, device="cuda") * 2 - 1).to(layer.X.dtype))
    tf32 = precision == "tf32"
    Wop = layer.W if tf32 else layer.Wb
    ybar = torch.rand((M, D), generator=g, device="cuda") * 2 - 1
    stream = torch.cuda.current_stream()
    lib, ctx = _lib(), rt.context()

    def step(ev):
        if ev: ev[0].record(stream)
        # the seed is known: the forward epilogue also forms dZ = ybar .* act'(H) (+ column sums)
        if tf32:
            gemm(layer.X, Wop, precision="tf32", epilogue="bias_act_seed", act="sigmoid", bias=layer.b, seed=ybar,
                 out=layer.H, out2_lp=layer.dZ, colsum=layer.colsum)
        else:
            gemm(layer.X, Wop, epilogue="bias_act_seed", act="sigmoid", bias=layer.b, seed=ybar, out_lp=layer.H,
                 out2_lp=layer.dZ, colsum=layer.colsum)
        if ev: ev[1].record(stream)
        if ev: ev[2].record(stream)
        gemm(layer.dZ, Wop, b_mn=True, precision=precision, out=layer.dX)
        if ev: ev[3].record(stream)
        gemm(layer.dZ, layer.X, a_mn=True, b_mn=True, precision=precision, out=layer.dW)
        if ev: ev[4].record(stream)
        rt.check(lib.sg_colsum_finalize(ctx, _p(layer.colsum), (M + 31) // 32, layer.colsum.stride(0), D,
                                        _p(layer.db), rt.stream_ptr()))
        if ev: ev[5].record(stream)

    ms, evs = _timed(step, max(5, args.dense_steps), args.warmup, dist, stream, per_step_events=6)
    names = ["fwd_gemm", "act_grad", "dX_gemm", "dW_gemm", "db_finalize"]
    kms = {n: statistics.mean(e[i].elapsed_time(e[i + 1]) for e in evs) for i, n in enumerate(names)}
    gf = 2.0 * M * D * D
    gemm_ms = kms["fwd_gemm"] + kms["dX_gemm"] + kms["dW_gemm"]
    achieved = 3 * gf / (gemm_ms * 1e-3) / 1e12
    esz = 4 if tf32 else 2
    # context: cuBLAS on the same box and shapes (the library baseline; not on the product path)
    torch.backends.cuda.matmul.allow_tf32 = True
    xa, wa, dza = layer.X.contiguous(), Wop.contiguous(), layer.dZ.contiguous()
    cublas = {}
    for nm, fn in (("fwd_gemm", lambda: xa @ wa.T), ("dX_gemm", lambda: dza @ wa), ("dW_gemm", lambda: dza.T @ xa)):
        for _ in range(3):
            fn()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(10):
            fn()
        s1.record(stream)
        torch.cuda.synchronize()
        cublas[nm] = round(gf / (s0.elapsed_time(s1) / 10 * 1e-3) / 1e12, 1)
    peak = measured_tf32_peak(stream) if tf32 else peaks["bf16_tflops"]
    return {
        "workload": f"c3 Dense 4096->4096 sigmoid fwd+pullback (dX, dW, db), batch 8192, {precision} tcgen05",
        "key": f"c3 {precision}",
        "value": round(3 * gf / (ms * 1e-3) / 1e12, 1), "unit": "TFLOP/s", "ms_per_step": round(ms, 4),
        "flops_per_step": 3 * gf,
        "kernels_ms": {k: round(v, 4) for k, v in kms.items()},
        "gemm_TFLOPs": {k: round(gf / (kms[k] * 1e-3) / 1e12, 1) for k in ("fwd_gemm", "dX_gemm", "dW_gemm")},
        "roofline": {"bound": "tensor", "kernel": "gemm_tc_kernel / gemm_tc_pair_kernel (fwd, dX, dW aggregated)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4),
                     "peak_kind": "measured cuBLAS TF32 8192^3, best of 10 (burst)" if tf32 else "burst",
                     "tf32_spec_frac": round(achieved / TF32_PEAK_TFLOPS, 4) if tf32 else None,
                     "traffic": None if tf32 else traffic_of("gemm_bf16_fwd_c3", True),
                     "traffic_algorithmic_bytes": esz * (M * D + D * D + M * D)},
        "gpu_launches_per_step": 4,
        "seed_fused_into_forward": True,
        "cublas_TFLOPs_same_shapes": cublas,
        "l2": f"working set ~{808 if tf32 else 544} MB per step > 126 MB L2",
    }


def count_launches(fn):
    """Kernels launched by one call of fn (torch.profiler / CUPTI), or None."""
    import torch

    try:
        from torch.profiler import ProfilerActivity, profile

        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        return sum(1 for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA)
    except Exception:  # profiler unavailable: report nothing rather than a guess
        return None


def mlp_bench(args, world, rank, dist, peaks, name, sizes, acts, batch, loss, graph, lr=1e-4):
    """Dense-chain training step (fwd + loss + pullback + [allreduce] + SGD)."""
    import torch

    from paper_1811_01457_b200.dense import Chain, Dense
    from paper_1811_01457_b200.train import Trainer

    rng = np.random.default_rng(11)
    chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(len(acts))]).init_params(rng)
    tr = Trainer(chain, batch, loss=loss, lr=lr, precision="bf16", dp=world > 1, graph=graph)
    lb = tr.local_batch
    g = torch.Generator(device="cuda").manual_seed(100 + rank)
    X = torch.rand((lb, sizes[0]), generator=g, device="cuda")
    if loss == "softmax_xent":
        Y = torch.zeros((lb, sizes[-1]), device="cuda")
        Y[torch.arange(lb, device="cuda"), torch.randint(0, sizes[-1], (lb,), generator=g, device="cuda")] = 1
    else:
        Y = torch.rand((lb, sizes[-1]), generator=g, device="cuda") * 2 - 1
    stream = torch.cuda.current_stream()
    steps = args.mlp_steps if name != "c1" else max(args.mlp_steps, 50)
    # SM clocks during the timed steps (the bench's short windows run at boost
    # clocks; sustained, c4 / c5 sit at the power limit: DESIGN §4,
    # profiles/r02c_power_probe.log -- NVML's power reading averages over ~1 s,
    # too long for these windows, so it is not reported here)
    with ClockSampler(torch.cuda.current_device()) as clk:
        ms, _ = _timed(lambda ev: tr.step(X, Y), steps, max(3, args.warmup), dist, stream)
    loss_v = float(tr.engine.loss.item())
    replicas_ok = tr.replicas_identical() if world > 1 else True
    small = tr.engine.small is not None  # the whole step in one cooperative launch
    # the whole step as issued eagerly: minibatch load (sg_cast_2d), forward,
    # loss, pullback, [all-reduce], SGD -- the graph replays exactly these
    launches = count_launches(lambda: tr.step(X, Y) if small else (tr.engine.load_batch(X, Y), tr._device_step()))
    no_graph_ms = layer_ms = None
    if small:  # beside it: the layer-by-layer tensor-core path in a CUDA graph
        tr2 = Trainer(chain, batch, loss=loss, lr=lr, precision="bf16", dp=world > 1, graph=True, small=False)
        layer_ms, _ = _timed(lambda ev: tr2.step(X, Y), steps, max(3, args.warmup), dist, stream)
        tr2.close()
    elif tr.use_graph:  # the same step without the graph (launch overhead exposed)
        tr2 = Trainer(chain, batch, loss=loss, lr=lr, precision="bf16", dp=world > 1, graph=False)
        no_graph_ms, _ = _timed(lambda ev: tr2.step(X, Y), steps, max(3, args.warmup), dist, stream)
        tr2.close()
    chain_ms = None
    if name == "c5" and world == 1:  # the persistent-GEMM-chain variant beside it (opt-in, bit-identical)
        os.environ["SGB200_CHAIN"] = "1"
        try:
            trc = Trainer(chain, batch, loss=loss, lr=lr, precision="bf16", graph=True)
            chain_ms, _ = _timed(lambda ev: trc.step(X, Y), steps, max(3, args.warmup), dist, stream)
            trc.close()
        finally:
            del os.environ["SGB200_CHAIN"]
    flops = tr.engine.flops_per_step() * world
    # bytes the step touches: parameters (fp32 + bf16 shadow + gradients) and
    # the per-layer activations / cotangents (bf16) of this rank's batch
    n_par = sum(sizes[i] * sizes[i + 1] + sizes[i + 1] for i in range(len(acts)))
    ws_mb = (n_par * 10 + lb * sum(sizes) * 2 * 3 + lb * (sizes[0] + sizes[-1]) * 4) / 1e6
    tr.close()
    tflops = flops / (ms * 1e-3) / 1e12
    if small:  # latency-bound: the roofline is the launch, not a pipe
        roof = {"bound": "latency", "kernel": "k_mlp_small_step (one launch per step)",
                "achieved_us_per_step": round(ms * 1e3, 2), "TFLOPs": round(tflops, 2)}
    else:
        roof = {"bound": "tensor", "kernel": "whole step (GEMM-dominated)", "achieved": round(tflops / world, 1),
                "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                "frac": round(tflops / world / peaks["bf16_tflops_sustained"], 4),
                "peak_kind": "sustained", "traffic": None}
    rec = {
        "workload": f"{name} MLP {'-'.join(map(str, sizes))} ({'/'.join(acts)}, {loss}) train step, "
                    f"global batch {batch}, "
                    + ("fp32, whole step in one cooperative launch (sg_mlp_small_step)" if small else "bf16 tcgen05")
                    + (f", DP x{world} NCCL" if world > 1 else ""),
        "value": round(batch / (ms * 1e-3), 1), "unit": "samples/s", "ms_per_step": round(ms, 4),
        "flops_per_step": flops, "TFLOPs": round(tflops, 1),
        "roofline": roof,
        "compute_precision": tr.compute_precision, "clocks": clk.summary(),
        "l2": (f"working set ~{ws_mb:.0f} MB per step > 126 MB L2 (no flush needed)" if ws_mb > 126 else
               f"working set ~{ws_mb:.1f} MB per step stays L2-resident between steps (no flush: the step is "
               "latency-bound, one launch; a flush would dominate it)"),
        "cuda_graph": bool(tr.use_graph) and not small, "loss_last": loss_v, "n_gpus": world,
        "gpu_launches_per_step": launches,
        "ms_per_step_without_graph": None if no_graph_ms is None else round(no_graph_ms, 4),
        "layer_path_ms_per_step": None if layer_ms is None else round(layer_ms, 4),
        "gemm_chain_ms_per_step": None if chain_ms is None else round(chain_ms, 4),
        "replicas_identical": replicas_ok,
        "scaling": "strong (global batch fixed)",
    }
    return rec


def summary_of(rec):
    """Compact per-workload digest (value, ms/step, roofline fraction) of the
    headline and every secondary workload, printed as the line's LAST key so a
    tail-truncated log still shows every number."""
    def one(r, name):
        roof = r.get("roofline") or {}
        return {"w": name, "v": r.get("value"), "u": r.get("unit"), "ms": r.get("ms_per_step"),
                "frac": roof.get("frac"), "launches": r.get("gpu_launches_per_step")}

    out = [one(rec, "c2 fp32 (headline)")]
    if rec.get("e2e"):
        out[0]["e2e"] = rec["e2e"].get("value")
    for r in rec.get("secondary", []):
        name = r.get("workload", "?")
        if "error" in r:
            out.append({"w": name[:40], "error": r["error"][:120]})
            continue
        e = one(r, r.get("key", name.split(" ")[0]))
        if "gemm_TFLOPs" in r:
            e["gemm"] = r["gemm_TFLOPs"]
        out.append(e)
    return out


def secondary_benches(args, world, rank, dist, out=None):
    peaks = load_peaks()
    out = [] if out is None else out
    todo = [w.strip() for w in args.secondary.split(",") if w.strip()]
    for w in todo:
        try:
            if w == "c3" and world == 1:
                out.append(dense_c3_bench(args, dist, peaks))
            elif w in ("c2scalar", "c2col", "c2f64"):
                out.append(broadcast_variant_bench(args, dist, peaks, {"c2scalar": "scalar", "c2col": "col",
                                                                      "c2f64": "f64"}[w]))
            elif w == "c3tf32" and world == 1:
                out.append(dense_c3_bench(args, dist, peaks, precision="tf32"))
            elif w == "c4":
                out.append(mlp_bench(args, world, rank, dist, peaks, "c4", (4096,) * 5,
                                     ("tanh",) * 3 + ("identity",), 65536, "mse", graph=True))
            elif w == "c5":
                out.append(mlp_bench(args, world, rank, dist, peaks, "c5", (1024,) * 17,
                                     ("tanh",) * 15 + ("identity",), 32768, "mse", graph=True))
            elif w == "c1":
                out.append(mlp_bench(args, world, rank, dist, peaks, "c1", (784, 32, 10),
                                     ("sigmoid", "identity"), 128, "softmax_xent", graph=True, lr=0.05))
        except Exception as e:  # report, do not lose the headline line
            out.append({"workload": w, "error": f"{type(e).__name__}: {e}"[:500]})
    return out


def cpu_baseline_mlp(name, sizes, acts, batch, loss, mode, rows=None):
    """Oracle port of the reference's Dense step (fwd + loss + pullback + SGD) on the host.

    mode "exact": the reference's own matmul order (ascending-k, C restatement,
    1 core); mode "blas": numpy/OpenBLAS fp64 restatement (all cores), on a
    row slice of `rows` samples when the full batch would take too long.
    """
    import math as _m

    from oracle import dense as OD

    rng = np.random.default_rng(0)
    n = rows or batch
    params = []
    for i in range(len(acts)):
        r = _m.sqrt(6.0 / (sizes[i] + sizes[i + 1]))
        params.append((rng.uniform(-r, r, (sizes[i + 1], sizes[i])), np.zeros(sizes[i + 1])))
    X = rng.uniform(0, 1, (n, sizes[0]))
    if loss == "softmax_xent":
        Y = np.zeros((n, sizes[-1]))
        Y[np.arange(n), rng.integers(0, sizes[-1], n)] = 1.0
    else:
        Y = rng.uniform(-1, 1, (n, sizes[-1]))
    OD.mlp_step(params, X, Y, acts, loss, mode=mode)  # warm
    t0 = time.perf_counter()
    reps = 0
    while True:
        OD.mlp_step(params, X, Y, acts, loss, mode=mode)
        reps += 1
        if time.perf_counter() - t0 > 2.0:
            break
    sec = (time.perf_counter() - t0) / reps
    return {"workload": name, "value": round(n / sec, 2), "unit": "samples/s",
            "kind": "port", "mode": mode,
            "cores": 1 if mode == "exact" else len(os.sched_getaffinity(0)),
            "sample": f"{n} rows of the {batch}-row batch" if rows else f"full batch {batch}",
            "s_per_step_sample": round(sec, 4)}


def import_reference():
    """The unmodified reference (pure Python + numpy) installed into
    baseline/_ref by `pip install --target baseline/_ref` (git-ignored; it
    travels to the GPU box with the snapshot), or None."""
    p = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(p, "ssagrad")):
        return None
    if p not in sys.path:
        sys.path.insert(0, p)
    try:
        import ssagrad

        return ssagrad
    except Exception:  # pragma: no cover - broken install: report the port instead
        return None


def reference_broadcast(rows=32):
    """The reference's own c2 path on a bounded sample: fused_map_with_partials
    (the per-element dual interpreter that the augmented forward's fused_pack
    runs, forward_ad.py:194-223 / interp.py:334-352; its row 0 is the primal)
    + fused_map_pullback (forward_ad.py:226-235), single-threaded."""
    from ssagrad import DenseTensor, parse_ir
    from ssagrad.forward_ad import fused_map_pullback, fused_map_with_partials
    from ssagrad.ir import tensor_type

    m = parse_ir(AFFSIG)
    rng = np.random.default_rng(0)
    C = C_COLS
    x = rng.uniform(-2, 2, (rows, C)).astype(np.float32).astype(np.float64)
    a = rng.uniform(-2, 2, C).astype(np.float32).astype(np.float64)
    b = rng.uniform(-2, 2, C).astype(np.float32).astype(np.float64)
    yb = rng.uniform(-1, 1, (rows, C)).astype(np.float32).astype(np.float64)
    n = rows * C
    t0 = time.perf_counter()
    primal, parts = fused_map_with_partials(m, "affsig", [DenseTensor(a), DenseTensor(x), DenseTensor(b)])
    t1 = time.perf_counter()
    fused_map_pullback(parts, [tensor_type(C), tensor_type(rows, C), tensor_type(C)], DenseTensor(yb))
    t2 = time.perf_counter()
    sec = t2 - t0
    return {
        "value": round(n * BYTES_PER_ELEM / sec / 1e9, 6),
        "unit": "GB/s",
        "cores": 1,
        "kind": "reference",
        "sample": f"{rows}x{C} = {n} elements through the unmodified reference (baseline/_ref): "
                  "fused_map_with_partials + fused_map_pullback, 20 B/elem algorithmic",
        "us_per_elem_pack": round((t1 - t0) / n * 1e6, 3),
        "us_per_elem_pullback": round((t2 - t1) / n * 1e6, 4),
        "extrapolated_s_at_2^28": round(sec / n * (1 << 28), 1),
        "host_cores_available": len(os.sched_getaffinity(0)),
    }


def _ref_c2_worker_init():
    import_reference()


def _ref_c2_worker(job):
    """One worker's sample (its own rows) through the unmodified reference."""
    seed, rows = job
    from ssagrad import DenseTensor, parse_ir
    from ssagrad.forward_ad import fused_map_pullback, fused_map_with_partials
    from ssagrad.ir import tensor_type

    m = parse_ir(AFFSIG)
    rng = np.random.default_rng(seed)
    C = C_COLS
    x = rng.uniform(-2, 2, (rows, C)).astype(np.float32).astype(np.float64)
    a = rng.uniform(-2, 2, C).astype(np.float32).astype(np.float64)
    b = rng.uniform(-2, 2, C).astype(np.float32).astype(np.float64)
    yb = rng.uniform(-1, 1, (rows, C)).astype(np.float32).astype(np.float64)
    _, parts = fused_map_with_partials(m, "affsig", [DenseTensor(a), DenseTensor(x), DenseTensor(b)])
    fused_map_pullback(parts, [tensor_type(C), tensor_type(rows, C), tensor_type(C)], DenseTensor(yb))
    return rows * C


def reference_broadcast_parallel(rows=32):
    """The reference's c2 path on ALL host cores: the reference itself is
    single-threaded Python, and elements are independent, so one process per
    core runs it on its own `rows` x 4096 sample (pool warmed up first: the
    imports are not timed); throughput = all elements / wall time."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    ctx = mp.get_context("spawn")  # no fork of a process holding a CUDA context
    with ctx.Pool(cores, initializer=_ref_c2_worker_init) as pool:
        pool.map(_ref_c2_worker, [(i, 1) for i in range(cores)])  # warm-up: imports, first calls
        t0 = time.perf_counter()
        n = sum(pool.map(_ref_c2_worker, [(100 + i, rows) for i in range(cores)]))
        sec = time.perf_counter() - t0
    return {"value": round(n * BYTES_PER_ELEM / sec / 1e9, 6), "unit": "GB/s", "cores": cores,
            "kind": "reference",
            "sample": f"{cores} processes x {rows}x{C_COLS} elements (disjoint samples) through the unmodified "
                      "reference (baseline/_ref): fused_map_with_partials + fused_map_pullback, 20 B/elem "
                      "algorithmic; the reference is single-threaded, elements are independent",
            "wall_s": round(sec, 3)}


def _reference_chain_module(sizes, acts, n, loss):
    """A Dense chain's loss IR built with the reference's own emitter, exactly
    as nn_train's trunk builds layers (nn_train.py:189-196):
    wt = transpose(W); z = matmul(h, wt); zb = add(z, b); h = act(zb), then the
    c1 softmax-CE IR, MSE, or 'dot' (sum(h * Y): pulls the seed
    Y back through a single layer, the c3 fwd + pullback)."""
    from ssagrad import Module
    from ssagrad.ir import F64, tensor_type
    from ssagrad.structure import SEmitter, flatten

    module = Module()
    em = SEmitter("chain", (F64,), module)
    pairs = [(em.param(f"W{k}", tensor_type(sizes[k + 1], sizes[k])), em.param(f"b{k}", tensor_type(sizes[k + 1])))
             for k in range(len(sizes) - 1)]
    x = em.param("X", tensor_type(n, sizes[0]))
    y = em.param("Y", tensor_type(n, sizes[-1]))
    h = x
    for (w, b), act in zip(pairs, acts):
        wt = em.emit("transpose", (w,), None, "wt")
        z = em.emit("matmul", (h, wt), None, "z")
        zb = em.emit("add", (z, b), None, "zb")
        h = zb if act == "identity" else em.emit(act, (zb,), None, "h")
    if loss == "softmax_xent":
        e = em.emit("exp", (h,), None, "e")
        ssum = em.emit("reduce_sum", (e,), {"axis": 1}, "s")
        s2 = em.emit("reshape", (ssum,), {"shape": (n, 1)}, "s2")
        p = em.emit("div", (e, s2), None, "p")
        lp = em.emit("log", (p,), None, "lp")
        t = em.emit("mul", (y, lp), None, "t")
        tot = em.emit("reduce_sum", (t,), {"axis": "all"}, "tot")
        sc = em.const_f64(-1.0 / n, "sc")
    elif loss == "mse":
        d = em.emit("sub", (h, y), None, "d")
        sq = em.emit("mul", (d, d), None, "sq")
        tot = em.emit("reduce_sum", (sq,), {"axis": "all"}, "tot")
        sc = em.const_f64(1.0 / n, "sc")
    else:
        t = em.emit("mul", (h, y), None, "t")
        tot = em.emit("reduce_sum", (t,), {"axis": "all"}, "tot")
        sc = em.const_f64(1.0, "sc")
    loss_v = em.emit("mul", (tot, sc), None, "loss")
    module.add(flatten(em.finish((loss_v,))))
    return module


def reference_mlp(name, sizes, acts, batch, loss, rows=None, lr=0.05, unit="samples/s"):
    """The reference's own training step: grad (augment + Machine.call of the
    aug and pb functions, reverse_ad.py:619-663) of the chain's loss IR, then
    SGD p - lr * g (nn_train.py:365-372), on the full batch or on a row slice
    (every matmul is linear in the rows, so samples/s extrapolate)."""
    from ssagrad import DenseTensor, grad

    n = rows or batch
    rng = np.random.default_rng(0)
    params = []
    for i in range(len(acts)):
        r = np.sqrt(6.0 / (sizes[i] + sizes[i + 1]))
        params.append((rng.uniform(-r, r, (sizes[i + 1], sizes[i])), np.zeros(sizes[i + 1])))
    X = rng.uniform(0, 1, (n, sizes[0]))
    if loss == "softmax_xent":
        Y = np.zeros((n, sizes[-1]))
        Y[np.arange(n), rng.integers(0, sizes[-1], n)] = 1.0
    else:
        Y = rng.uniform(-1, 1, (n, sizes[-1]))
    module = _reference_chain_module(sizes, acts, n, loss)
    args = []
    for W, b in params:
        args += [DenseTensor(W), DenseTensor(b)]
    args += [DenseTensor(X), DenseTensor(Y)]
    fn = module.get("chain")
    grad(module, "chain", tuple(args))  # builds (and caches) the aug / pb IR once
    t0 = time.perf_counter()
    reps = 0
    while True:
        g = grad(module, "chain", tuple(args))
        [W - lr * g[fn.params[2 * k][0]].data for k, (W, _) in enumerate(params)]
        [b - lr * g[fn.params[2 * k + 1][0]].data for k, (_, b) in enumerate(params)]
        reps += 1
        if time.perf_counter() - t0 > 1.0 or rows:
            break
    sec = (time.perf_counter() - t0) / reps
    rec = {"workload": name, "value": round(n / sec, 4), "unit": "samples/s", "kind": "reference", "cores": 1,
           "sample": f"{n} rows of the {batch}-row batch (extrapolated: cost is linear in rows)" if rows
           else f"full batch {batch}",
           "s_per_step_sample": round(sec, 4)}
    if unit == "TFLOP/s":  # c3: one layer's fwd + dX + dW
        rec["value"] = round(6.0 * n * sizes[0] * sizes[1] / sec / 1e12, 9)
        rec["unit"] = "TFLOP/s"
    return rec


def reference_arm(args, world, rank):
    """`bench.py --impl reference`: the reference's own CPU implementation of
    the path on this box's host cores -- the unmodified reference from
    baseline/_ref when installed (kind "reference"), else the oracle's port
    of its algorithm (kind "port") -- on the same workloads and metrics."""
    if rank != 0:
        return None
    t0 = time.perf_counter()
    ref = import_reference()
    vals = []
    for _ in range(max(1, min(args.steps, 3))):
        vals.append(reference_broadcast_parallel(rows=args.ref_rows) if ref
                    else cpu_baseline_broadcast(rows=args.ref_rows))
    v = statistics.median(r["value"] for r in vals)
    cb = dict(vals[-1])
    cb["value"] = v
    secondary = []
    if ref:
        one = reference_broadcast(rows=args.ref_rows)
        secondary.append({"workload": "c2 (reference, one core)", **one})
        secondary += [
            reference_mlp("c1 MLP 784-32-10 train step (reference grad + SGD)", (784, 32, 10), ("sigmoid", "identity"),
                          128, "softmax_xent"),
            reference_mlp("c3 Dense 4096->4096 sigmoid fwd+pullback (reference, row slice)", (4096, 4096),
                          ("sigmoid",), 8192, "dot", rows=1, unit="TFLOP/s"),
            reference_mlp("c4 MLP 4x4096 train step (reference, row slice)", (4096,) * 5,
                          ("tanh",) * 3 + ("identity",), 65536, "mse", rows=1, lr=1e-4),
            reference_mlp("c5 MLP 16x1024 train step (reference, row slice)", (1024,) * 17,
                          ("tanh",) * 15 + ("identity",), 32768, "mse", rows=4, lr=1e-4),
        ]
    secondary += [
        cpu_baseline_mlp("c1 MLP 784-32-10 train step (port: reference matmul order, C)", (784, 32, 10),
                         ("sigmoid", "identity"), 128, "softmax_xent", "exact"),
        cpu_baseline_mlp("c4 MLP 4x4096 train step (port: numpy-BLAS fp64, row slice)", (4096,) * 5,
                         ("tanh",) * 3 + ("identity",), 65536, "mse", "blas", rows=256),
    ]
    if ref:
        port = cpu_baseline_broadcast(rows=args.ref_rows)
        secondary.append({"workload": "c2 (port: the oracle's per-element interpreter)", **port})
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": c2_config(args.rows, C_COLS, world),
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "secondary": secondary,
        "wall_s": round(time.perf_counter() - t0, 1),
        "summary": [{"w": r["workload"][:48], "v": r.get("value"), "u": r.get("unit"), "kind": r.get("kind")}
                    for r in secondary],
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--rows", type=int, default=R_ROWS)
    ap.add_argument("--ref-rows", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--secondary", default="c2scalar,c2col,c2f64,c1,c3,c3tf32,c4,c5",
                    help="comma list of extra workloads measured in the same run (c2scalar,c2col,c2f64,c1,c3,c3tf32,c4,c5)")
    ap.add_argument("--dense-steps", type=int, default=20)
    ap.add_argument("--mlp-steps", type=int, default=10)
    args = ap.parse_args()
    world, rank, local = dist_env()

    if args.impl == "reference":
        rec = reference_arm(args, world, rank)
        if rec is not None:
            print(json.dumps(rec), flush=True)
        return

    dist = init_dist(world, local)
    rec = broadcast_bench(args, world, rank, local, dist)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ref = import_reference()
        rec["cpu_baseline"] = reference_broadcast_parallel(rows=args.ref_rows) if ref else \
            cpu_baseline_broadcast(rows=args.ref_rows)
        rec["cpu_baseline"]["secondary"] = [
            reference_mlp("c1", (784, 32, 10), ("sigmoid", "identity"), 128, "softmax_xent") if ref else
            cpu_baseline_mlp("c1", (784, 32, 10), ("sigmoid", "identity"), 128, "softmax_xent", "exact")]
    if args.secondary:
        # the headline is measured: a secondary workload that hangs (e.g. a
        # collective at a world size this run could not test) must not take
        # the line with it -- after the limit rank 0 prints what it has
        partial = []
        rec["secondary"] = partial
        limit = float(os.environ.get("SGB200_BENCH_SECONDARY_LIMIT", "900"))

        def give_up():
            if rank == 0:
                rec["secondary_timeout_s"] = limit
                rec["summary"] = summary_of(rec)
                print(json.dumps(rec), flush=True)
            os._exit(0)

        dog = threading.Timer(limit, give_up)
        dog.daemon = True
        dog.start()
        secondary_benches(args, world, rank, dist, out=partial)
        dog.cancel()
    if rank == 0:
        rec["summary"] = summary_of(rec)  # last key: survives a tail-truncated log
        print(json.dumps(rec), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
