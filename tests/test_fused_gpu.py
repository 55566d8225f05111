"""GPU parity of the fused broadcast kernels against the reference.

Golden vectors come from the unmodified reference (tests/golden); larger
cases are checked against the pinned oracle.  Tolerances (rel metric of
the reference suite, pkg/tests/conftest.py:137-144):
  f64 device path: 1e-13 (only libm ulps differ; + - * / round like Python),
  f32 device path: 1e-6 (BASELINE.json north star, fp32 elementwise).
"""

import math
import re

import numpy as np
import pytest

from conftest import decode, max_rel
from oracle import scalar as OS

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1811_01457_b200 import fused as F  # noqa: E402
from paper_1811_01457_b200.ir import F64, tensor_type  # noqa: E402

TOL = {torch.float64: 1e-13, torch.float32: 1e-6}


def dev_args(case, dtype):
    out = []
    for a in case["args"]:
        v = decode(a)
        out.append(torch.tensor(v, dtype=dtype, device="cuda") if isinstance(v, np.ndarray) else v)
    return out


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_partials_match_reference(golden_fused, fused_module, dtype):
    for case in golden_fused["cases"]:
        args = dev_args(case, dtype)
        if not any(isinstance(a, torch.Tensor) for a in args):
            args = [float(a) for a in args]
        primal, parts = F.fused_map_with_partials(fused_module, case["fn"], args, dtype=dtype)
        assert max_rel(primal, decode(case["primal"])) <= TOL[dtype], case["fn"]
        for p, g in zip(parts, case["partials"]):
            assert max_rel(p, decode(g)) <= TOL[dtype], case["fn"]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_forward_matches_reference(golden_fused, fused_module, dtype):
    for case in golden_fused["cases"]:
        args = dev_args(case, dtype)
        y = F.fused_map(fused_module, case["fn"], args, dtype=dtype)
        assert max_rel(y, decode(case["primal"])) <= TOL[dtype], case["fn"]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_fused_grad_matches_reference_pullback(golden_fused, fused_module, dtype):
    # K2 computes reduce_like(ybar * partial_i) directly from the inputs
    for case in golden_fused["cases"]:
        if case["pullback"] is None:
            continue
        args = dev_args(case, dtype)
        ybar = torch.tensor(decode(case["ybar"]), dtype=dtype, device="cuda")
        y, cots = F.fused_map_grad(fused_module, case["fn"], args, ybar, want_primal=True)
        assert max_rel(y, decode(case["primal"])) <= TOL[dtype], case["fn"]
        for c, want, a in zip(cots, case["pullback"], args):
            w = decode(want)
            if isinstance(a, float):
                assert max_rel(float(c.item()), w) <= TOL[dtype], case["fn"]
            else:
                assert tuple(c.shape) == tuple(np.shape(w)), case["fn"]
                assert max_rel(c, w) <= TOL[dtype], case["fn"]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_pullback_api_matches_reference(golden_fused, fused_module, dtype):
    for case in golden_fused["cases"]:
        if case["pullback"] is None:
            continue
        args = dev_args(case, dtype)
        _, parts = F.fused_map_with_partials(fused_module, case["fn"], args, dtype=dtype)
        types = [tensor_type(*a.shape) if isinstance(a, torch.Tensor) else F64 for a in args]
        ybar = torch.tensor(decode(case["ybar"]), dtype=dtype, device="cuda")
        got = F.fused_map_pullback(parts, types, ybar)
        for g, want in zip(got, case["pullback"]):
            assert max_rel(g, decode(want)) <= TOL[dtype], case["fn"]


def test_domain_errors_raise_reference_eval_error(golden_fused, fused_module):
    for err in golden_fused["errors"]:
        args = dev_args(err, torch.float64)
        with pytest.raises(F.EvalError) as ei:
            F.fused_map_with_partials(fused_module, err["fn"], args)
        e = ei.value
        assert (e.function, e.block, e.index) == (err["function"], err["block"], err["index"])
        assert err["message"].startswith(e.message)
    # the error word is cleared: a clean call afterwards succeeds
    F.fused_map(fused_module, "logp", [torch.ones(4, dtype=torch.float64, device="cuda")])


def test_step_limit_on_runaway_loop():
    from paper_1811_01457_b200.irtext import parse_ir

    m = parse_ir("""
func @spin(%x: f64) -> f64 {
^entry:
  jmp ^loop(%x)
^loop(%v: f64):
  %t = const bool true
  br %t, ^loop(%v), ^out(%v)
^out(%r: f64):
  ret %r
}
""")
    F.set_step_limit(10_000)
    try:
        with pytest.raises(F.EvalError) as ei:
            F.fused_map(m, "spin", [torch.ones(8, device="cuda")])
        assert ei.value.message == "step limit exhausted"
    finally:
        F.set_step_limit(F.DEFAULT_STEP_LIMIT)


@pytest.mark.parametrize("R,C", [(1024, 1024), (333, 77), (4096, 12)])
def test_affsig_rowwise_broadcast_vs_oracle(fused_module, R, C):
    # c2 pattern sigma(a*x+b), a,b of shape (C,), at sizes the oracle handles
    rng = np.random.default_rng(R + C)
    x = rng.uniform(-2, 2, (R, C)).astype(np.float32)
    a = rng.uniform(-2, 2, C).astype(np.float32)
    b = rng.uniform(-2, 2, C).astype(np.float32)
    yb = rng.uniform(-1, 1, (R, C)).astype(np.float32)
    args = [torch.from_numpy(v).cuda() for v in (a, x, b)]
    y, (da, dx, db) = F.fused_map_grad(fused_module, "affsig", args, torch.from_numpy(yb).cuda(),
                                       want_primal=True)
    p, parts = OS.vec_eval(fused_module, "affsig", [a.astype(np.float64), x.astype(np.float64),
                                                   b.astype(np.float64)])
    ybd = yb.astype(np.float64)
    assert max_rel(y, p) <= 1e-6
    assert max_rel(dx, ybd * parts[1]) <= 1e-6
    # broadcast-axis sums: each of the R terms is within 1e-6 (fp32 elementwise)
    # and they are accumulated in fp64, so |err| <= 1e-6 * sum|terms|
    for got, part in ((da, parts[0]), (db, parts[2])):
        terms = ybd * part
        err = np.abs(got.double().cpu().numpy() - OS.reduce_to(terms, (C,)))
        assert (err <= 1e-6 * np.maximum(1.0, np.abs(terms).sum(axis=0))).all()
    y2 = F.fused_map(fused_module, "affsig", args)
    assert torch.equal(y, y2)  # primal of K1 == primal of K2 (no FMA contraction)


def test_column_and_scalar_reductions(fused_module):
    # (R,1) operand -> row sums via warp shuffles; scalar -> block tree
    rng = np.random.default_rng(3)
    R, C = 257, 1000
    x = rng.uniform(-2, 2, (R, C))
    w = rng.uniform(-2, 2, (R, 1))
    s = 0.3
    yb = rng.uniform(-1, 1, (R, C))
    args = [torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), s]
    _, (dx, dw, ds) = F.fused_map_grad(fused_module, "mixed", args, torch.from_numpy(yb).cuda())
    p, parts = OS.vec_eval(fused_module, "mixed", [x, w, s])
    assert max_rel(dx, yb * parts[0]) <= 1e-13
    assert max_rel(dw, OS.reduce_to(yb * parts[1], (R, 1))) <= 1e-12
    assert abs(float(ds.item()) - OS.fused_map_pullback([parts[2]], [None], yb)[0]) <= 1e-10 * R * C


def test_deterministic_gradients(fused_module):
    torch.manual_seed(0)
    x = torch.rand(2048, 512, device="cuda") * 4 - 2
    a = torch.rand(512, device="cuda")
    b = torch.rand(512, device="cuda")
    yb = torch.rand(2048, 512, device="cuda")
    _, g1 = F.fused_map_grad(fused_module, "affsig", [a, x, b], yb)
    _, g2 = F.fused_map_grad(fused_module, "affsig", [a, x, b], yb)
    for u, v in zip(g1, g2):
        assert torch.equal(u, v)


def test_reference_style_inputs(fused_module):
    # reference DenseTensor-like objects and numpy arrays are accepted
    class DT:  # duck-typed reference DenseTensor (tensor.py:29-47)
        def __init__(self, a):
            self.data = np.asarray(a, dtype=np.float64)

    primal, parts = F.fused_map_with_partials(fused_module, "two", (DT([0.2, -0.9, 1.4, 0.05]), 0.7))
    want = [math.tanh(v + 0.7) for v in (0.2, -0.9, 1.4, 0.05)]
    assert max_rel(primal, np.array(want)) <= 1e-15
    assert primal.dtype == torch.float64
    p, q = F.fused_map_with_partials(fused_module, "two", (0.5, 0.25))
    assert isinstance(p, float) and abs(p - math.tanh(0.75)) < 1e-15
    assert len(q) == 2 and all(isinstance(v, float) for v in q)


def test_fuzz_corpus_matches_reference():
    """60 random scalar programs (reference progen, branches/loops/select/
    pow_int/itof) fused over 16-element vectors: primal and every partial
    within 1e-11 of the reference (f64; only libm ulps differ, amplified
    by up to a dozen chained transcendentals)."""
    import json
    import os

    from conftest import GOLDEN
    from paper_1811_01457_b200.irtext import parse_ir

    with open(os.path.join(GOLDEN, "fuzz.json")) as f:
        d = json.load(f)
    m = parse_ir(d["ir"])
    worst = 0.0
    for case in d["cases"]:
        args = [torch.tensor(decode(a), dtype=torch.float64, device="cuda") for a in case["args"]]
        primal, parts = F.fused_map_with_partials(m, case["fn"], args)
        worst = max(worst, max_rel(primal, decode(case["primal"])))
        for p, g in zip(parts, case["partials"]):
            worst = max(worst, max_rel(p, decode(g)))
        # K2 agrees with the pack contraction
        yb = torch.ones_like(args[0])
        _, cots = F.fused_map_grad(m, case["fn"], args, yb)
        for c, g in zip(cots, case["partials"]):
            worst = max(worst, max_rel(c, decode(g)))
    assert worst <= 1e-11, worst


def test_c2_full_size_against_fp64(fused_module):
    """BASELINE c2 at its full size (2^28 fp32 elements, a, b of shape (4096,)):
    the device path vs an fp64 evaluation of the same op (torch, test-side
    only): y and xbar elementwise <= 1e-6 (reference rel metric), abar/bbar (65536-term column
    sums) within 1e-6 * sum|terms|; the 8-chunk row split the e2e bench uses
    gives the same xbar bit for bit."""
    R, C = 1 << 16, 1 << 12
    g = torch.Generator(device="cuda").manual_seed(2)
    x = torch.rand((R, C), generator=g, device="cuda") * 4 - 2
    yb = torch.rand((R, C), generator=g, device="cuda") * 2 - 1
    a = torch.rand(C, generator=g, device="cuda") * 4 - 2
    b = torch.rand(C, generator=g, device="cuda") * 4 - 2
    y, (da, dx, db) = F.fused_map_grad(fused_module, "affsig", [a, x, b], yb, want_primal=True)
    # fp64 restatement, row block by row block (bounded memory)
    abs_a = torch.zeros(C, dtype=torch.float64, device="cuda")
    abs_b = torch.zeros_like(abs_a)
    ref_a = torch.zeros_like(abs_a)
    ref_b = torch.zeros_like(abs_a)
    worst_y = worst_x = 0.0
    for r0 in range(0, R, 8192):
        xs, ys = x[r0:r0 + 8192].double(), yb[r0:r0 + 8192].double()
        s = torch.sigmoid(a.double() * xs + b.double())
        ds = s * (1 - s)
        # the reference suite's metric |u - v| / max(1, |u|, |v|) (conftest.py:137-144)
        gy, want_x = y[r0:r0 + 8192].double(), ys * ds * a.double()
        gx = dx[r0:r0 + 8192].double()
        worst_y = max(worst_y, float(((gy - s).abs() / torch.maximum(gy.abs(), s.abs()).clamp_min(1.0)).max()))
        worst_x = max(worst_x, float(((gx - want_x).abs()
                                      / torch.maximum(gx.abs(), want_x.abs()).clamp_min(1.0)).max()))
        ta, tb = ys * ds * xs, ys * ds
        ref_a += ta.sum(0)
        ref_b += tb.sum(0)
        abs_a += ta.abs().sum(0)
        abs_b += tb.abs().sum(0)
    assert worst_y <= 1e-6 and worst_x <= 1e-6, (worst_y, worst_x)
    assert bool(((da.double() - ref_a).abs() <= 1e-6 * abs_a.clamp_min(1.0)).all())
    assert bool(((db.double() - ref_b).abs() <= 1e-6 * abs_b.clamp_min(1.0)).all())
    # the chunked public-API path of the e2e bench
    dx2 = torch.empty_like(dx)
    for r0 in range(0, R, R // 8):
        _, (_, part, _) = F.fused_map_grad(fused_module, "affsig", [a, x[r0:r0 + R // 8], b],
                                           yb[r0:r0 + R // 8])
        dx2[r0:r0 + R // 8] = part
    assert torch.equal(dx, dx2)


def test_c2_f64_at_scale_matches_fp64_arithmetic(fused_module):
    """c2's sub-function in f64 -- the reference's own dtype -- at 2^26
    elements: the device path does + - * / in IEEE f64 exactly as the
    reference's Python floats (--fmad=false), so against the same arithmetic
    in torch f64 (test-side) y and xbar agree to libm ulps (1e-14, reference
    rel metric) and the 16384-term column sums to 1e-12 * sum|terms|
    (summation order only)."""
    R, C = 1 << 14, 1 << 12
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand((R, C), generator=g, device="cuda", dtype=torch.float64) * 4 - 2
    yb = torch.rand((R, C), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
    a = torch.rand(C, generator=g, device="cuda", dtype=torch.float64) * 4 - 2
    b = torch.rand(C, generator=g, device="cuda", dtype=torch.float64) * 4 - 2
    y, (da, dx, db) = F.fused_map_grad(fused_module, "affsig", [a, x, b], yb, want_primal=True)
    z = a * x + b                         # mul then add: two roundings, like the IR
    s = 1.0 / (1.0 + torch.exp(-z))       # tensor.py:214-215
    ds = s * (1.0 - s)                    # forward_ad.py sigmoid rule y(1-y)
    want_x = yb * (ds * a)
    assert max_rel(y, s) <= 1e-14
    assert max_rel(dx, want_x) <= 1e-14
    ta, tb = yb * (ds * x), yb * ds
    for got, t in ((da, ta), (db, tb)):
        assert bool(((got - t.sum(0)).abs() <= 1e-12 * t.abs().sum(0).clamp_min(1.0)).all())


def test_shape_errors_are_value_errors(fused_module):
    # broadcast conflicts and wrong output shapes: ValueError like tensor.py:118-119
    a = torch.zeros(5, device="cuda")
    x = torch.zeros((3, 4), device="cuda")
    with pytest.raises(ValueError, match="broadcast"):
        F.fused_map(fused_module, "affsig", [a, x, a])
    with pytest.raises(ValueError):
        F.fused_map(fused_module, "affsig", [x[0], x, x[0]], out=torch.empty((4, 3), device="cuda"))


def test_random_broadcast_patterns_vs_oracle(fused_module):
    """Random trailing-aligned broadcast patterns (rank 1-4, size-1 axes,
    missing leading axes, one-element tensors, f64 scalars) for a 3-operand
    function: primal and every cotangent in f64 vs the oracle (tensor.py:
    108-140 broadcasting, 327-345 reduce_to).  Exercises every canonical
    2-D kind (FULL/ROW/COL/one-element/scalar), the row-owner and folded
    1-D modes, and the expand fallback for patterns that are not 2-D."""
    rng = np.random.default_rng(99)
    for case in range(24):
        rank = int(rng.integers(1, 5))
        out = tuple(int(v) for v in rng.integers(2, 7, rank))
        if case % 6 == 0:
            out = (int(rng.integers(300, 700)),) + out[1:]  # one long axis: many rows / folding
        shapes = []
        for _ in range(3):
            kind = rng.integers(0, 4)
            if kind == 0:
                shapes.append(None)  # f64 scalar
                continue
            drop = int(rng.integers(0, rank))  # missing leading axes
            shp = list(out[drop:])
            for d in range(len(shp)):
                if rng.random() < 0.4:
                    shp[d] = 1
            shapes.append(tuple(shp))
        if all(s is None or np.prod(s) < np.prod(out) for s in shapes):
            shapes[1] = out  # the output shape must be reached by some operand
        args, host = [], []
        for shp in shapes:
            if shp is None:
                v = float(rng.uniform(-1.5, 1.5))
                args.append(v)
                host.append(v)
            else:
                a = rng.uniform(-1.5, 1.5, shp)
                args.append(torch.from_numpy(a).cuda())
                host.append(a)
        yb = rng.uniform(-1, 1, out)
        y, bars = F.fused_map_grad(fused_module, "mixed", args, torch.from_numpy(yb).cuda(), want_primal=True)
        p, parts = OS.vec_eval(fused_module, "mixed", host)
        assert max_rel(y, p) <= 1e-13, (case, out, shapes)
        for i, (shp, bar) in enumerate(zip(shapes, bars)):
            want = OS.reduce_to(np.broadcast_to(yb * parts[i], out), () if shp is None else shp)
            assert max_rel(bar, want) <= 1e-11, (case, i, out, shapes)


def test_random_broadcast_patterns_f32(fused_module):
    """The same random patterns in fp32 (vectorised and scalar access paths):
    primal <= 1e-6 (reference rel metric), cotangents within 1e-6 * sum|terms|."""
    rng = np.random.default_rng(7)
    for case in range(16):
        rank = int(rng.integers(1, 4))
        out = tuple(int(v) for v in rng.integers(2, 9, rank))
        if case % 4 == 0:
            out = out[:-1] + (int(rng.choice([1024, 2048, 1000])),)  # wide rows: vector path
        shapes = []
        for _ in range(3):
            if rng.random() < 0.2:
                shapes.append(None)
                continue
            shp = [1 if rng.random() < 0.4 else d for d in out[int(rng.integers(0, rank)):]]
            shapes.append(tuple(shp))
        if all(s is None or np.prod(s) < np.prod(out) for s in shapes):
            shapes[0] = out
        args, host = [], []
        for shp in shapes:
            if shp is None:
                v = float(np.float32(rng.uniform(-1.5, 1.5)))
                args.append(v)
                host.append(v)
            else:
                a = rng.uniform(-1.5, 1.5, shp).astype(np.float32)
                args.append(torch.from_numpy(a).cuda())
                host.append(a.astype(np.float64))
        yb = rng.uniform(-1, 1, out).astype(np.float32)
        y, bars = F.fused_map_grad(fused_module, "mixed", args, torch.from_numpy(yb).cuda(), want_primal=True)
        p, parts = OS.vec_eval(fused_module, "mixed", host)
        assert max_rel(y, p) <= 1e-6, (case, out, shapes)
        for i, (shp, bar) in enumerate(zip(shapes, bars)):
            terms = np.broadcast_to(yb.astype(np.float64) * parts[i], out)
            tgt = () if shp is None else shp
            want = OS.reduce_to(terms, tgt)
            bound = OS.reduce_to(np.abs(terms), tgt)
            err = np.abs(np.asarray(bar.double().cpu().numpy()).reshape(np.shape(want)) - want)
            assert (err <= 1e-6 * np.maximum(1.0, bound) + 1e-7).all(), (case, i, out, shapes)


@pytest.mark.parametrize("xshape,ashape,msg", [((0,), (0,), "(0,) to (1,)"), ((0, 5), (5,), "(0, 5) to (1, 5)"),
                                               ((3, 0), (0,), "(0,) to (3, 1)")])
def test_empty_operands_raise_like_the_reference(fused_module, xshape, ashape, msg):
    """The reference broadcasts extents with max() (tensor.py:108-121), so an
    empty operand meets a result extent of 1 it cannot fill, and bcast_to
    raises ValueError("cannot broadcast ...") (tensor.py:124-140, from
    interp.py's _spread_flat) -- for fused_map and fused_map_with_partials
    alike (checked against the unmodified reference: the messages below are
    its own).  The device path raises the same, before any launch."""
    args = [torch.zeros(ashape, device="cuda", dtype=torch.float64) + 0.5,
            torch.zeros(xshape, device="cuda", dtype=torch.float64) + 0.2,
            torch.zeros(ashape, device="cuda", dtype=torch.float64) + 0.1]
    yb = torch.zeros(xshape, device="cuda", dtype=torch.float64)
    for call in (lambda: F.fused_map(fused_module, "affsig", args),
                 lambda: F.fused_map_with_partials(fused_module, "affsig", args),
                 lambda: F.fused_map_grad(fused_module, "affsig", args, yb)):
        with pytest.raises(ValueError, match=r"cannot broadcast " + re.escape(msg)):
            call()
    torch.cuda.synchronize()  # and nothing faulted on the device


@pytest.mark.parametrize("xshape,ashape", [((1,), (1,)), ((1, 1), (1,)), ((6, 1), (1,)), ((1, 7), (7,))])
def test_single_element_extents(fused_module, xshape, ashape):
    """One-element extents (the reference's broadcast algebra, tensor.py:108-140):
    forward and gradient values against the oracle."""
    rng = np.random.default_rng(len(xshape) * 10 + sum(xshape))
    x = rng.uniform(-2, 2, xshape)
    a = rng.uniform(-2, 2, ashape)
    b = rng.uniform(-2, 2, ashape)
    yb = rng.uniform(-1, 1, xshape)
    args = [torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()]
    y = F.fused_map(fused_module, "affsig", args)
    _, (da, dx, db) = F.fused_map_grad(fused_module, "affsig", args, torch.from_numpy(yb).cuda())
    torch.cuda.synchronize()
    p, parts = OS.vec_eval(fused_module, "affsig", [a, x, b])
    assert max_rel(y, p) <= 1e-13
    assert max_rel(dx, yb * parts[1]) <= 1e-13
    assert max_rel(da, OS.reduce_to(yb * parts[0], ashape)) <= 1e-12
    assert max_rel(db, OS.reduce_to(yb * parts[2], ashape)) <= 1e-12


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("xshape,ashape", [((1 << 20,), None), ((1 << 20,), (1 << 20,)), ((1, 1 << 18), (1 << 18,)),
                                           ((1 << 18, 1), (1 << 18, 1)), ((1000003,), (1,))])
def test_long_one_dimensional_extents(fused_module, dtype, xshape, ashape):
    """1-D and single-row / single-column problems of up to 2^20 elements (the
    runtime folds a long row into rows of a power-of-two width, or walks a
    column operand per row): values and the broadcast cotangents (full
    reductions for scalars, reduce_to otherwise) against the oracle."""
    rng = np.random.default_rng(sum(xshape))
    x = rng.uniform(-2, 2, xshape)
    yb = rng.uniform(-1, 1, xshape)
    if ashape is None:
        a, b = 0.7, -0.3
        args = [a, torch.from_numpy(x).to(dtype).cuda(), b]
        host = [a, x, b]
    else:
        a = rng.uniform(-2, 2, ashape)
        b = rng.uniform(-2, 2, ashape)
        args = [torch.from_numpy(a).to(dtype).cuda(), torch.from_numpy(x).to(dtype).cuda(),
                torch.from_numpy(b).to(dtype).cuda()]
        host = [a, x, b]
    if dtype == torch.float32:  # the oracle sees the fp32 inputs the device sees
        host = [h if isinstance(h, float) else h.astype(np.float32).astype(np.float64) for h in host]
        yb = yb.astype(np.float32).astype(np.float64)
    y = F.fused_map(fused_module, "affsig", args)
    _, (da, dx, db) = F.fused_map_grad(fused_module, "affsig", args, torch.from_numpy(yb).to(dtype).cuda())
    p, parts = OS.vec_eval(fused_module, "affsig", host)
    tol = TOL[dtype]
    assert max_rel(y, p) <= tol
    assert max_rel(dx, yb * parts[1]) <= tol
    for got, part, h in ((da, parts[0], host[0]), (db, parts[2], host[2])):
        if isinstance(h, float):
            want = float((yb * part).sum())
            assert abs(float(got.reshape(-1)[0]) - want) <= max(tol, 1e-12) * np.abs(yb * part).sum()
        else:
            assert max_rel(got, OS.reduce_to(yb * part, h.shape)) <= max(tol, 1e-12) * 10


def test_fuzz_corpus_in_fp32():
    """The same 60 reference-progen programs (branches, loops, select,
    pow_int, itof) through the fp32 kernels: primal, pack partials and K2
    cotangents against the fp64 kernels on the same fp32-representable
    inputs, within the north star's 1e-6 for fp32 elementwise work (the rel
    metric; measured worst 8.3e-7)."""
    import json
    import os

    from conftest import GOLDEN
    from paper_1811_01457_b200.irtext import parse_ir

    with open(os.path.join(GOLDEN, "fuzz.json")) as f:
        d = json.load(f)
    m = parse_ir(d["ir"])
    worst = 0.0
    for case in d["cases"]:
        a64 = [torch.tensor(np.asarray(decode(a), dtype=np.float32).astype(np.float64), dtype=torch.float64,
                            device="cuda") for a in case["args"]]
        a32 = [t.float() for t in a64]
        p64, parts64 = F.fused_map_with_partials(m, case["fn"], a64)
        p32, parts32 = F.fused_map_with_partials(m, case["fn"], a32)
        _, cots32 = F.fused_map_grad(m, case["fn"], a32, torch.ones_like(a32[0]))
        worst = max([worst, max_rel(p32.double(), p64)] + [max_rel(u.double(), v) for u, v in zip(parts32, parts64)]
                    + [max_rel(u.double(), v) for u, v in zip(cots32, parts64)])
    assert worst <= 1e-6, worst


def test_repeated_calls_do_not_grow_device_memory(fused_module):
    """Operands that do not fit the 2-D broadcast pattern are expanded into
    stream-ordered temporaries, and broadcast cotangents use partial-sum
    buffers: every call frees them (and its error paths do too, RAII), so
    device memory is flat over many calls -- only the first calls warm the
    pool."""
    rng = np.random.default_rng(9)
    x = torch.from_numpy(rng.uniform(-2, 2, (64, 3, 257))).cuda()
    a = torch.from_numpy(rng.uniform(-2, 2, (64, 1, 257))).cuda()  # not a 2-D pattern: expanded
    b = torch.from_numpy(rng.uniform(-2, 2, (3, 1))).cuda()
    yb = torch.from_numpy(rng.uniform(-1, 1, (64, 3, 257))).cuda()

    def call():
        F.fused_map(fused_module, "affsig", [a, x, b])
        F.fused_map_grad(fused_module, "affsig", [a, x, b], yb)

    for _ in range(10):
        call()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(200):
        call()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 <= 8 << 20, (free0, free1)


def test_broadcast_beyond_two_giga_elements(fused_module):
    """64-bit indexing in the fused kernels: 2^31 + 2^24 fp32 elements (8.7 GB
    per array), forward and gradient checked on the first and last rows, and
    the broadcast cotangents (sums over all rows) against fp64 row sums."""
    R, C = (1 << 19) + (1 << 12), 4096
    g = torch.Generator(device="cuda").manual_seed(6)
    x = torch.rand((R, C), generator=g, device="cuda") * 4 - 2
    a = torch.rand(C, generator=g, device="cuda") * 4 - 2
    b = torch.rand(C, generator=g, device="cuda") * 4 - 2
    yb = torch.ones((R, C), device="cuda")
    y = F.fused_map(fused_module, "affsig", [a, x, b])
    _, (da, dx, db) = F.fused_map_grad(fused_module, "affsig", [a, x, b], yb)
    torch.cuda.synchronize()
    for r in (0, 1, (1 << 19) - 1, R - 1):
        s = torch.sigmoid(a.double() * x[r].double() + b.double())
        assert max_rel(y[r], s) <= 1e-6
        assert max_rel(dx[r], a.double() * s * (1 - s)) <= 1e-6
    s_all = torch.sigmoid(a.double() * x.double() + b.double())  # 17 GB in fp64: still fits
    want_db = (s_all * (1 - s_all)).sum(0)
    del s_all
    assert float((db.double() - want_db).abs().max()) <= 1e-6 * float(want_db.abs().max())
