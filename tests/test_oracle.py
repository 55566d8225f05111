"""The oracle is pinned to the reference: every restatement in oracle/ must
reproduce the golden vectors produced by the unmodified reference
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import os

from conftest import GOLDEN, decode, load_npz, max_rel
from oracle import dense as OD
from oracle import scalar as OS


def _args(case):
    return [decode(a) for a in case["args"]]


def test_fused_cases_bit_identical(golden_fused, fused_module):
    # same scalar kernels, same operation order: equality is exact
    for case in golden_fused["cases"]:
        args = _args(case)
        primal, parts = OS.fused_map_with_partials(fused_module, case["fn"], args)
        assert np.array_equal(np.asarray(primal), np.asarray(decode(case["primal"]))), case["fn"]
        for p, g in zip(parts, case["partials"]):
            assert np.array_equal(np.asarray(p), np.asarray(decode(g))), case["fn"]


def test_fused_pullback_matches(golden_fused, fused_module):
    for case in golden_fused["cases"]:
        if case["pullback"] is None:
            continue
        args = _args(case)
        _, parts = OS.fused_map_with_partials(fused_module, case["fn"], args)
        shapes = [a.shape if isinstance(a, np.ndarray) else None for a in args]
        got = OS.fused_map_pullback(parts, shapes, decode(case["ybar"]))
        for g, want in zip(got, case["pullback"]):
            assert np.array_equal(np.asarray(g), np.asarray(decode(want))), case["fn"]


def test_vectorised_oracle_agrees(golden_fused, fused_module):
    for case in golden_fused["cases"]:
        fn = fused_module.get(case["fn"])
        if len(fn.blocks) != 1 or any(i.op == "call" for i in fn.blocks[0].body):
            continue
        args = _args(case)
        if not any(isinstance(a, np.ndarray) for a in args):
            continue
        primal, parts = OS.vec_eval(fused_module, case["fn"], args)
        assert max_rel(primal, decode(case["primal"])) <= 1e-14
        for p, g in zip(parts, case["partials"]):
            assert max_rel(p, decode(g)) <= 1e-14


def test_domain_errors_name_reference_site(golden_fused, fused_module):
    for err in golden_fused["errors"]:
        with pytest.raises(OS.OracleEvalError) as ei:
            OS.fused_map_with_partials(fused_module, err["fn"], _args(err))
        e = ei.value
        assert (e.function, e.block, e.index) == (err["function"], err["block"], err["index"])
        assert e.message == err["message"]


def test_matmul_exact_is_reference_bit_for_bit():
    z = load_npz("tensor.npz")
    for i in range(3):
        a, b, c = z[f"mm{i}_a"], z[f"mm{i}_b"], z[f"mm{i}_c"]
        assert np.array_equal(OD.matmul_exact(a, b), c)
        assert np.array_equal(OD.matmul_cumsum(a, b), c)


def test_strict_fp32_restatement_is_sequential():
    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, (5, 37)).astype(np.float32)
    b = rng.uniform(-1, 1, (37, 3)).astype(np.float32)
    got = OD.matmul_exact(a, b)
    for i in range(5):
        for j in range(3):
            acc = np.float32(a[i, 0] * b[0, j])
            for k in range(1, 37):
                acc = np.float32(acc + np.float32(a[i, k] * b[k, j]))
            assert got[i, j] == acc
    assert np.array_equal(OD.matmul_cumsum(a, b), got)


def test_reduce_to_matches_reference():
    z = load_npz("tensor.npz")
    x = z["rt_x"]
    assert np.array_equal(OS.reduce_to(x, (5,)), z["rt_to_5"])
    assert np.array_equal(OS.reduce_to(x, (4, 1)), z["rt_to_415"])
    assert np.array_equal(OS.reduce_to(x, (1, 4, 5)), z["rt_to_145"])
    assert OS.reduce_to(x, ()) == z["rt_to_all"][0]


@pytest.mark.parametrize("name,acts,loss", [
    ("mlp_c1_b32.npz", ("sigmoid", "identity"), "softmax_xent"),
    ("mlp_mse.npz", ("tanh", "tanh", "identity"), "mse"),
    ("mlp_bce.npz", ("tanh", "identity"), "bce"),
])
def test_mlp_step_matches_reference(name, acts, loss):
    z = load_npz(name)
    L = len(acts)
    params = [(z[f"W{k}"].astype(np.float64), z[f"b{k}"].astype(np.float64)) for k in range(L)]
    X, Y = z["X"].astype(np.float64), z["Y"].astype(np.float64)
    for mode in ("exact", "blas"):
        lv, grads, new = OD.mlp_step(params, X, Y, acts, loss, lr=float(z["lr"][0]), mode=mode)
        assert abs(lv - z["loss"][0]) <= 1e-13 * max(1.0, abs(lv))
        for k, (dW, db) in enumerate(grads):
            assert max_rel(dW, z[f"dW{k}"]) <= 1e-13, (mode, k)
            assert max_rel(db, z[f"db{k}"]) <= 1e-13, (mode, k)


def test_dense_backward_matches_reference_seed():
    z = load_npz("dense_sigmoid.npz")
    W, b = z["W0"].astype(np.float64), z["b0"].astype(np.float64)
    X, Ybar = z["X"].astype(np.float64), z["Y"].astype(np.float64)
    zb, h = OD.dense_forward(X, W, b, "sigmoid", "exact")
    dx, dW, db = OD.dense_backward(Ybar, X, W, zb, h, "sigmoid", "exact")
    assert max_rel(dx, z["dX"]) <= 1e-15
    assert max_rel(dW, z["dW0"]) <= 1e-15
    assert max_rel(db, z["db0"]) <= 1e-15


def test_oracle_reproduces_fuzz_corpus_exactly():
    import json
    import os

    from conftest import GOLDEN
    from paper_1811_01457_b200.irtext import parse_ir

    with open(os.path.join(GOLDEN, "fuzz.json")) as f:
        d = json.load(f)
    m = parse_ir(d["ir"])
    for case in d["cases"][:20]:
        args = [decode(a) for a in case["args"]]
        primal, parts = OS.fused_map_with_partials(m, case["fn"], args)
        assert np.array_equal(primal, decode(case["primal"])), case["fn"]
        for p, g in zip(parts, case["partials"]):
            assert np.array_equal(p, decode(g)), case["fn"]


def test_domain_conditions_match_reference_fixture():
    """oracle.dense.check_domain raises where the unmodified reference raised on
    tests/golden/domain.json (OverflowError from math.exp; DomainError -- which
    run_blocks wraps into EvalError -- from div / log, with the same message),
    and stays silent on the extreme-but-finite cases."""
    import json

    from oracle import dense as OD

    with open(os.path.join(GOLDEN, "domain.json")) as f:
        cases = json.load(f)
    assert len(cases) >= 8
    for c in cases:
        params = [(np.array(w), np.array(b)) for w, b in c["params"]]
        args = (params, np.array(c["X"]), np.array(c["Y"]), tuple(c["acts"]), c["loss_kind"])
        if c["raises"] == "OverflowError":
            with pytest.raises(OverflowError, match="^math range error$"):
                OD.check_domain(*args)
        elif c["raises"] == "EvalError":
            assert c["cause"] == "DomainError"
            with pytest.raises(OD.DomainError) as ei:
                OD.check_domain(*args)
            assert str(ei.value) == c["message"]
        else:
            assert OD.check_domain(*args) is None
