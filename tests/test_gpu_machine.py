"""GpuMachine: the reference's augmented IR (printed by the reference,
tests/golden/machine.json) evaluated with every tensor op on the device.

Covers SURVEY §8(f)1 (the two-seed DAN step, nn_train.py:337-375) and
§8(f)3 (arbitrary aug/pb IR, reverse_ad.py:619-663): analytic programs,
generated programs with branches/loops over tensors, fused_map via
fused_pack, and the DAN loss with BCE clamps (select masks), two heads and
two pullback seeds.  f64 throughout; only libm ulps differ from the
reference (exp/log/tanh), so the tolerance is 1e-12 (rel metric).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, decode, max_rel
from paper_1811_01457_b200.irtext import parse_ir


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "machine.json")) as f:
        return json.load(f)


def _args(case):
    out = []
    for a in case["args"]:
        if isinstance(a, dict) and "i64" in a:
            out.append(int(a["i64"]))
        else:
            out.append(decode(a))
    return out


def test_reference_printed_ir_parses(golden):
    # CPU: the independent .ssair reader accepts every augmented module
    for key in ("analytic", "corpus", "dan"):
        m = parse_ir(golden[key]["ir"])
        assert any(n.endswith("__aug") for n in m.functions)
        assert any(n.endswith("__pb") for n in m.functions)


gpu = pytest.mark.gpu


def _machine_grad(module, name, args, seeds=None):
    from paper_1811_01457_b200.gpu_machine import grad

    g = grad(module, name, tuple(args), seeds)
    fn = module.get(name)
    return [g[pv] for pv, ty in fn.params if ty.kind in ("f64", "tensor")]


@gpu
@pytest.mark.parametrize("key", ["analytic", "corpus"])
def test_gpu_machine_gradients_match_reference(golden, key):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    m = parse_ir(golden[key]["ir"])
    for case in golden[key]["cases"]:
        got = _machine_grad(m, case["fn"], _args(case))
        for g, want in zip(got, case["grads"]):
            assert max_rel(g, decode(want)) <= 1e-12, case["fn"]


@gpu
def test_dan_step_two_seeds_matches_reference(golden):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1811_01457_b200.gpu_machine import GpuMachine

    d = golden["dan"]
    m = parse_ir(d["ir"])
    fn = m.get(d["fn"])
    args = _args(d)
    # one augmented forward, two pullback replays of the same traces (nn_train.py:360-363)
    mach = GpuMachine(m)
    out = mach.call(d["fn"] + "__aug", tuple(args))
    c_loss, d_loss, blog, vstack = out
    g_c = mach.call(d["fn"] + "__pb", (blog, vstack, 1.0, 0.0))
    g_d = mach.call(d["fn"] + "__pb", (blog, vstack, 0.0, 1.0))
    assert abs(c_loss - d["losses"][0]) <= 1e-12 and abs(d_loss - d["losses"][1]) <= 1e-12
    diff = [i for i, (_, ty) in enumerate(fn.params) if ty.kind in ("f64", "tensor")]
    for k, (gc, gd) in enumerate(zip(g_c, g_d)):
        assert max_rel(gc, decode(d["g_c"][k])) <= 1e-12, k
        assert max_rel(gd, decode(d["g_d"][k])) <= 1e-12, k
    # SGD on the summed gradient (nn_train.py:365-372) -> the reference's new params
    n_w = len(d["new_params"])
    for k in range(n_w):
        p = np.asarray(args[diff[k]], dtype=np.float64)
        step = (g_c[k] + g_d[k]).double().cpu().numpy()
        assert max_rel(p - d["lr"] * step, decode(d["new_params"][k])) <= 1e-12, k


@gpu
def test_gpu_machine_domain_error_location():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1811_01457_b200.fused import EvalError
    from paper_1811_01457_b200.gpu_machine import eval_function

    m = parse_ir("""
func @f(%x: tensor<4xf64>) -> f64 {
^entry:
  %one = const f64 1.0
  %y = sub %x, %one
  %l = log %y
  %s = reduce_sum %l {axis = all}
  ret %s
}
""")
    with pytest.raises(EvalError) as ei:
        eval_function(m, "f", (np.array([2.0, 3.0, 0.5, 0.25]),))
    e = ei.value
    # reference: unary_math raises for the first element in row-major order
    assert (e.function, e.block, e.index) == ("f", "entry", 2)
    assert e.message == f"log of non-positive value {0.5 - 1.0!r}"
    s = eval_function(m, "f", (np.array([2.0, 3.0, 4.0, 5.0]),))[0]
    assert abs(s - float(np.sum(np.log(np.array([1.0, 2.0, 3.0, 4.0]))))) <= 1e-14


def _probe_acc(H, yd, alpha=0.1):
    """Host restatement of nn_train._domain_probe_acc (nn_train.py:378-393):
    test-side evaluation only (the probe is not on the accelerated path)."""
    X = np.column_stack([H, np.ones(H.shape[0])])
    t = np.array([1.0 if y == 1 else -1.0 for y in yd])
    acc = 0.0
    for tr, te in ((slice(0, None, 2), slice(1, None, 2)), (slice(1, None, 2), slice(0, None, 2))):
        gram = X[tr].T @ X[tr] + alpha * np.eye(X.shape[1])
        w = np.linalg.solve(gram, X[tr].T @ t[tr])
        acc += float(np.mean((X[te] @ w >= 0.0) == (t[te] > 0.0)))
    return acc / 2.0


@gpu
@pytest.mark.parametrize("lam", ["0.0", "1.0"])
def test_dan_training_reproduces_frozen_history(lam):
    """Acceptance criterion 7 (test_acceptance.py:293-322): the reference's
    50-epoch DAN trainings, every epoch record, reproduced on the GPU."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1811_01457_b200.dan import train_epochs
    from paper_1811_01457_b200.gpu_machine import GpuMachine

    with open(os.path.join(GOLDEN, "dan_train.json")) as f:
        d = json.load(f)
    m = parse_ir(d["ir"])
    cfg = d["cfg"]
    X = np.array(d["X"])
    yc, yd = np.array(d["yc"], dtype=np.float64), np.array(d["yd"], dtype=np.float64)
    params = [torch.tensor(decode(p), dtype=torch.float64, device="cuda") for p in d["params"]]
    ref = d["history"][lam]
    got = []

    def on_epoch(epoch, ps, c_mean, d_mean):
        yc_hat, yd_hat, H = GpuMachine(m).call(d["eval_fn"], tuple(ps) + (X,))
        yc_hat, H = yc_hat.cpu().numpy(), H.cpu().numpy()
        got.append({"epoch": epoch, "c_loss": c_mean, "d_loss": d_mean,
                    "class_acc": float(np.mean((yc_hat >= 0.5) == (yc == 1))),
                    "domain_probe_acc": _probe_acc(H, [int(v) for v in yd])})

    train_epochs(m, d["loss_fn"], params, X, yc, yd, lam=float(lam), lr=cfg["lr"],
                 epochs=cfg["epochs"], batch_size=cfg["batch_size"], seed=cfg["seed"], on_epoch=on_epoch)
    assert len(got) == len(ref)
    worst = 0.0
    for g, r in zip(got, ref):
        worst = max(worst, abs(g["c_loss"] - r["c_loss"]), abs(g["d_loss"] - r["d_loss"]))
        assert g["class_acc"] == r["class_acc"], g
        assert g["domain_probe_acc"] == r["domain_probe_acc"], g
    assert worst <= 1e-9, worst


def test_reference_printed_spmd_ir_parses():
    # CPU: vectorised aug/pb programs (per-lane traces, bmm) read back from text
    with open(os.path.join(GOLDEN, "spmd.json")) as f:
        d = json.load(f)
    m = parse_ir(d["ir"])
    for c in d["cases"]:
        assert f"{c['fn']}__aug__batched_B{c['lanes']}" in m.functions
        assert f"{c['fn']}__pb__batched_B{c['lanes']}" in m.functions


@gpu
def test_batched_grad_matches_reference():
    """spmd_batch.batched_grad (spmd_batch.py:718-745) on the
    GPU -- per-lane traces (TapeBatch), lane-divergent loop trips (powloop),
    and lanes carrying weights (@net: matmul -> bmm, one batched launch)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1811_01457_b200.gpu_machine import batched_grad

    with open(os.path.join(GOLDEN, "spmd.json")) as f:
        d = json.load(f)
    m = parse_ir(d["ir"])
    for c in d["cases"]:
        fn = m.get(c["fn"])
        g = batched_grad(m, c["fn"], c["lanes"], tuple(decode(a) for a in c["args"]),
                         tuple(decode(s) for s in c["seeds"]))
        got = [g[pv] for pv, ty in fn.params if ty.kind in ("f64", "tensor")]
        assert len(got) == len(c["grads"])
        for k, (gv, want) in enumerate(zip(got, c["grads"])):
            assert max_rel(gv, decode(want)) <= 1e-12, (c["fn"], k)


@gpu
@pytest.mark.parametrize("key", ["analytic", "corpus"])
def test_device_tape_backprop_matches_reference(golden, key):
    """the rule table on the device builder (CudaBuilder),
    swept over a runtime trace recorded on the GpuMachine (the reference's
    oracle.trace_grad, oracle.py:140-197), vs the reference's gradients."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1811_01457_b200.taping import trace_grad

    m = parse_ir(golden[key]["ir"])
    for case in golden[key]["cases"]:
        fn = m.get(case["fn"])
        g = trace_grad(m, case["fn"], tuple(_args(case)))
        got = [g[pv] for pv, ty in fn.params if ty.kind in ("f64", "tensor")]
        for gv, want in zip(got, case["grads"]):
            assert max_rel(gv, decode(want)) <= 1e-12, case["fn"]


def test_reference_transforms_come_from_the_installed_reference():
    """grad / batched_grad take the reference's own IR transforms (augment,
    vectorize: host-side IR, out of scope here) from an importable ssagrad or
    the bench's reference install (baseline/_ref); without either they fail
    with an ImportError that says what to do (no silent fallback)."""
    from paper_1811_01457_b200 import gpu_machine as G

    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    try:
        import ssagrad  # noqa: F401
        have = True
    except ImportError:
        have = os.path.isdir(os.path.join(ref, "ssagrad"))
    if not have:
        with pytest.raises(ImportError, match="reference's IR transform"):
            G._reference_transforms()
        return
    augment, vectorize = G._reference_transforms()
    assert callable(augment) and callable(vectorize)
