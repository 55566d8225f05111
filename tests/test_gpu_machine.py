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
