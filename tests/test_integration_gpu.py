"""INTEGRATION.md §2 exactly as written: the `Machine` subclass a maintainer
would add to the reference, with `_fused_map` / `_fused_pack` dispatched to
this repo's fused kernels, running reference programs through the
reference's own interpreter (`interp.py:190-292`) and its own reverse-mode
transform (`augment`, reverse_ad.py:619-630).  Checked against the
reference's CPU `Machine` on the same module and inputs: f64, only libm ulps
differ (1e-12, the rel metric).  The reference comes from an importable
`ssagrad` or the bench's install (baseline/_ref); skipped without either.
"""
import os
import sys

import numpy as np
import pytest

from conftest import max_rel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

try:
    import ssagrad  # noqa: F401
except ImportError:
    _ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(_ref, "ssagrad")):
        pytest.skip("the reference (ssagrad / baseline/_ref) is not installed", allow_module_level=True)
    sys.path.append(_ref)

from ssagrad import augment, parse_ir  # noqa: E402
from ssagrad.interp import Machine  # noqa: E402
from ssagrad.tensor import DenseTensor  # noqa: E402

import paper_1811_01457_b200 as sg  # noqa: E402


class GpuMachine(Machine):  # INTEGRATION.md §2, verbatim
    def _fused_map(self, ins, vals):                     # interp.py:322-332
        out = sg.fused_map(self.module, ins.attrs["fn"].name, vals)
        return out if isinstance(out, float) else DenseTensor(out.double().cpu().numpy())

    def _fused_pack(self, ins, vals):                    # interp.py:334-352
        primal, parts = sg.fused_map_with_partials(self.module, ins.attrs["fn"].name, vals)
        if isinstance(primal, float):
            return DenseTensor.from_flat((1 + len(parts),), [primal, *parts])
        rows = [primal] + list(parts)
        return DenseTensor(np.stack([r.double().cpu().numpy() for r in rows]))


SRC = """
func @gauss(%a: f64, %c: f64) -> f64 {
^entry:
  %p = mul %a, %c
  %n = neg %p
  %e = exp %n
  %one = const f64 1.0
  %d = add %one, %e
  %r = div %one, %d
  ret %r
}

func @mapped(%x: tensor<4x3xf64>, %b: f64) -> f64 {
^entry:
  %y = fused_map %x, %b {fn = @gauss}
  %s = reduce_sum %y {axis = all}
  ret %s
}

func @scalar(%u: f64, %v: f64) -> f64 {
^entry:
  %y = fused_map %u, %v {fn = @gauss}
  ret %y
}
"""


def _val(v):
    return np.asarray(v.data if isinstance(v, DenseTensor) else v, dtype=np.float64).reshape(-1)


def _close(a, b):
    for u, w in zip(a, b):
        assert max_rel(_val(u), _val(w)) <= 1e-12


@pytest.mark.parametrize("name,args", [
    ("mapped", (DenseTensor(np.linspace(-2.0, 1.3, 12).reshape(4, 3)), 0.7)),
    ("scalar", (0.3, -1.9)),
])
def test_machine_subclass_forward_and_pullback_match_reference(name, args):
    m = parse_ir(SRC)
    _close(GpuMachine(m).call(name, args), Machine(m).call(name, args))
    a, p = augment(m, name)
    out_g = GpuMachine(m).call(a.name, args)
    out_c = Machine(m).call(a.name, args)
    _close(out_g[:1], out_c[:1])
    cots_g = GpuMachine(m).call(p.name, (out_g[1], out_g[2], 1.0))
    cots_c = Machine(m).call(p.name, (out_c[1], out_c[2], 1.0))
    _close(cots_g, cots_c)
