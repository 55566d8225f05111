"""C-ABI boundary and codegen checks that need no GPU.

* the in-tree library loads and exports every symbol include/sgb200.h declares;
* every scalar IR function of the parity corpus lowers to CUDA C++ that
  NVRTC compiles for sm_100a, in f32 and f64, for every operand kind;
* the lowering rejects what the reference rejects (non-scalar ops,
  non-f64 parameters) and what the device cannot run (recursion).
"""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_1811_01457_b200 import runtime as rt
from paper_1811_01457_b200.codegen import CodegenError, lower
from paper_1811_01457_b200.irtext import parse_ir


def header_symbols():
    text = open(os.path.join(ROOT, "include", "sgb200.h")).read()
    return re.findall(r"SG_API\s+int\s+(sg_\w+)\s*\(", text)


def test_library_exports_every_declared_symbol():
    lib = rt.load_library()
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(rt.EXPORTS)
    assert lib.sg_version() >= 1


def test_context_creation_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(rt.RuntimeUnavailable):
        rt.context()


def _compile(lo, dtype, kinds, vec):
    arr = (ctypes.c_int * 16)(*(list(kinds) + [0] * (16 - len(kinds))))
    n = ctypes.c_size_t()
    st = rt.load_library().sg_ew_compile_only(lo.source.encode(), lo.k, dtype, arr, vec, 256, 1,
                                              ctypes.byref(n))
    if st:
        raise AssertionError(rt.last_error())
    return n.value


SCALAR_FNS = ["two", "sgau", "poly", "branchy", "gauss", "affsig", "cubeloop", "powloop3",
              "relusq", "pick", "callin", "divy", "mixed", "logp"]


@pytest.mark.parametrize("name", SCALAR_FNS)
def test_corpus_lowers_and_compiles(fused_module, name):
    lo = lower(fused_module, name)
    kinds = [0, 1, 2, 3, 4][: lo.k] if lo.k > 1 else [0]
    assert _compile(lo, rt.SG_F32, kinds, 4) > 0
    assert _compile(lo, rt.SG_F64, kinds, 2) > 0


def test_sites_cover_domain_errors(fused_module):
    lo = lower(fused_module, "logp")
    msgs = {s.message for s in lo.sites}
    assert "log of non-positive value" in msgs
    lo = lower(fused_module, "cubeloop")  # loops get step-budget sites
    assert any(s.message == "step limit exhausted" for s in lo.sites)


def test_rejects_non_scalar_and_bad_signatures(fused_module):
    with pytest.raises(ValueError):  # reference forward_ad._check_scalar_fn
        lower(fused_module, "mapped")
    m = parse_ir("""
func @ints(%x: f64, %n: i64) -> f64 {
^entry:
  ret %x
}
func @tens(%x: f64) -> f64 {
^entry:
  %t = const tensor<2xf64> [1.0, 2.0]
  %s = reduce_sum %t {axis = all}
  ret %s
}
func @rec(%x: f64) -> f64 {
^entry:
  %y = call %x {fn = @rec}
  ret %y
}
""")
    with pytest.raises(ValueError):
        lower(m, "ints")
    with pytest.raises(CodegenError):
        lower(m, "tens")
    with pytest.raises(CodegenError):
        lower(m, "rec")


def _reference():
    """The unmodified reference (CPU container only; absent on GPU boxes)."""
    import sys

    src = "/root/reference/pkg/src"
    if os.path.isdir(src) and src not in sys.path:
        sys.path.append(src)
    return pytest.importorskip("ssagrad", reason="reference not importable here")


def test_parser_matches_reference_structure(fused_module):
    ref = _reference()
    from fused_src import FUSED_SRC

    rm = ref.parse_ir(FUSED_SRC)
    for name, rf in rm.functions.items():
        mf = fused_module.get(name)
        assert [b.name for b in mf.blocks] == [b.name for b in rf.blocks]
        for mb, rb in zip(mf.blocks, rf.blocks):
            assert [mf.value_name(v) for v, _ in mb.params] == [rf.value_name(v) for v, _ in rb.params]
            assert [(i.op, [mf.value_name(o) for o in i.operands]) for i in mb.body] == \
                   [(i.op, [rf.value_name(o) for o in i.operands]) for i in rb.body]


def test_lowering_accepts_reference_module_objects():
    # drop-in: a Module built by the reference itself lowers unchanged
    ref = _reference()
    from fused_src import FUSED_SRC

    rm = ref.parse_ir(FUSED_SRC)
    lo = lower(rm, "affsig")
    assert _compile(lo, rt.SG_F32, [1, 0, 1], 4) > 0


def test_small_step_planner_limits():
    """sg_mlp_small_scratch_bytes (host-only planning of the one-launch step):
    accepts the c1 chain, rejects what the kernel cannot hold."""
    from paper_1811_01457_b200.dense import MlpSmallDesc, _lib

    lib = _lib()

    def plan(sizes, B, loss=0):
        d = MlpSmallDesc()
        d.L, d.B, d.loss, d.scale, d.lr = len(sizes) - 1, B, loss, 1.0 / B, 0.05
        for i, v in enumerate(sizes[:5]):
            d.sizes[i] = v
        off = 0
        for l in range(min(d.L, 4)):
            d.w_off[l], d.ldw[l] = off, (sizes[l] + 7) // 8 * 8
            off += sizes[l + 1] * d.ldw[l]
            d.b_off[l] = off
            off += sizes[l + 1]
        n = ctypes.c_int64()
        return lib.sg_mlp_small_scratch_bytes(ctypes.byref(d), ctypes.byref(n)), n.value

    rc, n = plan((784, 32, 10), 128)
    assert rc == 0 and n >= 256 + 128 * 8 + 128 * 32 * 4 + 128 * 42 * 4
    assert plan((784, 32, 10), 128, loss=2)[0] != 0         # BCE: layer path
    assert plan((784, 32, 10), 1024)[0] != 0                # batch beyond 512
    assert plan((2048, 32, 10), 128)[0] != 0                # width beyond 1024
    assert plan((8,) * 6, 64)[0] != 0                       # 5 layers
    assert plan((1024, 1024, 1024), 512)[0] != 0            # working set beyond shared memory


def test_bindings_reject_wrong_dtypes_and_shapes_before_any_launch():
    """The C descriptors carry no dtype: the Python bindings validate dtypes
    (an fp32 epilogue into a bf16 buffer would write past it) and inner
    dimensions (no silent truncation), raising ValueError before the library
    is called -- so these run on CPU tensors."""
    import torch

    from paper_1811_01457_b200.dense import dense_backward, dense_desc
    from paper_1811_01457_b200.gemm import bmm, gemm

    bf, f64 = torch.bfloat16, torch.float64
    A = torch.zeros((64, 32), dtype=bf)
    B = torch.zeros((48, 32), dtype=bf)
    with pytest.raises(ValueError, match="out must be"):
        gemm(A, B, out=torch.zeros((64, 48), dtype=bf))          # fp32 result into bf16
    with pytest.raises(ValueError, match="A must be"):
        gemm(A.float(), B, out=torch.zeros((64, 48)))             # fp32 operand for bf16 precision
    with pytest.raises(ValueError, match="out_lp is a bf16"):
        gemm(A.float(), B.float(), precision="tf32", out_lp=torch.zeros((64, 48), dtype=bf))
    with pytest.raises(ValueError, match="inner dimensions differ"):
        gemm(A, torch.zeros((48, 16), dtype=bf), out=torch.zeros((64, 48)))
    with pytest.raises(ValueError, match="needs aux"):
        gemm(A, B, epilogue="act_grad", out=torch.zeros((64, 48)))
    with pytest.raises(ValueError, match="cannot hold"):
        bmm(A[None], B[None], out=torch.zeros((1, 32, 48)))
    with pytest.raises(ValueError, match="out must be"):
        bmm(A[None].double(), B[None].double(), out=torch.zeros((1, 64, 48)), precision="strict_fp64")
    with pytest.raises(ValueError, match="b must be"):
        dense_desc(A, B, torch.zeros(48, dtype=f64), "tanh", "bf16")
    d = dense_desc(A, B, torch.zeros(48), "tanh", "bf16")
    dZ = torch.zeros((64, 48), dtype=bf)
    with pytest.raises(ValueError, match="dW must be"):
        dense_backward(d, dZ, torch.zeros((48, 32), dtype=bf), torch.zeros(48))
    with pytest.raises(ValueError, match="dX must be"):
        dense_backward(d, dZ, torch.zeros((48, 32)), torch.zeros(48), dX=torch.zeros((64, 32), dtype=f64))
    d64 = dense_desc(A.double(), B.double(), torch.zeros(48, dtype=f64), "tanh", "strict_fp64")
    with pytest.raises(ValueError, match="dZ must be"):
        dense_backward(d64, dZ.float(), torch.zeros((48, 32), dtype=f64), torch.zeros(48, dtype=f64))


def test_leading_dimension_of_size_one_views():
    """gemm's row stride of views with a size-1 dimension (torch reports them
    contiguous whatever their strides): a one-column slice of a padded buffer
    keeps the buffer's row stride."""
    import torch

    from paper_1811_01457_b200.gemm import _ld

    buf = torch.zeros((6, 8))
    assert _ld(buf[:, :1]) == 8
    assert _ld(buf[:1, :]) == 8
    assert _ld(buf[:, :5]) == 8
    assert _ld(torch.zeros((1, 24))) == 24


def test_ctypes_mirrors_match_the_c_header(tmp_path):
    """Every ctypes mirror of an include/sgb200.h struct has the C layout:
    the same size and field offsets as gcc computes from the header."""
    import shutil
    import subprocess

    from paper_1811_01457_b200.dense import DenseDesc, DenseGrad, MlpSmallDesc
    from paper_1811_01457_b200.gemm import ChainProblem, GemmDesc

    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    mirrors = {"sg_tensor": rt.SgTensor, "sg_gemm_desc": GemmDesc, "sg_chain_problem": ChainProblem,
               "sg_dense_desc": DenseDesc, "sg_dense_grad": DenseGrad, "sg_mlp_small_desc": MlpSmallDesc}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "sgb200.h"', "int main(void) {"]
    for cname, cls in mirrors.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("  return 0;\n}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        cname, field, value = line.split()
        got[(cname, field)] = int(value)
    for cname, cls in mirrors.items():
        assert got[(cname, "size")] == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[(cname, fname)] == getattr(cls, fname).offset, (cname, fname)


def test_broadcast_rule_rejects_empty_operands_like_the_reference():
    """fused._broadcast: the reference's max() extents (tensor.py:108-121) and
    its can_expand check (tensor.py:124-132): an empty operand raises the
    reference's ValueError before anything reaches the device."""
    import numpy as np

    from paper_1811_01457_b200.fused import _broadcast

    assert _broadcast([np.zeros((3, 1)), np.zeros((4,)), 0.5]) == (3, 4)
    assert _broadcast([np.zeros((1,)), np.zeros((6, 1))]) == (6, 1)
    for shapes, msg in (([(0,), (0,)], "(0,) to (1,)"), ([(5,), (0, 5)], "(0, 5) to (1, 5)"),
                        ([(0,), (3, 0)], "(0,) to (3, 1)")):
        with pytest.raises(ValueError, match=r"cannot broadcast " + re.escape(msg)):
            _broadcast([np.zeros(s) for s in shapes])
    with pytest.raises(ValueError, match="do not broadcast"):
        _broadcast([np.zeros((3,)), np.zeros((4,))])


def test_chain_problem_limit_matches_the_library():
    """gemm.CHAIN_MAX_PROBLEMS (ChainEngine falls back to the layer path above
    it) is the kernel's own MAX_PROBS (gemm_chain.cu)."""
    import re as _re

    from paper_1811_01457_b200.gemm import CHAIN_MAX_PROBLEMS

    src = open(os.path.join(ROOT, "paper_1811_01457_b200", "csrc", "gemm_chain.cu")).read()
    assert int(_re.search(r"constexpr int MAX_PROBS = (\d+);", src).group(1)) == CHAIN_MAX_PROBLEMS
