"""GpuMachine: evaluate reference IR programs with every tensor op on the device.

Drop-in for ``ssagrad.interp.Machine`` (interp.py:177-356): same
``call(name, args)`` and block-walker semantics (``run_blocks``,
interp.py:95-138: shared step budget, ``EvalError(function, block, index,
message)`` wrapping a ``DomainError``), so the reference's augmented
forward/pullback pairs (``augment``, reverse_ad.py:619-630) run on the
B200 unchanged -- this is the ``GpuMachine`` of SURVEY §8(b)/(f)3.

Value model (reference: DenseTensor | float | int | bool | Tape):

* tensors are torch CUDA tensors (f64 by default, the reference dtype);
* f64 scalars, i64, bool and traces stay host-side Python values, exactly
  as the reference computes scalar bookkeeping;
* every tensor-valued op runs on the device through this repo's kernels:
  elementwise ops, comparisons and masks through the NVRTC fused-broadcast
  kernels (one tiny scalar function per op, compiled once), ``matmul``
  through ``sg_gemm`` (STRICT_FP64: the reference's ascending-k fold, bit-
  exact), reductions through ``sg_reduce_to``, ``fused_map``/``fused_pack``
  through the fused kernels.  Pure data movement (transpose, reshape,
  stack, slicing, broadcast materialisation) uses torch tensor views.
"""

from __future__ import annotations

import ctypes
import math

from . import fused as F
from . import runtime as rt
from .gemm import bmm, gemm
from .ir import kind_of
from .irtext import parse_ir

DEFAULT_STEP_LIMIT = 2_000_000  # interp.py:23

_OPS_SRC = """
func @add(%a: f64, %b: f64) -> f64 {
^entry:
  %r = add %a, %b
  ret %r
}
func @sub(%a: f64, %b: f64) -> f64 {
^entry:
  %r = sub %a, %b
  ret %r
}
func @mul(%a: f64, %b: f64) -> f64 {
^entry:
  %r = mul %a, %b
  ret %r
}
func @div(%a: f64, %b: f64) -> f64 {
^entry:
  %r = div %a, %b
  ret %r
}
func @neg(%a: f64) -> f64 {
^entry:
  %r = neg %a
  ret %r
}
func @exp(%a: f64) -> f64 {
^entry:
  %r = exp %a
  ret %r
}
func @log(%a: f64) -> f64 {
^entry:
  %r = log %a
  ret %r
}
func @tanh(%a: f64) -> f64 {
^entry:
  %r = tanh %a
  ret %r
}
func @sigmoid(%a: f64) -> f64 {
^entry:
  %r = sigmoid %a
  ret %r
}
func @relu(%a: f64) -> f64 {
^entry:
  %r = relu %a
  ret %r
}
func @lt(%a: f64, %b: f64) -> f64 {
^entry:
  %c = lt %a, %b
  %one = const f64 1.0
  %zero = const f64 0.0
  %r = select %c, %one, %zero
  ret %r
}
func @gt(%a: f64, %b: f64) -> f64 {
^entry:
  %c = gt %a, %b
  %one = const f64 1.0
  %zero = const f64 0.0
  %r = select %c, %one, %zero
  ret %r
}
func @eq(%a: f64, %b: f64) -> f64 {
^entry:
  %c = eq %a, %b
  %one = const f64 1.0
  %zero = const f64 0.0
  %r = select %c, %one, %zero
  ret %r
}
func @selmask(%m: f64, %a: f64, %b: f64) -> f64 {
^entry:
  %zero = const f64 0.0
  %z = eq %m, %zero
  %r = select %z, %b, %a
  ret %r
}
"""

_OPS = parse_ir(_OPS_SRC)
_POW: dict = {}


def _pow_module(n: int):
    if n not in _POW:
        _POW[n] = parse_ir(f"""
func @pow(%a: f64) -> f64 {{
^entry:
  %r = pow_int %a {{n = {n}}}
  ret %r
}}
""")
    return _POW[n]


class Tape:
    """Persistent LIFO trace (interp.py:38-61); empty tape has rest None."""

    __slots__ = ("top", "rest")

    def __init__(self, top=None, rest=None):
        self.top = top
        self.rest = rest

    @property
    def empty(self) -> bool:
        return self.rest is None

    def __len__(self):
        n, t = 0, self
        while not t.empty:
            n, t = n + 1, t.rest
        return n


EMPTY_TAPE = Tape()


class TapeBatch:
    """One independent tape per lane (interp.py:64-70)."""

    __slots__ = ("lanes",)

    def __init__(self, lanes):
        self.lanes = tuple(lanes)


def _lane_value(v, lane_shape):
    """A lane's top coerced to the per-lane shape, or None (interp.py:368-380)."""
    if lane_shape:
        if _is_tensor(v) and tuple(v.shape) == tuple(lane_shape):
            return v
        return None
    if isinstance(v, bool):
        return 1.0 if v else 0.0
    if isinstance(v, (int, float)):
        return float(v)
    if _is_tensor(v) and v.dim() == 0:
        return v
    return None


def _is_tensor(v) -> bool:
    import torch

    return isinstance(v, torch.Tensor)


class GpuMachine:
    """Evaluator over a module with tensor ops on the GPU."""

    def __init__(self, module, step_limit: int = DEFAULT_STEP_LIMIT, dtype=None):
        import torch

        self.module = module
        self.budget = [step_limit]
        self.dtype = dtype or torch.float64

    # ------------------------------------------------------------ values
    def to_device(self, v):
        """Reference runtime value -> machine value (DenseTensor -> CUDA tensor)."""
        import numpy as np
        import torch

        if isinstance(v, torch.Tensor):
            return v.to(device="cuda", dtype=self.dtype).contiguous()
        if isinstance(v, np.ndarray):
            return torch.from_numpy(np.ascontiguousarray(v)).to(device="cuda", dtype=self.dtype)
        if hasattr(v, "data") and isinstance(getattr(v, "data"), np.ndarray):
            return torch.from_numpy(np.ascontiguousarray(v.data)).to(device="cuda", dtype=self.dtype)
        return v

    # ------------------------------------------------------------- calls
    def call(self, name: str, args: tuple) -> tuple:
        fn = self.module.get(name)
        return self.run_blocks(fn, tuple(self.to_device(a) for a in args))

    def run_blocks(self, fn, args: tuple) -> tuple:
        """interp.run_blocks (interp.py:95-138) with device tensor ops."""
        if len(args) != len(fn.params):
            raise F.EvalError(fn.name, "", -1, f"expected {len(fn.params)} arguments, got {len(args)}")
        blocks = {b.name: b for b in fn.blocks}
        env = {}
        cur = fn.blocks[0]
        binds = args
        while True:
            for (vid, _), v in zip(cur.params, binds):
                env[vid] = v
            for i, ins in enumerate(cur.body):
                self.budget[0] -= 1
                if self.budget[0] < 0:
                    raise F.EvalError(fn.name, cur.name, i, "step limit exhausted")
                try:
                    env[ins.result] = self.dispatch(ins, env)
                except rt.DomainError as e:
                    raise F.EvalError(fn.name, cur.name, i, str(e)) from e
            self.budget[0] -= 1
            if self.budget[0] < 0:
                raise F.EvalError(fn.name, cur.name, len(cur.body), "step limit exhausted")
            t = cur.term
            if t is None:
                raise F.EvalError(fn.name, cur.name, len(cur.body), "missing terminator")
            if hasattr(t, "values"):
                return tuple(env[v] for v in t.values)
            if hasattr(t, "then_target"):
                if bool(env[t.cond]):
                    cur, binds = blocks[t.then_target], tuple(env[a] for a in t.then_args)
                else:
                    cur, binds = blocks[t.else_target], tuple(env[a] for a in t.else_args)
            else:
                cur, binds = blocks[t.target], tuple(env[a] for a in t.args)

    # ----------------------------------------------------- elementwise
    def _ew(self, name: str, *vals, module=None):
        """Device elementwise op through the fused kernels (broadcasting)."""
        m = module or _OPS
        try:
            return F.fused_map(m, name, list(vals), dtype=self.dtype)
        except F.EvalError as e:
            raise rt.DomainError(e.message) from None

    def _binary(self, op, x, y):
        if not _is_tensor(x) and not _is_tensor(y):
            if isinstance(x, int) and isinstance(y, int) and not isinstance(x, bool):
                if op == "div":
                    raise rt.DomainError("div is not defined on i64")
                return {"add": x + y, "sub": x - y, "mul": x * y}[op]
            if op == "div":  # tensor.py:197-202
                if y == 0.0:
                    raise rt.DomainError("division by zero")
                return x / y
            return {"add": x + y, "sub": x - y, "mul": x * y}[op]
        if op == "div" and not _is_tensor(y) and y == 0.0:
            raise rt.DomainError("division by zero")
        return self._ew(op, x, y)  # a zero divisor element raises "division by zero" (tensor.py:203-204)

    def _unary(self, op, x):
        if not _is_tensor(x):
            if op == "exp":
                return math.exp(x)
            if op == "log":
                if x <= 0.0:
                    raise rt.DomainError(f"log of non-positive value {x!r}")
                return math.log(x)
            if op == "tanh":
                return math.tanh(x)
            if op == "sigmoid":
                return 1.0 / (1.0 + math.exp(-x))
            if op == "relu":
                return x if x > 0.0 else 0.0
            raise rt.DomainError(op)
        if op == "log":
            try:
                return F.fused_map(_OPS, "log", [x], dtype=self.dtype)
            except F.EvalError as e:  # first failing element in row-major order, like unary_math
                v = float(x.reshape(-1)[e.element].item())
                raise rt.DomainError(f"log of non-positive value {v!r}") from None
        return self._ew(op, x)

    # ----------------------------------------------------- reductions
    def _reduce_to(self, x, shape):
        """tensor.reduce_to (tensor.py:327-345) on the device; () -> float."""
        import torch

        lib = rt.load_library()
        if shape:
            out = torch.empty(tuple(shape), dtype=x.dtype, device="cuda")
            od = rt.tensor_desc(out)
        else:
            out = torch.empty((1,), dtype=x.dtype, device="cuda")
            od = rt.tensor_desc(out)
            od.ndim = 0
        ad = rt.tensor_desc(x.contiguous())
        rt.check(lib.sg_reduce_to(rt.context(), ctypes.byref(ad), None, ctypes.byref(od), rt.stream_ptr()),
                 "reduce_to")
        return float(out.item()) if not shape else out

    def _reduce_sum(self, x, axis):
        """tensor.reduce_sum (tensor.py:295-318)."""
        if axis == "all":
            return self._reduce_to(x, ())
        if axis == "tail":
            lead = (x.shape[0],) + (1,) * (x.dim() - 1)
            return self._reduce_to(x, lead).reshape(x.shape[0])
        ax = int(axis)
        if not 0 <= ax < x.dim():
            raise ValueError(f"axis {ax} out of range for shape {tuple(x.shape)}")
        if x.dim() == 1:
            return self._reduce_to(x, ())
        keep = tuple(1 if d == ax else s for d, s in enumerate(x.shape))
        return self._reduce_to(x, keep).reshape(tuple(s for d, s in enumerate(x.shape) if d != ax))

    def _matmul(self, a, b):
        """tensor.matmul (tensor.py:351-361): strict ascending-k fold on the GPU."""
        import torch

        if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[0]:
            raise ValueError(f"matmul shapes {tuple(a.shape)} x {tuple(b.shape)}")
        out = torch.empty((a.shape[0], b.shape[1]), dtype=a.dtype, device="cuda")
        prec = "strict_fp64" if a.dtype == torch.float64 else "strict_fp32"
        gemm(a.contiguous(), b.contiguous(), b_mn=True, precision=prec, out=out)
        return out

    def _bmm(self, a, b):
        """tensor.bmm (tensor.py:364-369): every lane's strict fold in ONE batched launch."""
        import torch

        if a.dim() != 3 or b.dim() != 3 or a.shape[0] != b.shape[0] or a.shape[2] != b.shape[1]:
            raise ValueError(f"bmm shapes {tuple(a.shape)} x {tuple(b.shape)}")
        out = torch.empty((a.shape[0], a.shape[1], b.shape[2]), dtype=a.dtype, device="cuda")
        prec = "strict_fp64" if a.dtype == torch.float64 else "strict_fp32"
        bmm(a.contiguous(), b.contiguous(), out, b_mn=True, precision=prec)
        return out

    # ----------------------------------------------------------- tapes
    # Per-lane traces of vectorised programs (spmd_batch.py, interp.py:271-318):
    # a TapeBatch holds one persistent tape per lane.
    def _tape_push(self, t, v, per_lane: bool):
        if isinstance(t, Tape) and per_lane:
            t = TapeBatch((t,) * v.shape[0])
        if isinstance(t, TapeBatch):
            if per_lane:
                rows = list(v.unbind(0)) if _is_tensor(v) else list(v)
                return TapeBatch(tuple(Tape(r, l) for r, l in zip(rows, t.lanes)))
            return TapeBatch(tuple(Tape(v, l) for l in t.lanes))
        return Tape(v, t)

    def _tape_top(self, t, ty):
        import torch

        if isinstance(t, TapeBatch):
            lane_shape = tuple(ty.shape[1:])
            vals = [_lane_value(l.top, lane_shape) if not l.empty else None for l in t.lanes]
            if lane_shape:
                z = torch.zeros(lane_shape, dtype=self.dtype, device="cuda")
                return torch.stack([z if v is None else v for v in vals], 0)
            host = [0.0 if v is None else v for v in vals]
            if all(not _is_tensor(v) for v in host):
                return torch.tensor(host, dtype=self.dtype, device="cuda").reshape(tuple(ty.shape))
            return torch.stack([v.reshape(()).to(self.dtype) if _is_tensor(v)
                                else torch.tensor(float(v), dtype=self.dtype, device="cuda")
                                for v in host]).reshape(tuple(ty.shape))
        if t.empty:
            return self._zero(ty)
        return t.top

    def _zero(self, ty):
        import torch

        k = kind_of(ty)
        if k == "f64":
            return 0.0
        if k == "i64":
            return 0
        if k == "bool":
            return False
        if k == "tensor":
            return torch.zeros(tuple(ty.shape), dtype=self.dtype, device="cuda")
        if k == "tape":
            return EMPTY_TAPE
        if k == "tapes":
            return TapeBatch((EMPTY_TAPE,) * int(ty.lanes))
        raise ValueError(f"no zero for {ty}")

    # -------------------------------------------------------- dispatch
    def dispatch(self, ins, env):
        import torch

        op = ins.op
        a = ins.operands
        if op == "const":
            ty = ins.attrs["ty"]
            v = ins.attrs["value"]
            k = kind_of(ty)
            if k == "tensor":
                return torch.tensor(list(v), dtype=self.dtype, device="cuda").reshape(tuple(ty.shape))
            return float(v) if k == "f64" else (int(v) if k == "i64" else bool(v))
        if op in ("add", "sub", "mul", "div"):
            return self._binary(op, env[a[0]], env[a[1]])
        if op == "neg":
            x = env[a[0]]
            return self._ew("neg", x) if _is_tensor(x) else -x
        if op in ("exp", "log", "tanh", "sigmoid", "relu"):
            return self._unary(op, env[a[0]])
        if op == "pow_int":
            n = int(ins.attrs["n"])
            x = env[a[0]]
            if _is_tensor(x):
                return self._ew("pow", x, module=_pow_module(n))
            acc = 1.0
            for _ in range(n):
                acc = acc * x
            return acc
        if op == "itof":
            return float(env[a[0]])
        if op in ("lt", "gt", "eq"):
            x, y = env[a[0]], env[a[1]]
            if _is_tensor(x) or _is_tensor(y):
                return self._ew(op, x, y)  # 0/1 mask (tensor.py:261-273)
            return x < y if op == "lt" else (x > y if op == "gt" else x == y)
        if op == "select":
            c, x, y = env[a[0]], env[a[1]], env[a[2]]
            if isinstance(c, bool):
                return x if c else y
            if isinstance(x, TapeBatch):  # per-lane trace merge (interp.py:233-238)
                keep = c.ne(0).tolist()
                return TapeBatch(tuple(xt if k else yt for k, xt, yt in zip(keep, x.lanes, y.lanes)))
            return self._ew("selmask", c, x, y)  # tensor.py:276-281
        if op == "matmul":
            return self._matmul(env[a[0]], env[a[1]])
        if op == "bmm":
            return self._bmm(env[a[0]], env[a[1]])
        if op == "transpose":
            return env[a[0]].transpose(-1, -2).contiguous()
        if op == "reshape":
            return env[a[0]].reshape(tuple(ins.attrs["shape"])).contiguous()
        if op == "reduce_sum":
            return self._reduce_sum(env[a[0]], ins.attrs.get("axis", "all"))
        if op == "bcast":
            x = env[a[0]]
            shape = tuple(ins.attrs["shape"])
            if _is_tensor(x):
                return x.expand(shape).contiguous()
            return torch.full(shape, float(x), dtype=self.dtype, device="cuda")
        if op == "reduce_to":
            x = env[a[0]]
            shape = tuple(ins.attrs["shape"])
            if tuple(x.shape) == shape:
                return x
            return self._reduce_to(x, shape)
        if op == "stack":
            vals = [env[o] for o in a]
            if all(not _is_tensor(v) for v in vals):
                return torch.tensor(vals, dtype=self.dtype, device="cuda")
            return torch.stack(vals, ins.attrs.get("axis", 0)).contiguous()
        if op == "unstack":
            x = env[a[0]]
            sl = x.select(ins.attrs.get("axis", 0), ins.attrs["index"])
            return float(sl.item()) if sl.dim() == 0 else sl.contiguous()
        if op == "fused_map":
            vals = [env[o] for o in a]
            return F.fused_map(self.module, ins.attrs["fn"].name, vals, dtype=self.dtype)
        if op == "fused_pack":
            return self._fused_pack(ins.attrs["fn"].name, [env[o] for o in a])
        if op == "call":
            return self.run_blocks(self.module.get(ins.attrs["fn"].name), tuple(env[o] for o in a))[0]
        if op == "tape_new":
            return EMPTY_TAPE
        if op == "tape_push":
            return self._tape_push(env[a[0]], env[a[1]], bool(ins.attrs.get("per_lane", False)))
        if op == "tape_top":
            return self._tape_top(env[a[0]], ins.attrs["ty"])
        if op == "tape_rest":
            t = env[a[0]]
            if isinstance(t, TapeBatch):
                return TapeBatch(tuple(l.rest if not l.empty else l for l in t.lanes))
            return t.rest if not t.empty else t
        if op == "tape_spread":
            return TapeBatch((env[a[0]],) * int(ins.attrs["lanes"]))
        if op == "tape_expect_empty":
            t = env[a[0]]
            lanes = t.lanes if isinstance(t, TapeBatch) else (t,)
            left = [len(l) for l in lanes if not l.empty]
            if left:
                raise rt.DomainError(f"trace should be used up, {max(left)} entries remain")
            return True
        raise rt.DomainError(f"op '{op}' has no evaluation rule")

    def _fused_pack(self, name, vals):
        """``fused_pack`` (interp.py:334-352): (1+k, *shape) on the device."""
        import torch

        if not any(_is_tensor(v) for v in vals):
            p, parts = F.fused_map_with_partials(self.module, name, [float(v) for v in vals], dtype=self.dtype)
            return torch.tensor([p, *parts], dtype=self.dtype, device="cuda")
        primal, parts = F.fused_map_with_partials(self.module, name, vals, dtype=self.dtype)
        return torch.stack([primal] + list(parts))


def eval_function(module, name: str, args: tuple, step_limit: int = DEFAULT_STEP_LIMIT) -> tuple:
    """``interp.eval_function`` (interp.py:383-390) on the GPU."""
    return GpuMachine(module, step_limit).call(name, args)


def _reference_transforms():
    """The reference's host-side IR transforms (``augment``, ``vectorize``:
    reverse_ad.py:619-630, spmd_batch.py) -- out of this repo's scope (they
    emit IR, they compute nothing).  Taken from an importable ``ssagrad``, else
    from the reference install this repo's bench uses (``baseline/_ref``)."""
    try:
        import ssagrad
    except ImportError:
        import os
        import sys

        ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
        if not os.path.isdir(os.path.join(ref, "ssagrad")):
            raise ImportError("grad / batched_grad need the reference's IR transform (ssagrad.augment / "
                              "vectorize) for a module without {name}__aug / __pb: install the reference "
                              "(baseline/_ref) or pass augment= / vectorize=, or parse a pre-augmented module")
        sys.path.append(ref)
        import ssagrad
    return ssagrad.augment, ssagrad.vectorize


def grad(module, name: str, args: tuple, seeds: tuple | None = None, step_limit: int = DEFAULT_STEP_LIMIT,
         augment=None) -> dict:
    """``reverse_ad.grad`` (reverse_ad.py:633-663) running the aug/pb pair on the GPU.

    The source transform itself is the reference's (``augment``, passed in
    or imported from ``ssagrad``); alternatively the module may already
    contain ``{name}__aug`` / ``{name}__pb`` (e.g. parsed from text).
    """
    fn = module.get(name)
    if seeds is None:
        if len(fn.results) != 1 or kind_of(fn.results[0]) != "f64":
            raise ValueError(f"@{name} has results {fn.results}; seeds are required")
        seeds = (1.0,)
    if len(seeds) != len(fn.results):
        raise ValueError(f"expected {len(fn.results)} seeds, got {len(seeds)}")
    aug, pb = f"{name}__aug", f"{name}__pb"
    if aug not in module.functions or pb not in module.functions:
        if augment is None:
            augment = _reference_transforms()[0]  # the reference transform (host-side IR)
        augment(module, name)
    m = GpuMachine(module, step_limit)
    out = m.call(aug, tuple(args))
    n = len(fn.results)
    cots = m.call(pb, (out[n], out[n + 1]) + tuple(seeds))
    res = {}
    i = 0
    for pv, ty in fn.params:
        if kind_of(ty) in ("f64", "tensor"):
            res[pv] = cots[i]
            i += 1
    return res


def batched_grad(module, name: str, lanes: int, stacked_args: tuple, seeds: tuple,
                 step_limit: int = DEFAULT_STEP_LIMIT, vectorize=None) -> dict:
    """``spmd_batch.batched_grad`` (spmd_batch.py:718-745) on the GPU: one
    batched augmented forward and one batched pullback of the vectorised
    ``{name}__aug`` / ``{name}__pb`` (lane axis first on every argument and
    seed); per-lane traces live in :class:`TapeBatch`, and every lane's
    matmul runs inside ONE batched launch (``bmm``).  The vectorising
    transform is the reference's (passed in / imported), or the module
    already holds ``{name}__aug__batched_B{lanes}`` (parsed from text)."""
    fn = module.get(name)
    vaug, vpb = f"{name}__aug__batched_B{lanes}", f"{name}__pb__batched_B{lanes}"
    if vaug not in module.functions or vpb not in module.functions:
        augment, ref_vectorize = _reference_transforms()  # the reference transforms (host-side IR)
        vectorize = vectorize or ref_vectorize
        a, p = augment(module, name)
        vectorize(module, a.name, lanes)
        vectorize(module, p.name, lanes)
    m = GpuMachine(module, step_limit)
    outs = m.call(vaug, tuple(stacked_args))
    n = len(fn.results)
    cots = m.call(vpb, (outs[n], outs[n + 1]) + tuple(seeds))
    res = {}
    i = 0
    for pv, ty in fn.params:
        if kind_of(ty) in ("f64", "tensor"):
            res[pv] = cots[i]
            i += 1
    return res
