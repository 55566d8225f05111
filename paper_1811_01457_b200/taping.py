"""Runtime-taped gradients on the GPU: the rule backend of SURVEY §8(b)2.

The reference writes every pullback rule once against a small builder
protocol (rules.py:11-21) and evaluates the rules eagerly with
``NumericBuilder`` (rules.py:242-311), e.g. in ``oracle.tape_backprop``
(oracle.py:156-181), its gradient cross-check that is independent of the
IR transform.  This module is the device third backend:

* :class:`CudaBuilder` -- the builder protocol on device values (torch CUDA
  tensors through this repo's kernels: fused elementwise kernels, the
  strict GEMM, ``sg_reduce_to``; scalars stay host floats);
* :data:`SAVES` / :func:`rule_backward` -- the per-op pullback rules
  (rules.py:40-218) restated against that protocol;
* :func:`trace_eval` / :func:`tape_backprop` / :func:`trace_grad` -- the
  tracer and the reverse sweep of oracle.py:77-200 over a
  :class:`~.gpu_machine.GpuMachine`: values are boxed with a slot id that
  moves with them across block arguments and calls, every executed
  differentiable primitive is recorded with its saved operands, and one
  backwards sweep applies the rules.
"""

from __future__ import annotations

from .gpu_machine import DEFAULT_STEP_LIMIT, GpuMachine, _is_tensor
from .ir import BOOL, F64, I64, kind_of, tensor_type


# ------------------------------------------------------------- builder
class CudaBuilder:
    """Builder protocol (rules.py:11-21) evaluated on the device."""

    def __init__(self, machine: GpuMachine):
        self.m = machine

    def add(self, a, b):
        return self.m._binary("add", a, b)

    def sub(self, a, b):
        return self.m._binary("sub", a, b)

    def mul(self, a, b):
        return self.m._binary("mul", a, b)

    def div(self, a, b):
        return self.m._binary("div", a, b)

    def neg(self, a):
        return self.m._ew("neg", a) if _is_tensor(a) else -a

    def const_f64(self, x):
        return float(x)

    def const_tensor(self, shape, values):
        import torch

        return torch.tensor(list(values), dtype=self.m.dtype, device="cuda").reshape(tuple(shape))

    def pow_int(self, a, n):
        from .gpu_machine import _pow_module

        if _is_tensor(a):
            return self.m._ew("pow", a, module=_pow_module(int(n)))
        acc = 1.0
        for _ in range(int(n)):
            acc = acc * a
        return acc

    def gt_zero_mask(self, a):
        if _is_tensor(a):
            return self.m._ew("gt", a, 0.0)
        return 1.0 if a > 0.0 else 0.0

    def select(self, c, x, y):
        if isinstance(c, bool):
            return x if c else y
        return self.m._ew("selmask", c, x, y)

    def matmul(self, a, b):
        return self.m._matmul(a, b)

    def bmm(self, a, b):
        return self.m._bmm(a, b)

    def transpose(self, a):
        return a.transpose(-1, -2).contiguous()

    def reshape(self, a, shape):
        return a.reshape(tuple(shape)).contiguous()

    def bcast(self, a, shape):
        import torch

        shape = tuple(shape)
        if not _is_tensor(a):
            return torch.full(shape, float(a), dtype=self.m.dtype, device="cuda")
        return a.expand(shape).contiguous()

    def take(self, a, index, axis):
        sl = a.select(int(axis), int(index))
        return float(sl.item()) if sl.dim() == 0 else sl.contiguous()

    def reduce_like(self, x, ref_ty):
        """rules.py:302-311: sum a cotangent down to its operand's type."""
        import torch

        if kind_of(ref_ty) == "f64":
            return self.m._reduce_to(x, ()) if _is_tensor(x) else x
        shape = tuple(ref_ty.shape)
        if not _is_tensor(x):
            return torch.full(shape, float(x), dtype=self.m.dtype, device="cuda")
        if tuple(x.shape) == shape:
            return x
        return self.m._reduce_to(x, shape)


# --------------------------------------------------------------- rules
# Saved values per op (rules.py:195-218): "o0"/"o1" operands, "res" result.
SAVES = {
    "add": (), "sub": (), "neg": (), "transpose": (), "reshape": (), "reduce_sum": (),
    "bcast": (), "reduce_to": (), "stack": (), "unstack": (),
    "mul": ("o0", "o1"), "div": ("o0", "o1"), "matmul": ("o0", "o1"), "bmm": ("o0", "o1"),
    "exp": ("res",), "tanh": ("res",), "sigmoid": ("res",),
    "log": ("o0",), "relu": ("o0",), "pow_int": ("o0",), "select": ("o0",),
    "fused_map": ("pack",),
}


def _numel(shape) -> int:
    n = 1
    for d in shape:
        n *= int(d)
    return n


def rule_backward(op, b, attrs, ts, sv, ybar):
    """Cotangents of op's operands (None for non-differentiable ones),
    rules.py:40-185 evaluated on builder ``b``."""
    if op == "add":
        return b.reduce_like(ybar, ts[0]), b.reduce_like(ybar, ts[1])
    if op == "sub":
        return b.reduce_like(ybar, ts[0]), b.reduce_like(b.neg(ybar), ts[1])
    if op == "mul":
        x, y = sv
        return b.reduce_like(b.mul(ybar, y), ts[0]), b.reduce_like(b.mul(ybar, x), ts[1])
    if op == "div":  # d(x/y) = ybar/y, -ybar*x/(y*y)
        x, y = sv
        return (b.reduce_like(b.div(ybar, y), ts[0]),
                b.reduce_like(b.neg(b.div(b.mul(ybar, x), b.mul(y, y))), ts[1]))
    if op == "neg":
        return (b.neg(ybar),)
    if op == "exp":
        return (b.mul(ybar, sv[0]),)
    if op == "log":
        return (b.div(ybar, sv[0]),)
    if op == "tanh":  # saved result h: 1 - h*h
        return (b.mul(ybar, b.sub(b.const_f64(1.0), b.mul(sv[0], sv[0]))),)
    if op == "sigmoid":  # saved result s: s (1 - s)
        return (b.mul(ybar, b.mul(sv[0], b.sub(b.const_f64(1.0), sv[0]))),)
    if op == "relu":
        return (b.mul(ybar, b.gt_zero_mask(sv[0])),)
    if op == "pow_int":
        n = int(attrs["n"])
        if n == 0:
            return (b.mul(ybar, b.const_f64(0.0)),)
        return (b.mul(ybar, b.mul(b.const_f64(float(n)), b.pow_int(sv[0], n - 1))),)
    if op == "select":  # the condition has no cotangent
        zero = b.const_f64(0.0)
        return (None, b.reduce_like(b.select(sv[0], ybar, zero), ts[1]),
                b.reduce_like(b.select(sv[0], zero, ybar), ts[2]))
    if op in ("matmul", "bmm"):  # (ybar . v^T, a^T . ybar)
        a, v = sv
        mm = b.matmul if op == "matmul" else b.bmm
        return mm(ybar, b.transpose(v)), mm(b.transpose(a), ybar)
    if op == "transpose":
        return (b.transpose(ybar),)
    if op == "reshape":
        return (b.reshape(ybar, ts[0].shape),)
    if op == "reduce_sum":
        src = tuple(ts[0].shape)
        axis = attrs.get("axis", "all")
        if axis == "all" or (axis != "tail" and len(src) == 1):
            return (b.bcast(ybar, src),)
        if axis == "tail":
            kept = (src[0],) + (1,) * (len(src) - 1)
        else:
            kept = src[:axis] + (1,) + src[axis + 1:]
        return (b.bcast(b.reshape(ybar, kept), src),)
    if op == "bcast":
        return (b.reduce_like(ybar, ts[0]),)
    if op == "reduce_to":
        return (b.bcast(ybar, ts[0].shape),)
    if op == "stack":
        axis = attrs.get("axis", 0)
        return tuple(b.take(ybar, i, axis) for i in range(len(ts)))
    if op == "unstack":  # one-hot of the taken slice times the (reshaped) cotangent
        src = tuple(ts[0].shape)
        axis, index = attrs.get("axis", 0), attrs["index"]
        inner = _numel(src[axis + 1:])
        hot = [0.0] * _numel(src)
        for o in range(_numel(src[:axis])):
            base = (o * src[axis] + index) * inner
            hot[base:base + inner] = [1.0] * inner
        onehot = b.const_tensor(src, hot)
        if len(src) == 1:
            return (b.mul(onehot, ybar),)
        return (b.mul(onehot, b.reshape(ybar, src[:axis] + (1,) + src[axis + 1:])),)
    if op == "fused_map":  # pack row 1+i is d f / d operand_i (rules.py:177-185)
        (pack,) = sv
        return tuple(b.reduce_like(b.mul(ybar, b.take(pack, 1 + i, 0)), t) for i, t in enumerate(ts))
    raise KeyError(op)


# -------------------------------------------------------------- tracer
class Tracked:
    """A runtime value with the trace slot it was produced in."""

    __slots__ = ("v", "slot")

    def __init__(self, v, slot: int):
        self.v = v
        self.slot = slot

    def __bool__(self):  # branch conditions reach the block walker boxed
        return bool(self.v)


class TraceNode:
    __slots__ = ("op", "attrs", "arg_slots", "arg_types", "saved", "out_slot")

    def __init__(self, op, attrs, arg_slots, arg_types, saved, out_slot):
        self.op, self.attrs, self.arg_slots = op, attrs, arg_slots
        self.arg_types, self.saved, self.out_slot = arg_types, saved, out_slot


class Trace:
    def __init__(self):
        self.nodes: list[TraceNode] = []
        self.params: list = []  # (vid, type, slot)
        self.result_slots: tuple = ()


def _rt_type(v):
    if isinstance(v, bool):
        return BOOL
    if isinstance(v, int):
        return I64
    if _is_tensor(v):
        return tensor_type(*v.shape)
    return F64


class TracingMachine(GpuMachine):
    """GpuMachine whose dispatch records the differentiable primitives
    (oracle.py:77-137): operands are unboxed for the device ops, results
    boxed with fresh slots, block arguments and call results keep theirs."""

    def __init__(self, module, step_limit: int = DEFAULT_STEP_LIMIT, dtype=None):
        super().__init__(module, step_limit, dtype)
        self.trace = Trace()
        self._slots = 0

    def _box(self, v) -> Tracked:
        t = Tracked(v, self._slots)
        self._slots += 1
        return t

    def run_traced(self, name: str, args: tuple) -> tuple:
        fn = self.module.get(name)
        boxed = tuple(self._box(self.to_device(a)) for a in args)
        self.trace.params = [(vid, ty, b.slot) for (vid, ty), b in zip(fn.params, boxed)]
        out = self.run_blocks(fn, boxed)
        self.trace.result_slots = tuple(b.slot for b in out)
        return tuple(b.v for b in out)

    def dispatch(self, ins, env):
        op = ins.op
        boxed = tuple(env[o] for o in ins.operands)
        vals = tuple(b.v for b in boxed)
        if op == "call":  # callee bodies are traced inline, slots flow through
            return self.run_blocks(self.module.get(ins.attrs["fn"].name), boxed)[0]
        if op == "fused_map":
            pack = self._fused_pack(ins.attrs["fn"].name, list(vals))
            row0 = pack.select(0, 0)
            res = self._box(float(row0.item()) if row0.dim() == 0 else row0.contiguous())
            self.trace.nodes.append(TraceNode(op, ins.attrs, tuple(b.slot for b in boxed),
                                              tuple(_rt_type(v) for v in vals), (pack,), res.slot))
            return res
        value = GpuMachine.dispatch(self, ins, dict(zip(ins.operands, vals)))
        res = self._box(value)
        saves = SAVES.get(op)
        if saves is not None:
            saved = tuple(value if s == "res" else vals[0] if s == "o0" else vals[1] for s in saves)
            self.trace.nodes.append(TraceNode(op, ins.attrs, tuple(b.slot for b in boxed),
                                              tuple(_rt_type(v) for v in vals), saved, res.slot))
        return res


def trace_eval(module, name: str, args: tuple, step_limit: int = DEFAULT_STEP_LIMIT):
    """Evaluate @name on the GPU while recording its trace (oracle.py:140-150)."""
    m = TracingMachine(module, step_limit)
    out = m.run_traced(name, args)
    return out, m.trace, m


def tape_backprop(trace: Trace, seeds: tuple, builder) -> dict:
    """One reverse sweep (oracle.py:153-181): cotangents of the traced
    function's differentiable parameters, zeros for unreached ones."""
    if len(seeds) != len(trace.result_slots):
        raise ValueError(f"expected {len(trace.result_slots)} seeds, got {len(seeds)}")
    acc: dict = {}

    def accumulate(slot, v):
        cur = acc.get(slot)
        acc[slot] = v if cur is None else builder.add(cur, v)

    for slot, seed in zip(trace.result_slots, seeds):
        accumulate(slot, seed)
    for node in reversed(trace.nodes):
        ybar = acc.get(node.out_slot)
        if ybar is None:
            continue
        cots = rule_backward(node.op, builder, node.attrs, node.arg_types, node.saved, ybar)
        for slot, cot in zip(node.arg_slots, cots):
            if cot is not None:
                accumulate(slot, cot)
    out = {}
    for vid, ty, slot in trace.params:
        if kind_of(ty) in ("f64", "tensor"):
            got = acc.get(slot)
            out[vid] = builder.reduce_like(0.0, ty) if got is None else got
    return out


def trace_grad(module, name: str, args: tuple, seeds: tuple | None = None,
               step_limit: int = DEFAULT_STEP_LIMIT) -> dict:
    """``oracle.trace_grad`` (oracle.py:189-197) with the device builder."""
    fn = module.get(name)
    if seeds is None:
        seeds = (1.0,) * len(fn.results)
    seeds = tuple(seeds)
    _, trace, m = trace_eval(module, name, args, step_limit)
    return tape_backprop(trace, tuple(m.to_device(s) for s in seeds), CudaBuilder(m))
