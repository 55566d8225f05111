"""Fused broadcast of a user scalar function and its adjoint, on the B200.

Drop-in counterparts of the reference's broadcast entry points:

* :func:`fused_map` -- the ``fused_map`` IR op (``interp.py:322-332``):
  ``y[e] = f(args[e'])`` with trailing-aligned broadcasting;
* :func:`fused_map_with_partials` -- ``forward_ad.fused_map_with_partials``
  (``forward_ad.py:194-223``): primal plus one partial per argument, via the
  ``fused_pack`` layout ``(1+k, *shape)`` (``interp.py:334-352``);
* :func:`fused_map_pullback` -- ``forward_ad.fused_map_pullback``
  (``forward_ad.py:226-235``): ``reduce_like(ybar * partial_i, type_i)``;
* :func:`fused_map_grad` -- the fused adjoint kernel (K2): recomputes the
  duals from the inputs and writes every operand's cotangent in one pass,
  which is what the pullback of ``fused_map`` computes
  (``rules.py:177-185``) without materialising the pack.

Arguments are ``torch`` CUDA tensors, numpy arrays, reference
``DenseTensor`` objects (anything with an ndarray ``.data``) or Python
floats.  Tensors compute in their own dtype (f32 or f64); all-scalar calls
compute in f64 and return floats, like the reference.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import runtime as rt
from .codegen import Lowered, check_scalar_fn, lower
from .ir import kind_of

DEFAULT_STEP_LIMIT = 2_000_000  # reference interp.py:23


class EvalError(Exception):
    """Mirror of the reference ``interp.EvalError`` (interp.py:26-35)."""

    def __init__(self, function: str, block: str, index: int, message: str):
        self.function = function
        self.block = block
        self.index = index
        self.message = message
        where = f"@{function} ^{block}" if block else f"@{function}"
        if index >= 0:
            where += f" instr {index}"
        super().__init__(f"{where}: {message}")


# ------------------------------------------------------------ kernel cache

_lock = threading.Lock()
_lowered: dict = {}   # (id(module), name, fingerprint) -> Lowered
_kernels: dict = {}   # (ctx, key, dtype) -> sg_kernel*


def _fingerprint(module, fn) -> tuple:
    out = []
    seen = set()
    stack = [fn]
    while stack:
        f = stack.pop()
        if f.name in seen:
            continue
        seen.add(f.name)
        out.append((f.name, id(f), sum(len(b.body) for b in f.blocks), len(f.blocks)))
        for b in f.blocks:
            for ins in b.body:
                if ins.op == "call":
                    stack.append(module.get(ins.attrs["fn"].name))
    return tuple(sorted(out))


def lowered_for(module, name: str) -> Lowered:
    fn = module.get(name)
    key = (id(module), name, _fingerprint(module, fn))
    with _lock:
        lo = _lowered.get(key)
    if lo is None:
        lo = lower(module, name)
        with _lock:
            _lowered[key] = lo
    return lo


def kernel_for(lo: Lowered, dtype_c: int) -> int:
    ctx = rt.context()
    key = (ctx, lo.key, dtype_c)
    with _lock:
        h = _kernels.get(key)
    if h is None:
        lib = rt.load_library()
        out = ctypes.c_void_p()
        rt.check(lib.sg_ew_compile(ctx, lo.source.encode(), lo.key.encode(), lo.k, dtype_c,
                                   ctypes.byref(out)), "sg_ew_compile")
        h = out.value
        with _lock:
            _kernels[key] = h
    return h


# -------------------------------------------------------- argument intake

def _as_device(v, dtype=None):
    import torch

    if isinstance(v, torch.Tensor):
        t = v
    elif isinstance(v, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(v))
    elif hasattr(v, "data") and isinstance(getattr(v, "data"), np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(v.data))  # reference DenseTensor
    else:
        return None
    if t.dim() == 0:
        raise ValueError("tensors have rank >= 1; use a plain float for scalars")
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    if not t.is_cuda:
        t = t.to("cuda", non_blocking=False)
    return t.contiguous()


def _intake(args, dtype=None):
    """Split args into device tensors / floats and pick the compute dtype."""
    import torch

    tens = [v for v in args if _is_tensorish(v)]
    if dtype is None:
        dtype = torch.float64
        for v in tens:
            dt = v.dtype if isinstance(v, torch.Tensor) else None
            if dt is None:
                arr = v if isinstance(v, np.ndarray) else v.data
                dt = torch.float32 if arr.dtype == np.float32 else torch.float64
            if dt == torch.float32:
                dtype = torch.float32
                break
    out = []
    for v in args:
        if _is_tensorish(v):
            out.append(_as_device(v, dtype))
        else:
            out.append(float(v))
    return out, dtype


def _is_tensorish(v) -> bool:
    import torch

    if isinstance(v, (torch.Tensor, np.ndarray)):
        return True
    return hasattr(v, "data") and isinstance(getattr(v, "data"), np.ndarray)


def _broadcast(vals) -> tuple:
    shape: tuple = ()
    for v in vals:
        if isinstance(v, float):
            continue
        s = tuple(v.shape)
        n = max(len(shape), len(s))
        out = []
        for i in range(1, n + 1):
            a = shape[-i] if i <= len(shape) else 1
            b = s[-i] if i <= len(s) else 1
            if a != b and a != 1 and b != 1:
                raise ValueError(f"shapes {shape} and {s} do not broadcast")
            out.append(max(a, b))
        shape = tuple(reversed(out))
    # tensor.py:124-132 (can_expand, via bcast_to in interp.py's _spread_flat):
    # with the max() rule above a zero extent meets 1 as 1, and an empty
    # operand cannot fill it -- the reference raises ValueError
    for v in vals:
        if isinstance(v, float):
            continue
        s = tuple(v.shape)
        if any(s[-i] != shape[-i] and s[-i] != 1 for i in range(1, len(s) + 1)):
            raise ValueError(f"cannot broadcast {s} to {shape}")
    return shape


def _descs(vals, dtype_c):
    return [rt.scalar_desc(v, dtype_c) if isinstance(v, float) else rt.tensor_desc(v) for v in vals]


def _raise_eval(lo: Lowered, ctx: int, stream: int) -> None:
    lib = rt.load_library()
    elem = ctypes.c_int64()
    site = ctypes.c_int32()
    st = lib.sg_ew_check(ctx, stream, ctypes.byref(elem), ctypes.byref(site))
    if st == rt.SG_OK:
        return
    if st != rt.SG_EDOMAIN:
        rt.check(st, "sg_ew_check")
    s = lo.sites[site.value - 1]
    err = EvalError(s.function, s.block, s.index, s.message)
    err.element = int(elem.value)  # flat index of the first failing element
    raise err


def check_errors(module, name: str, stream=None) -> None:
    """Synchronise and raise the first element error of earlier unchecked calls."""
    _raise_eval(lowered_for(module, name), rt.context(), rt.stream_ptr(stream))


def set_step_limit(limit: int) -> None:
    rt.check(rt.load_library().sg_ew_set_step_limit(rt.context(), int(limit)))


# ------------------------------------------------------------- public API

def fused_map(module, name: str, args, *, dtype=None, out=None, check: bool = True,
              stream=None):
    """``y = f.(args...)`` on the device (reference ``fused_map`` op)."""
    import torch

    fn = module.get(name)
    check_scalar_fn(fn)
    if len(args) != len(fn.params):
        raise ValueError(f"@{fn.name} takes {len(fn.params)} arguments, got {len(args)}")
    lo = lowered_for(module, name)
    vals, dtype = _intake(args, dtype)
    shape = _broadcast(vals)
    dtype_c = rt.dtype_code(dtype)
    kern = kernel_for(lo, dtype_c)
    ctx = rt.context()
    st = rt.stream_ptr(stream)
    y = out if out is not None else torch.empty(shape or (1,), dtype=dtype, device="cuda")
    yd = rt.tensor_desc(y)
    if not shape:
        yd.ndim = 0
    arr = rt.desc_array(_descs(vals, dtype_c))
    rt.check(rt.load_library().sg_ew_forward(ctx, kern, len(vals), arr, ctypes.byref(yd), st),
             "fused_map")
    if check:
        _raise_eval(lo, ctx, st)
    if not shape:
        return float(y.reshape(-1)[0].item())
    return y


def fused_map_with_partials(module, name: str, args, step_limit: int = DEFAULT_STEP_LIMIT, *,
                            dtype=None, stream=None):
    """(primal, [partial_i]) -- reference ``forward_ad.py:194-223``."""
    import torch

    fn = module.get(name)
    check_scalar_fn(fn)
    if len(args) != len(fn.params):
        raise ValueError(f"@{fn.name} takes {len(fn.params)} arguments, got {len(args)}")
    lo = lowered_for(module, name)
    vals, dtype = _intake(args, dtype)
    shape = _broadcast(vals)
    k = len(vals)
    dtype_c = rt.dtype_code(dtype)
    kern = kernel_for(lo, dtype_c)
    ctx = rt.context()
    if step_limit != DEFAULT_STEP_LIMIT:
        set_step_limit(step_limit)
    st = rt.stream_ptr(stream)
    pack = torch.empty((1 + k,) + (shape or (1,)), dtype=dtype, device="cuda")
    pd = rt.tensor_desc(pack)
    arr = rt.desc_array(_descs(vals, dtype_c))
    try:
        rt.check(rt.load_library().sg_ew_pack(ctx, kern, k, arr, ctypes.byref(pd), st),
                 "fused_map_with_partials")
        _raise_eval(lo, ctx, st)
    finally:
        if step_limit != DEFAULT_STEP_LIMIT:
            set_step_limit(DEFAULT_STEP_LIMIT)
    if not shape:
        rows = pack.reshape(-1).tolist()
        return rows[0], rows[1:]
    return pack[0], [pack[1 + i] for i in range(k)]


def fused_map_grad(module, name: str, args, ybar, *, want_primal: bool = False,
                   check: bool = True, stream=None, outs=None):
    """Fused adjoint (K2): cotangent of every argument in one pass.

    Returns ``(primal_or_None, cotangents)``.  Tensor arguments get a
    tensor cotangent of their own shape (``reduce_to`` of the broadcast,
    ``tensor.py:327-345``); scalar arguments get a one-element tensor
    (call ``float()`` on it; kept on the device to avoid a sync).
    """
    import torch

    fn = module.get(name)
    check_scalar_fn(fn)
    lo = lowered_for(module, name)
    vals, dtype = _intake(args, None if not isinstance(ybar, torch.Tensor) else ybar.dtype)
    shape = _broadcast(vals)
    yb = _as_device(ybar, dtype)
    if tuple(yb.shape) != shape:
        raise ValueError(f"ybar shape {tuple(yb.shape)} != result shape {shape}")
    dtype_c = rt.dtype_code(dtype)
    kern = kernel_for(lo, dtype_c)
    ctx = rt.context()
    st = rt.stream_ptr(stream)
    if outs is None:
        outs = [torch.empty((1,) if isinstance(v, float) else tuple(v.shape), dtype=dtype,
                            device="cuda") for v in vals]
    y = torch.empty(shape, dtype=dtype, device="cuda") if want_primal else None
    bars = rt.desc_array([rt.tensor_desc(o) for o in outs])
    yd = rt.tensor_desc(y) if y is not None else None
    arr = rt.desc_array(_descs(vals, dtype_c))
    ybd = rt.tensor_desc(yb)
    rt.check(rt.load_library().sg_ew_grad(ctx, kern, len(vals), arr, ctypes.byref(ybd),
                                          ctypes.byref(yd) if yd is not None else None, bars, st),
             "fused_map_grad")
    if check:
        _raise_eval(lo, ctx, st)
    return y, tuple(outs)


def reduce_to(x, shape, *, out=None, stream=None):
    """``tensor.reduce_to`` (tensor.py:327-345) on the device: sum the
    broadcast-expanded axes of ``x`` down to ``shape`` (``()`` -> float)."""
    import torch

    xd = _as_device(x)
    shape = tuple(shape)
    if out is None:
        out = torch.empty(shape or (1,), dtype=xd.dtype, device="cuda")
    od = rt.tensor_desc(out)
    if not shape:
        od.ndim = 0
    ad = rt.tensor_desc(xd)
    rt.check(rt.load_library().sg_reduce_to(rt.context(), ctypes.byref(ad), None, ctypes.byref(od),
                                            rt.stream_ptr(stream)), "reduce_to")
    return float(out.item()) if not shape else out


def fused_map_pullback(partials, arg_types, ybar):
    """``reduce_like(ybar * partial_i, type_i)`` -- reference forward_ad.py:226-235."""
    import torch

    yb = _as_device(ybar)
    out = []
    lib = rt.load_library()
    ctx = rt.context()
    st = rt.stream_ptr()
    for part, ty in zip(partials, arg_types):
        p = _as_device(part, yb.dtype)
        if kind_of(ty) == "f64":
            o = torch.empty((1,), dtype=yb.dtype, device="cuda")
            od = rt.tensor_desc(o)
            od.ndim = 0
        else:
            o = torch.empty(tuple(ty.shape), dtype=yb.dtype, device="cuda")
            od = rt.tensor_desc(o)
        ad, bd = rt.tensor_desc(yb), rt.tensor_desc(p)
        rt.check(lib.sg_reduce_to(ctx, ctypes.byref(ad), ctypes.byref(bd), ctypes.byref(od), st),
                 "fused_map_pullback")
        out.append(float(o.item()) if kind_of(ty) == "f64" else o)
    return tuple(out)
