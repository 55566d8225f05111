"""Oracle for ``fused_map`` / ``fused_pack`` -- TEST INFRASTRUCTURE ONLY.

Two restatements of the reference's per-element semantics:

* :func:`eval_scalar` / :func:`eval_dual` -- a pure-Python block walker
  over the IR, restating ``interp.run_blocks`` (interp.py:95-138) with the
  scalar branch of ``Machine.dispatch`` (interp.py:194-269) and the dual
  rules of ``_DualRunner.dispatch`` (forward_ad.py:56-149).  Exact for any
  control flow; used for small cases.
* :func:`vec_eval` -- the same rules evaluated once over whole numpy
  arrays, for straight-line sub-functions (every element takes the same
  path), used at sizes the Python loop cannot reach.  Every ufunc here is
  correctly rounded for + - * /, and ``np.exp``/``np.tanh``/``np.log`` are
  within an ulp of ``math.*``.

Both compute in float64 (reference ``tensor.py:39``).
"""

from __future__ import annotations

import math

import numpy as np


class OracleEvalError(Exception):
    """Same fields as the reference ``interp.EvalError`` (interp.py:26-35)."""

    def __init__(self, function, block, index, message):
        self.function, self.block, self.index, self.message = function, block, index, message
        super().__init__(f"@{function} ^{block} instr {index}: {message}")


class _Domain(Exception):
    pass


def _kind(ty):
    return getattr(ty, "kind", str(ty))


def _sigmoid(x):  # tensor.py:214-215
    return 1.0 / (1.0 + math.exp(-x))


def _pow_int(x, n):  # tensor.py:222-227, left-to-right repeated multiply
    acc = 1.0
    for _ in range(n):
        acc = acc * x
    return acc


def _log(x):  # tensor.py:230-233
    if x <= 0.0:
        raise _Domain(f"log of non-positive value {x!r}")
    return math.log(x)


def _run(module, fn, args, step, budget):
    """Block walker: interp.run_blocks (interp.py:95-138)."""
    blocks = {b.name: b for b in fn.blocks}
    env = {}
    cur = fn.blocks[0]
    binds = tuple(args)
    while True:
        for (vid, _), v in zip(cur.params, binds):
            env[vid] = v
        for i, ins in enumerate(cur.body):
            budget[0] -= 1
            if budget[0] < 0:
                raise OracleEvalError(fn.name, cur.name, i, "step limit exhausted")
            try:
                env[ins.result] = step(ins, env, budget)
            except _Domain as e:
                raise OracleEvalError(fn.name, cur.name, i, str(e)) from None
        budget[0] -= 1
        if budget[0] < 0:
            raise OracleEvalError(fn.name, cur.name, len(cur.body), "step limit exhausted")
        t = cur.term
        if hasattr(t, "values"):
            return tuple(env[v] for v in t.values)
        if hasattr(t, "then_target"):
            if env[t.cond]:
                cur, binds = blocks[t.then_target], tuple(env[a] for a in t.then_args)
            else:
                cur, binds = blocks[t.else_target], tuple(env[a] for a in t.else_args)
        else:
            cur, binds = blocks[t.target], tuple(env[a] for a in t.args)


def eval_scalar(module, name, args, budget=None):
    """Primal value of a scalar function at one point (interp.py:190-269)."""
    budget = budget if budget is not None else [2_000_000]

    def step(ins, env, budget):
        op, a = ins.op, ins.operands
        if op == "const":
            k = _kind(ins.attrs["ty"])
            v = ins.attrs["value"]
            return float(v) if k == "f64" else (int(v) if k == "i64" else bool(v))
        if op in ("add", "sub", "mul", "div"):
            x, y = env[a[0]], env[a[1]]
            if op == "div":
                if y == 0.0:
                    raise _Domain("division by zero")
                return x / y
            return x + y if op == "add" else (x - y if op == "sub" else x * y)
        if op == "neg":
            return -env[a[0]]
        if op == "exp":
            return math.exp(env[a[0]])
        if op == "log":
            return _log(env[a[0]])
        if op == "tanh":
            return math.tanh(env[a[0]])
        if op == "sigmoid":
            return _sigmoid(env[a[0]])
        if op == "relu":
            x = env[a[0]]
            return x if x > 0.0 else 0.0
        if op == "pow_int":
            return _pow_int(env[a[0]], ins.attrs["n"])
        if op == "itof":
            return float(env[a[0]])
        if op in ("lt", "gt", "eq"):
            x, y = env[a[0]], env[a[1]]
            return x < y if op == "lt" else (x > y if op == "gt" else x == y)
        if op == "select":
            return env[a[1]] if env[a[0]] else env[a[2]]
        if op == "call":
            callee = module.get(ins.attrs["fn"].name)
            return _run(module, callee, tuple(env[o] for o in a), step, budget)[0]
        raise _Domain(f"op '{op}' has no scalar evaluation rule")

    return _run(module, module.get(name), tuple(args), step, budget)[0]


class Dual:
    __slots__ = ("p", "t")

    def __init__(self, p, t):
        self.p, self.t = p, t


def eval_dual(module, name, args, budget=None):
    """[primal, d/d arg_0, ...] at one point: pack_rows (forward_ad.py:178-191)."""
    budget = budget if budget is not None else [2_000_000]
    k = len(args)

    def lift(v):
        return v if isinstance(v, Dual) else Dual(float(v), (0.0,) * k)

    def step(ins, env, budget):
        op, a = ins.op, ins.operands
        if op == "const":
            kd = _kind(ins.attrs["ty"])
            v = ins.attrs["value"]
            if kd == "f64":
                return Dual(float(v), (0.0,) * k)
            return int(v) if kd == "i64" else bool(v)
        if op in ("add", "sub", "mul"):
            x, y = env[a[0]], env[a[1]]
            if isinstance(x, int) and isinstance(y, int) and not isinstance(x, bool):
                return x + y if op == "add" else (x - y if op == "sub" else x * y)
            x, y = lift(x), lift(y)
            if op == "add":
                return Dual(x.p + y.p, tuple(s + t for s, t in zip(x.t, y.t)))
            if op == "sub":
                return Dual(x.p - y.p, tuple(s - t for s, t in zip(x.t, y.t)))
            return Dual(x.p * y.p, tuple(s * y.p + x.p * t for s, t in zip(x.t, y.t)))
        if op == "div":  # forward_ad.py:83-88
            x, y = lift(env[a[0]]), lift(env[a[1]])
            if y.p == 0.0:
                raise _Domain("division by zero")
            p = x.p / y.p
            return Dual(p, tuple((s - p * t) / y.p for s, t in zip(x.t, y.t)))
        if op == "neg":
            x = env[a[0]]
            return -x if isinstance(x, int) else Dual(-x.p, tuple(-t for t in x.t))
        if op == "exp":
            x = env[a[0]]
            y = math.exp(x.p)
            return Dual(y, tuple(y * t for t in x.t))
        if op == "log":
            x = env[a[0]]
            return Dual(_log(x.p), tuple(t / x.p for t in x.t))
        if op == "tanh":
            x = env[a[0]]
            y = math.tanh(x.p)
            d = 1.0 - y * y
            return Dual(y, tuple(d * t for t in x.t))
        if op == "sigmoid":
            x = env[a[0]]
            y = _sigmoid(x.p)
            d = y * (1.0 - y)
            return Dual(y, tuple(d * t for t in x.t))
        if op == "relu":  # derivative at exactly zero is zero (forward_ad.py:114-118)
            x = env[a[0]]
            d = 1.0 if x.p > 0.0 else 0.0
            return Dual(x.p if x.p > 0.0 else 0.0, tuple(d * t for t in x.t))
        if op == "pow_int":
            x = env[a[0]]
            n = ins.attrs["n"]
            y = _pow_int(x.p, n)
            if n == 0:
                return Dual(y, (0.0,) * k)
            d = float(n) * _pow_int(x.p, n - 1)
            return Dual(y, tuple(d * t for t in x.t))
        if op == "itof":
            return Dual(float(env[a[0]]), (0.0,) * k)
        if op in ("lt", "gt", "eq"):
            x, y = env[a[0]], env[a[1]]
            x = x.p if isinstance(x, Dual) else x
            y = y.p if isinstance(y, Dual) else y
            return x < y if op == "lt" else (x > y if op == "gt" else x == y)
        if op == "select":
            return env[a[1]] if env[a[0]] else env[a[2]]
        if op == "call":
            callee = module.get(ins.attrs["fn"].name)
            return _run(module, callee, tuple(env[o] for o in a), step, budget)[0]
        raise _Domain(f"op '{op}' is not scalar; forward mode runs scalar code only")

    seeded = tuple(Dual(float(v), tuple(1.0 if j == i else 0.0 for j in range(k)))
                   for i, v in enumerate(args))
    out = lift(_run(module, module.get(name), seeded, step, budget)[0])
    return [out.p, *out.t]


# ----------------------------------------------------------- broadcasting

def broadcast_shapes(*shapes):
    """tensor.py:108-121 (trailing alignment)."""
    out = ()
    for s in shapes:
        n = max(len(out), len(s))
        r = []
        for i in range(1, n + 1):
            a = out[-i] if i <= len(out) else 1
            b = s[-i] if i <= len(s) else 1
            if a != b and a != 1 and b != 1:
                raise ValueError(f"shapes {out} and {s} do not broadcast")
            r.append(max(a, b))
        out = tuple(reversed(r))
    return out


def reduce_to(x: np.ndarray, shape: tuple):
    """tensor.py:327-345: fold extra leading axes, then extent-1 axes, ascending."""
    arr = np.asarray(x, dtype=np.float64)
    while arr.ndim > len(shape) and arr.ndim > 1:
        arr = _fold(arr, 0)
    if not shape:
        return float(np.cumsum(arr.reshape(-1))[-1]) if arr.size > 1 else float(arr.reshape(-1)[0])
    for ax in range(len(shape)):
        if shape[ax] == 1 and arr.shape[ax] != 1:
            arr = np.expand_dims(_fold(arr, ax), ax)
    return arr


def _fold(arr, axis):  # tensor.py:287-292
    if arr.shape[axis] == 1:
        return arr.take(0, axis=axis)
    return np.cumsum(arr, axis=axis).take(-1, axis=axis)


def fused_map_with_partials(module, name, args):
    """Per-element restatement of forward_ad.py:194-223 (small inputs)."""
    k = len(args)
    shapes = [np.shape(a) for a in args if isinstance(a, np.ndarray)]
    shape = broadcast_shapes(*shapes) if shapes else ()
    if not shape:
        rows = eval_dual(module, name, [float(a) for a in args])
        return rows[0], rows[1:]
    flat = [np.broadcast_to(a, shape).reshape(-1) if isinstance(a, np.ndarray)
            else np.full(int(np.prod(shape)), float(a)) for a in args]
    budget = [2_000_000_000]
    cols = [eval_dual(module, name, [float(f[i]) for f in flat], budget)
            for i in range(flat[0].size)]
    cols = np.array(cols, dtype=np.float64).T
    return cols[0].reshape(shape), [cols[1 + i].reshape(shape) for i in range(k)]


def fused_map_pullback(partials, arg_types_shapes, ybar):
    """forward_ad.py:226-235 with reduce_like (rules.py:302-311)."""
    out = []
    for part, shp in zip(partials, arg_types_shapes):
        prod = np.asarray(ybar, dtype=np.float64) * np.asarray(part, dtype=np.float64)
        if shp is None:  # f64 operand: full fold (reduce_sum "all", tensor.py:303-307)
            arr = prod
            while arr.ndim > 1:
                arr = _fold(arr, 0)
            out.append(float(np.cumsum(arr)[-1]) if arr.size > 1 else float(arr[0]))
        elif tuple(prod.shape) == tuple(shp):
            out.append(prod)
        else:
            out.append(reduce_to(prod, tuple(shp)))
    return tuple(out)


# ------------------------------------------------------ vectorised (numpy)

def vec_eval(module, name, args, dual=True):
    """Evaluate a straight-line scalar function over broadcast arrays.

    Returns (primal, [partials]) (or the primal alone with dual=False).
    Raises OracleEvalError naming the first failing element's site.
    """
    fn = module.get(name)
    if len(fn.blocks) != 1:
        raise ValueError("vec_eval handles straight-line functions only")
    k = len(args)
    arrs = [np.asarray(a, dtype=np.float64) if isinstance(a, np.ndarray) else float(a) for a in args]
    shape = broadcast_shapes(*[a.shape for a in arrs if isinstance(a, np.ndarray)])
    env = {}
    for i, (vid, _) in enumerate(fn.params):
        p = np.broadcast_to(arrs[i], shape) if isinstance(arrs[i], np.ndarray) else np.full(shape, arrs[i])
        t = [np.full(shape, 1.0 if j == i else 0.0) for j in range(k)] if dual else None
        env[vid] = (p, t)
    blk = fn.blocks[0]

    def zeros():
        return [np.zeros(shape) for _ in range(k)] if dual else None

    for idx, ins in enumerate(blk.body):
        op, a = ins.op, ins.operands
        if op == "const":
            env[ins.result] = (np.full(shape, float(ins.attrs["value"])), zeros())
            continue
        x = env[a[0]] if a else None
        y = env[a[1]] if len(a) > 1 else None
        if op in ("add", "sub"):
            s = 1.0 if op == "add" else -1.0
            p = x[0] + y[0] if op == "add" else x[0] - y[0]
            t = [xt + s * yt if op == "add" else xt - yt for xt, yt in zip(x[1], y[1])] if dual else None
        elif op == "mul":
            p = x[0] * y[0]
            t = [xt * y[0] + x[0] * yt for xt, yt in zip(x[1], y[1])] if dual else None
        elif op == "div":
            bad = y[0] == 0.0
            if bad.any():
                raise OracleEvalError(name, blk.name, idx, f"division by zero at element {int(np.argmax(bad.reshape(-1)))}")
            p = x[0] / y[0]
            t = [(xt - p * yt) / y[0] for xt, yt in zip(x[1], y[1])] if dual else None
        elif op == "neg":
            p = -x[0]
            t = [-xt for xt in x[1]] if dual else None
        elif op == "exp":
            p = np.exp(x[0])
            t = [p * xt for xt in x[1]] if dual else None
        elif op == "log":
            bad = x[0] <= 0.0
            if bad.any():
                raise OracleEvalError(name, blk.name, idx, f"log of non-positive value at element {int(np.argmax(bad.reshape(-1)))}")
            p = np.log(x[0])
            t = [xt / x[0] for xt in x[1]] if dual else None
        elif op == "tanh":
            p = np.tanh(x[0])
            d = 1.0 - p * p
            t = [d * xt for xt in x[1]] if dual else None
        elif op == "sigmoid":
            p = 1.0 / (1.0 + np.exp(-x[0]))
            d = p * (1.0 - p)
            t = [d * xt for xt in x[1]] if dual else None
        elif op == "relu":
            d = (x[0] > 0.0).astype(np.float64)
            p = np.where(x[0] > 0.0, x[0], 0.0)
            t = [d * xt for xt in x[1]] if dual else None
        elif op == "pow_int":
            n = ins.attrs["n"]
            acc = np.ones(shape)
            for _ in range(n):
                acc = acc * x[0]
            p = acc
            if n == 0:
                t = zeros()
            else:
                acc2 = np.ones(shape)
                for _ in range(n - 1):
                    acc2 = acc2 * x[0]
                d = float(n) * acc2
                t = [d * xt for xt in x[1]] if dual else None
        elif op in ("lt", "gt", "eq"):  # compare primals -> per-element bool
            f = {"lt": np.less, "gt": np.greater, "eq": np.equal}[op]
            p, t = f(x[0], y[0]), None
        elif op == "select":  # bool condition picks the whole dual
            c, u, v = env[a[0]][0], env[a[1]], env[a[2]]
            p = np.where(c, u[0], v[0])
            t = [np.where(c, ut, vt) for ut, vt in zip(u[1], v[1])] if dual else None
        else:
            raise ValueError(f"vec_eval: op '{op}' not supported")
        env[ins.result] = (p, t)
    res = env[blk.term.values[0]]
    if not dual:
        return res[0]
    return res[0], res[1]
