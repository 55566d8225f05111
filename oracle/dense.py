"""Oracle for the Dense layer, losses and the SGD step -- TEST INFRASTRUCTURE ONLY.

Restates the IR the reference emits for a Dense layer
(``nn_train._batch_trunk`` / ``_batch_head``, nn_train.py:189-210):

    wt = transpose(W); z = matmul(h, wt); zb = add(z, b); h' = act(zb)

and its pullback through the reference adjoint rules (rules.py):
``_sigmoid`` ybar*(y*(1-y)) (rules.py:87-89), ``_tanh`` ybar*(1-y*y)
(rules.py:82-84), ``_add`` reduce_like -> column sums (rules.py:45-46,
tensor.py:327-345), ``_matmul`` (ybar . v^T, a^T . ybar) (rules.py:113-115),
``_transpose`` (rules.py:123-124).

Two arithmetic modes:

* ``exact`` -- the reference's own order: ascending-k products rounded
  separately (tensor.py:351-361) via the C restatement in
  ``csrc/strict_gemm.c``; bit-identical to the reference in float64 and
  the strict-fp32 GEMM contract in float32;
* ``blas`` -- numpy/OpenBLAS fp64 (reassociated), for full-size tolerance
  checks and as the multi-threaded "best CPU" line.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            subprocess.run(["make", "-s"], cwd=_HERE, check=True)
        lib = ctypes.CDLL(_LIB)
        for name in ("oracle_gemm_f32", "oracle_gemm_f64"):
            f = getattr(lib, name)
            f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_long] * 3
            f.restype = None
        _lib = lib
    return _lib


def matmul_exact(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Ascending-k, no-FMA product in the inputs' dtype (tensor.py:351-361)."""
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ValueError(f"matmul shapes {a.shape} x {b.shape}")
    dt = np.float32 if (a.dtype == np.float32 and b.dtype == np.float32) else np.float64
    a = np.ascontiguousarray(a, dtype=dt)
    b = np.ascontiguousarray(b, dtype=dt)
    c = np.empty((a.shape[0], b.shape[1]), dtype=dt)
    fn = _load().oracle_gemm_f32 if dt == np.float32 else _load().oracle_gemm_f64
    fn(a.ctypes.data, b.ctypes.data, c.ctypes.data, a.shape[0], a.shape[1], b.shape[1])
    return c


def matmul_cumsum(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """The reference kernel's own formulation (products, cumsum over k), row-chunked."""
    out = np.empty((a.shape[0], b.shape[1]), dtype=np.result_type(a, b))
    rows = max(1, int(2 ** 24 // max(1, a.shape[1] * b.shape[1])))
    for i in range(0, a.shape[0], rows):
        prod = a[i:i + rows, :, None] * b[None, :, :]
        out[i:i + rows] = prod[:, 0, :] if a.shape[1] == 1 else np.cumsum(prod, axis=1)[:, -1, :]
    return out


def colsum_exact(x: np.ndarray) -> np.ndarray:
    """reduce_to((B, n) -> (n,)): sequential fold over rows (tensor.py:337-338)."""
    if x.shape[0] == 1:
        return x[0].copy()
    return np.cumsum(x, axis=0)[-1]


def act_fwd(z: np.ndarray, act: str) -> np.ndarray:
    if act == "sigmoid":
        return 1.0 / (1.0 + np.exp(-z))
    if act == "tanh":
        return np.tanh(z)
    if act == "relu":
        return np.where(z > 0.0, z, 0.0)
    if act == "identity":
        return z
    raise ValueError(act)


def act_bwd(ybar: np.ndarray, y: np.ndarray, z: np.ndarray, act: str) -> np.ndarray:
    """Adjoint rules with the reference's operation order."""
    if act == "sigmoid":  # rules.py:87-89 mul(ybar, mul(y, sub(1, y)))
        return ybar * (y * (1.0 - y))
    if act == "tanh":  # rules.py:82-84 mul(ybar, sub(1, mul(y, y)))
        return ybar * (1.0 - y * y)
    if act == "relu":  # rules.py:92-94 mul(ybar, gt_zero_mask(a))
        return ybar * (z > 0.0).astype(ybar.dtype)
    if act == "identity":
        return ybar
    raise ValueError(act)


def dense_forward(x, W, b, act, mode="blas"):
    """Returns (z+b, h) for h = act(x . W^T + b)."""
    if mode == "exact":
        z = matmul_exact(x, np.ascontiguousarray(W.T))
    else:
        z = x @ W.T
    zb = z + b
    return zb, act_fwd(zb, act)


def dense_backward(hbar, x, W, zb, h, act, mode="blas", need_dx=True):
    """(dx, dW, db) of one Dense layer given the cotangent of its output."""
    dz = act_bwd(hbar, h, zb, act)
    db = colsum_exact(dz)
    if mode == "exact":
        dx = matmul_exact(dz, W) if need_dx else None
        dWt = matmul_exact(np.ascontiguousarray(x.T), dz)
        dW = np.ascontiguousarray(dWt.T)
    else:
        dx = dz @ W if need_dx else None
        dW = dz.T @ x
    return dx, dW, db


# ----------------------------------------------------------------- losses

def softmax_xent(z: np.ndarray, Y: np.ndarray):
    """Loss IR of SURVEY §8(d) c1: e=exp(z); s=rowsum(e); p=e/s;
    loss = reduce_sum(Y*log p, all) * (-1/n).  Returns (loss, dL/dz)."""
    n = z.shape[0]
    e = np.exp(z)
    s = np.cumsum(e, axis=1)[:, -1:]
    p = e / s
    t = Y * np.log(p)
    tot = float(np.cumsum(np.cumsum(t, axis=0)[-1])[-1])
    loss = tot * (-1.0 / n)
    dz = (p * Y.sum(axis=1, keepdims=True) - Y) * (1.0 / n)
    return loss, dz


def mse(z: np.ndarray, Y: np.ndarray):
    """loss = reduce_sum((z-Y)^2, all) * (1/n); dL/dz = 2 (z-Y) / n."""
    n = z.shape[0]
    d = z - Y
    tot = float(np.cumsum(np.cumsum(d * d, axis=0)[-1])[-1])
    return tot * (1.0 / n), (d * (1.0 / n)) + (d * (1.0 / n))


BCE_LO, BCE_HI = 1e-7, 1.0 - 1e-7


def bce(z: np.ndarray, Y: np.ndarray):
    """One-logit head + clamped mean BCE: ``_batch_head``'s reshape/sigmoid
    (nn_train.py:209-210) then ``_bce_mean`` (nn_train.py:213-227):
    p = sigmoid(z); p2 = clamp via lt/select, gt/select into [1e-7, 1-1e-7];
    loss = reduce_sum(y log p2 + (1-y) log(1-p2), all) * (-1/n).
    Gradient in the pullback's order (rules.py:53-58 mul, :77-79 log,
    select passes the cotangent only where the prediction was kept,
    :87-89 sigmoid).  z, Y: (n, 1).  Returns (loss, dL/dz (n, 1))."""
    n = z.shape[0]
    zf = z.reshape(n)
    y = Y.reshape(n)
    p = 1.0 / (1.0 + np.exp(-zf))
    under = p < BCE_LO
    p1 = np.where(under, BCE_LO, p)
    over = p1 > BCE_HI
    p2 = np.where(over, BCE_HI, p1)
    yn = 1.0 - y
    pn = 1.0 - p2
    s = y * np.log(p2) + yn * np.log(pn)
    loss = float(np.cumsum(s)[-1]) * (-1.0 / n)
    g = np.full(n, -1.0 / n)
    p2bar = -((g * yn) / pn) + (g * y) / p2
    pbar = np.where(under | over, 0.0, p2bar)
    dz = pbar * (p * (1.0 - p))
    return loss, dz.reshape(n, 1)


LOSS_FNS = {"softmax_xent": softmax_xent, "mse": mse, "bce": bce}


class DomainError(ValueError):
    """The reference's DomainError (tensor.py:25-26)."""


def _exp_checked(x: float) -> float:
    return math.exp(x)  # OverflowError("math range error") exactly as the reference's unary_math


def check_domain(params, X, Y, acts, loss="softmax_xent"):
    """Restates where the reference's float64 evaluation of a Dense chain's
    loss IR raises (the conditions the device kernels flag, SG_DOM_*):

    * ``sigmoid`` activations / the BCE head: ``scalar_sigmoid`` calls
      ``math.exp(-z)`` per element (tensor.py:214-215, 245-250) ->
      OverflowError, uncaught by run_blocks;
    * softmax cross-entropy (the c1 loss IR): ``exp`` per element
      (OverflowError), ``div`` by a zero row sum (tensor.py:197-205) and
      ``log`` of p <= 0 (tensor.py:230-233) -> DomainError, in that op order.

    Raises what the reference raises (DomainError here; run_blocks wraps it
    into EvalError, interp.py:117-119); returns None otherwise."""
    h = np.asarray(X, dtype=np.float64)
    for (W, b), act in zip(params, acts):
        zb = h @ np.asarray(W, dtype=np.float64).T + np.asarray(b, dtype=np.float64)
        if act == "sigmoid":
            for v in zb.reshape(-1):
                _exp_checked(-float(v))
        h = act_fwd(zb, act)
    if loss == "bce":
        for v in h.reshape(-1):
            _exp_checked(-float(v))
    elif loss == "softmax_xent":
        e = np.array([[_exp_checked(float(v)) for v in row] for row in h])
        s = np.cumsum(e, axis=1)[:, -1:]
        if bool((s == 0.0).any()):
            raise DomainError("division by zero")
        with np.errstate(over="ignore", divide="ignore", invalid="ignore"):
            p = e / s
        for v in p.reshape(-1):
            if v <= 0.0:
                raise DomainError(f"log of non-positive value {float(v)!r}")


def mlp_step(params, X, Y, acts, loss="softmax_xent", lr=0.05, mode="blas"):
    """One training step of a Dense chain: forward, loss, pullback, SGD.

    params = [(W, b), ...]; returns (loss, grads[(dW, db)], new_params).
    """
    hs = [X]
    zs = []
    for (W, b), act in zip(params, acts):
        zb, h = dense_forward(hs[-1], W, b, act, mode)
        zs.append(zb)
        hs.append(h)
    lv, gbar = LOSS_FNS[loss](hs[-1], Y)
    grads = [None] * len(params)
    for l in range(len(params) - 1, -1, -1):
        W, b = params[l]
        dx, dW, db = dense_backward(gbar, hs[l], W, zs[l], hs[l + 1], acts[l], mode, need_dx=l > 0)
        grads[l] = (dW, db)
        gbar = dx
    new = [(W - lr * dW, b - lr * db) for (W, b), (dW, db) in zip(params, grads)]
    return lv, grads, new
