"""The two-headed DAN training step on the GPU.

Mirror of ``nn_train.dan_step`` / ``train`` (nn_train.py:337-375, 418-450):
one augmented forward of the minibatch loss, two pullback replays of the
same traces with seeds (1, 0) and (0, 1), and plain SGD on the summed
gradient.  The loss IR and its aug/pb pair are the reference's own
(built by ``build_loss_ir`` + ``augment``, or read back from their printed
text); every tensor op runs on the device through :class:`GpuMachine`, in
f64 with the reference's operation order, so results match the reference
to libm ulps (exp/tanh/log).
"""

from __future__ import annotations

import random

from .gpu_machine import GpuMachine
from .irtext import parse_ir

_SGD = parse_ir("""
func @sgd(%p: f64, %gc: f64, %gd: f64, %lr: f64) -> f64 {
^entry:
  %g = add %gc, %gd
  %s = mul %lr, %g
  %r = sub %p, %s
  ret %r
}
""")


def dan_step(module, loss_name: str, params: list, X, Yc, Yd, lam: float, lr: float,
             machine: GpuMachine | None = None):
    """One step: returns (new_params, c_loss, d_loss); params are device tensors
    in ``_weight_args`` order [W, b, W, b, ...] (nn_train.py:99-103)."""
    from . import fused as F

    m = machine or GpuMachine(module)
    out = m.call(loss_name + "__aug", tuple(params) + (X, Yc, Yd, float(lam)))
    c_loss, d_loss, blog, vstack = out
    g_c = m.call(loss_name + "__pb", (blog, vstack, 1.0, 0.0))
    g_d = m.call(loss_name + "__pb", (blog, vstack, 0.0, 1.0))
    # W - lr * (g_c + g_d): the update of nn_train.py:365-372, same operation order
    new = [F.fused_map(_SGD, "sgd", [p, gc, gd, float(lr)], dtype=m.dtype)
           for p, gc, gd in zip(params, g_c, g_d)]
    return new, c_loss, d_loss


def train_epochs(module, loss_name: str, params: list, X, Yc, Yd, *, lam: float, lr: float,
                 epochs: int, batch_size: int, seed: int, on_epoch=None):
    """The loop of ``nn_train.train`` (nn_train.py:418-450) without the
    host-side evaluation: shuffles with ``random.Random(seed + 2)``, steps
    through full minibatches, and calls ``on_epoch(epoch, params, c_mean,
    d_mean)`` after each epoch.  X, Yc, Yd are host arrays of the full set."""
    import numpy as np
    import torch

    m = GpuMachine(module)
    n = X.shape[0]
    order_rng = random.Random(seed + 2)
    nb = n // batch_size
    Xd = torch.as_tensor(np.asarray(X), dtype=torch.float64, device="cuda")
    Ycd = torch.as_tensor(np.asarray(Yc), dtype=torch.float64, device="cuda")
    Ydd = torch.as_tensor(np.asarray(Yd), dtype=torch.float64, device="cuda")
    for epoch in range(epochs):
        order = list(range(n))
        order_rng.shuffle(order)
        c_sum = d_sum = 0.0
        for k in range(nb):
            idx = torch.as_tensor(order[k * batch_size:(k + 1) * batch_size], device="cuda")
            params, c, d = dan_step(module, loss_name, params, Xd.index_select(0, idx).contiguous(),
                                    Ycd.index_select(0, idx).contiguous(),
                                    Ydd.index_select(0, idx).contiguous(), lam, lr, m)
            c_sum += c
            d_sum += d
        if on_epoch is not None:
            on_epoch(epoch, params, c_sum / nb, d_sum / nb)
    return params
