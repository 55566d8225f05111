"""Training step driver: single GPU, CUDA graphs, and minibatch data parallelism.

Reference step: ``dan_step`` (nn_train.py:337-375) -- one augmented forward,
pullback(s), then ``p - lr * g`` over the flat parameter list.  The
reference is single-process; data parallelism is the build's
addition: the minibatch rows are sharded over ranks, each
shard's loss is scaled by the *global* 1/B (the reference's mean scale,
nn_train.py:226), and an all-reduce SUM of the flat gradient buffer
reproduces the single-GPU gradient up to summation order.  Buckets are
one layer each, launched (async, NCCL over NVLink/NVSwitch) as soon as
that layer's dW/db are enqueued, so they overlap the rest of the pullback.
"""

from __future__ import annotations

import numpy as np

from .dense import Chain, ChainEngine
from .tape import Tape


class DataParallel:
    """Bucketed, overlapped all-reduce of a flat gradient buffer.

    ``G`` is the flat gradient tensor and ``buckets`` a list of
    ``(lo, hi)`` slices (one per layer, in parameter order).  ``ready(i)``
    is called when bucket i is final on the compute stream; ``finish()``
    makes the compute stream wait for every reduction.
    """

    def __init__(self, G, buckets, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.G = G
        self.buckets = list(buckets)
        self.group = group
        self.world = dist.get_world_size(group)
        self.works = []

    def ready(self, i: int) -> None:
        lo, hi = self.buckets[i]
        w = self.dist.all_reduce(self.G[lo:hi], op=self.dist.ReduceOp.SUM, group=self.group,
                                 async_op=True)
        self.works.append(w)

    def finish(self) -> None:
        for w in self.works:
            w.wait()
        self.works.clear()

    def broadcast_params(self, P, src: int = 0) -> None:
        self.dist.broadcast(P, src=src, group=self.group)


class Trainer:
    """Dense-chain training on one GPU, optionally data-parallel over a process group.

    ``batch`` is the GLOBAL minibatch; with ``dp`` each rank holds
    ``batch / world`` rows (weak per-rank work shrinks, strong scaling of
    the global step).
    """

    def __init__(self, chain: Chain, batch: int, loss: str = "mse", lr: float = 0.05,
                 precision: str = "bf16", dp: bool = False, group=None, graph: bool = False):
        self.lr = float(lr)
        self.world = 1
        if dp:
            import torch.distributed as dist

            self.world = dist.get_world_size(group)
        if batch % self.world:
            raise ValueError(f"global batch {batch} not divisible by {self.world} ranks")
        self.local_batch = batch // self.world
        self.engine = ChainEngine(chain, self.local_batch, loss, precision, global_batch=batch)
        self.dp = None
        if dp:
            self.dp = DataParallel(self.engine.G, self.engine.bucket_bounds, group)
            self.engine.grad_ready = self.dp.ready
            self.dp.broadcast_params(self.engine.P)
            if self.engine.S is not None:
                self.engine.S.copy_(self.engine.P.to(self.engine.S.dtype))
        self.graph = None
        self.use_graph = graph and self.dp is None
        self._eager_steps = 0

    def _device_step(self):
        e = self.engine
        e.forward()
        e.loss_and_seed()
        e.pullback()
        if self.dp is not None:
            self.dp.finish()
        e.sgd(self.lr)

    def step(self, X, Y):
        """One training step on (X, Y) already on the device; returns the loss (device)."""
        self.engine.load_batch(X, Y)
        if self.use_graph and self._eager_steps > 0:
            # the first step ran eagerly (one-time kernel attribute setup);
            # capture once without warm-up so no extra update is applied
            if self.graph is None:
                self.graph = Tape.capture(self._device_step, warmup=0)
            self.graph.replay()
        else:
            self._device_step()
            self._eager_steps += 1
        return self.engine.loss

    def gradient(self, X, Y):
        """Loss and parameter gradients without the update (the pullback API)."""
        e = self.engine
        e.load_batch(X, Y)
        e.forward()
        e.loss_and_seed()
        e.pullback()
        if self.dp is not None:
            self.dp.finish()
        return float(e.loss.item()), e.get_grads()


def shard_rows(X: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Rows of the global minibatch owned by ``rank`` (contiguous blocks)."""
    n = X.shape[0] // world
    return X[rank * n:(rank + 1) * n]
