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

import collections
import ctypes

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


def nccl_unique_id(group=None) -> bytes:
    """Rank 0's 128-byte NCCL id (``sg_dp_unique_id``), broadcast to every
    rank of ``group`` over the host rendezvous (host-only: runs on gloo too)."""
    import torch.distributed as dist

    from . import runtime as rt

    lib = rt.load_library()
    lib.sg_dp_unique_id.argtypes = [ctypes.POINTER(ctypes.c_uint8), ctypes.c_size_t]
    uid = (ctypes.c_uint8 * 128)()
    if dist.get_rank(group) == 0:
        rt.check(lib.sg_dp_unique_id(uid, 128), "sg_dp_unique_id")
    box = [bytes(uid)]
    src = 0 if group is None else dist.get_global_rank(group, 0)
    dist.broadcast_object_list(box, src=src, group=group)
    return box[0]


class NcclDataParallel:
    """The same bucketed all-reduce through the library's own NCCL
    communicator (``sg_dp_*``, include/sgb200.h): each bucket forks from the
    compute stream onto the communicator's stream and ``finish`` joins it
    back, all stream-ordered -- so a data-parallel step, collectives
    included, can be captured in one CUDA graph.  ``torch.distributed`` is
    only the rendezvous (the 128-byte NCCL id from rank 0) and the one-time
    parameter broadcast.
    """

    def __init__(self, G, buckets, group=None):
        import torch.distributed as dist

        from . import runtime as rt

        self.dist, self.rt = dist, rt
        self.G = G
        self.buckets = list(buckets)
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        lib = rt.load_library()
        P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        U8 = ctypes.POINTER(ctypes.c_uint8)
        lib.sg_dp_unique_id.argtypes = [U8, SZ]
        lib.sg_dp_init.argtypes = [P, U8, SZ, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)]
        lib.sg_dp_allreduce.argtypes = [P, P, I64, I32, P]
        lib.sg_dp_wait.argtypes = [P, P]
        lib.sg_dp_finalize.argtypes = [P]
        self.lib = lib
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_unique_id(group))
        h = ctypes.c_void_p()
        rt.check(lib.sg_dp_init(rt.context(), uid, 128, self.rank, self.world, ctypes.byref(h)), "sg_dp_init")
        self.handle = h
        self.dtype = rt.dtype_code(G.dtype)

    def ready(self, i: int) -> None:
        lo, hi = self.buckets[i]
        self.rt.check(self.lib.sg_dp_allreduce(self.handle, self.G[lo:hi].data_ptr(), hi - lo, self.dtype,
                                               self.rt.stream_ptr()), "sg_dp_allreduce")

    def finish(self) -> None:
        self.rt.check(self.lib.sg_dp_wait(self.handle, self.rt.stream_ptr()), "sg_dp_wait")

    def broadcast_params(self, P, src: int = 0) -> None:
        self.dist.broadcast(P, src=src, group=self.group)

    def close(self) -> None:
        if self.handle:
            self.lib.sg_dp_finalize(self.handle)
            self.handle = None


def _default_dp_backend(group) -> str:
    import torch.distributed as dist

    from . import runtime as rt

    if dist.get_backend(group) != "nccl":
        return "torch"
    try:
        return "sg" if rt.load_library().sg_dp_available() else "torch"
    except rt.RuntimeUnavailable:
        return "torch"


class Trainer:
    """Dense-chain training on one GPU, optionally data-parallel over a process group.

    ``batch`` is the GLOBAL minibatch; with ``dp`` each rank holds
    ``batch / world`` rows (weak per-rank work shrinks, strong scaling of
    the global step).  ``dp_backend``: "sg" (the library's NCCL
    communicator, default under an NCCL process group; CUDA-graph capturable)
    or "torch" (``torch.distributed`` async all-reduce; the gloo CPU path).
    """

    MAX_GRAPHS = 4

    @property
    def compute_precision(self) -> str:
        """What the step computes in (``ChainEngine.compute_precision``): a
        c1-sized chain runs its one-launch step in fp32 whatever the request."""
        return self.engine.compute_precision

    def __init__(self, chain: Chain, batch: int, loss: str = "mse", lr: float = 0.05,
                 precision: str = "bf16", dp: bool = False, group=None, graph: bool = False,
                 dp_backend: str | None = None, small: bool = True):
        self.lr = float(lr)
        self.world = 1
        if dp:
            import torch.distributed as dist

            self.world = dist.get_world_size(group)
        if batch % self.world:
            raise ValueError(f"global batch {batch} not divisible by {self.world} ranks")
        self.local_batch = batch // self.world
        # small chains on one GPU: the whole step is one launch (sg_mlp_small_step)
        self.engine = ChainEngine(chain, self.local_batch, loss, precision, global_batch=batch,
                                  small=small and not dp)
        self.dp = None
        if dp:
            backend = dp_backend or _default_dp_backend(group)
            if backend not in ("sg", "torch"):
                raise ValueError(f"unknown dp backend {backend!r}")
            cls = NcclDataParallel if backend == "sg" else DataParallel
            import os

            slices = int(os.environ.get("SGB200_DP_L0_SLICES", "4"))
            min_params = int(os.environ.get("SGB200_DP_L0_SLICE_MIN", str(8 << 20)))
            self.engine.enable_first_layer_slices(slices, min_params)  # before the bucket list is handed over
            self.dp = cls(self.engine.G, self.engine.bucket_bounds, group)
            self.engine.grad_ready = self.dp.ready
            self.dp.broadcast_params(self.engine.P)
            if self.engine.S is not None:
                self.engine.S.copy_(self.engine.P.to(self.engine.S.dtype))
        self.graph = None
        # torch.distributed's async work handles are host-side objects; the
        # library's communicator is stream-ordered and can live in a graph
        self.use_graph = graph and (self.dp is None or isinstance(self.dp, NcclDataParallel))
        self._graphs = collections.OrderedDict()  # (X, Y) buffers -> captured step (LRU)
        self._seen = collections.OrderedDict()    # pairs stepped once, not captured yet (LRU)
        self._last_key = None
        self._small_graph = None  # the one-launch step last replayed (graphs keyed per (X, Y, lr) in _graphs)

    def _device_step(self):
        # NVTX ranges per phase (the C-ABI calls inside carry their own)
        from torch.cuda import nvtx

        e = self.engine
        with nvtx.range("sgb200.forward"):
            e.forward(fuse_loss=True)
        with nvtx.range("sgb200.loss"):
            e.loss_and_seed()
        with nvtx.range("sgb200.pullback"):
            e.pullback()
        if self.dp is not None:
            with nvtx.range("sgb200.allreduce_wait"):
                self.dp.finish()
        with nvtx.range("sgb200.sgd"):
            e.sgd(self.lr)

    def step(self, X, Y):
        """One training step on (X, Y) already on the device; returns the loss (device)."""
        if self.engine.small is not None:  # the whole step is one launch
            if not self.use_graph:
                return self.engine.small_step(X, Y, self.lr)
            # a CUDA-graph replay issues it in ~3 us of host time instead of
            # the ~9 us of a cooperative launch (the c1 step is a 16 us kernel):
            # first call per (X, Y, lr) eager, the next one captures, then replays
            key = ("small", X.data_ptr(), Y.data_ptr(), tuple(X.shape), tuple(Y.shape), X.stride(0), Y.stride(0),
                   X.dtype, Y.dtype, self.lr)
            g = self._graphs.get(key)
            if g is None and key in self._seen:  # second step on this pair: capture (as below)
                g = Tape.capture(lambda: self.engine.small_step(X, Y, self.lr), warmup=0)
                self._graphs[key] = g
                del self._seen[key]
                while len(self._graphs) > self.MAX_GRAPHS:
                    self._graphs.popitem(last=False)
            elif g is None:
                self._seen[key] = True
                while len(self._seen) > 4 * self.MAX_GRAPHS:
                    self._seen.popitem(last=False)
                return self.engine.small_step(X, Y, self.lr)
            self._graphs.move_to_end(key)
            self._small_graph = g
            g.replay()
            return self.engine.loss
        if not self.use_graph:
            self.engine.load_batch(X, Y)
            self._device_step()
            return self.engine.loss
        # CUDA graphs of the whole step, the minibatch load included (it reads X
        # and Y in place, so a graph is keyed by their buffers): the first step
        # on a (X, Y) pair runs eagerly (one-time kernel attribute setup), the
        # second captures -- without warm-up, so no extra update is applied --
        # and later ones replay.  A few pairs are kept (double-buffered loaders).
        key = (X.data_ptr(), Y.data_ptr(), tuple(X.shape), tuple(Y.shape), X.stride(0), Y.stride(0),
               X.dtype, Y.dtype)
        # (a pair is captured on its second step, consecutive or not, so
        # loaders that alternate a few buffers replay too)
        g = self._graphs.get(key)
        if g is None and key in self._seen:
            g = Tape.capture(lambda: (self.engine.load_batch(X, Y), self._device_step()), warmup=0)
            self._graphs[key] = g
            del self._seen[key]
            while len(self._graphs) > self.MAX_GRAPHS:
                self._graphs.popitem(last=False)
        elif g is None:
            self._seen[key] = True
            while len(self._seen) > 4 * self.MAX_GRAPHS:
                self._seen.popitem(last=False)
        self._last_key = key
        if g is not None:
            self._graphs.move_to_end(key)
            self.graph = g
            g.replay()
        else:
            self.engine.load_batch(X, Y)
            self._device_step()
        return self.engine.loss

    def check(self) -> None:
        """Raise what the reference would have raised on the steps run since
        the last check (synchronises): OverflowError for math.exp overflow,
        EvalError(DomainError) for division by zero / log of p <= 0 in the
        loss (runtime.domain_check; include/sgb200.h SG_DOM_*).  The values
        themselves are computed stably whatever the flags say."""
        from . import runtime as rt

        rt.domain_check(function="loss")

    def replicas_identical(self) -> bool:
        """Data parallel: the parameter replicas are bit-identical on all ranks."""
        if self.dp is None:
            return True
        return replicas_identical(self.engine.P, self.dp.group)

    def close(self) -> None:
        """Release the data-parallel communicator (its NCCL comm and the SMs it
        keeps free of the GEMM grids) and the captured graphs.  Idempotent;
        also runs when the Trainer is garbage-collected."""
        dp, self.dp = getattr(self, "dp", None), None
        self.graph = self._small_graph = None
        if getattr(self, "_graphs", None):
            self._graphs.clear()
        if getattr(self, "engine", None) is not None:
            self.engine.grad_ready = None
        if dp is not None and hasattr(dp, "close"):
            import torch

            torch.cuda.synchronize()  # in-flight collectives finish before the comm goes
            dp.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def gradient(self, X, Y):
        """Loss and parameter gradients without the update (the pullback API)."""
        e = self.engine
        e.load_batch(X, Y)
        e.forward(fuse_loss=True)
        e.loss_and_seed()
        e.pullback()
        if self.dp is not None:
            self.dp.finish()
        self.check()
        return float(e.loss.item()), e.get_grads()


def replicas_identical(t, group=None) -> bool:
    """True when ``t`` is bit-identical on every rank of ``group`` (SURVEY
    §8(e): every rank applies the same SGD to the same all-reduced gradient,
    so the parameter replicas must never drift; checked, not assumed).
    Compares an order-independent integer checksum of the raw bits plus the
    element count, gathered over the group."""
    import torch
    import torch.distributed as dist

    raw = t.detach().contiguous().view(-1)
    bits = raw.view(torch.int32) if raw.element_size() == 4 else raw.view(torch.int64)
    words = bits.to(torch.int64)
    pos = torch.arange(words.numel(), device=words.device, dtype=torch.int64)
    sig = torch.stack([words.sum(), (words * (pos % 65521 + 1)).sum(), torch.tensor(words.numel(), device=words.device)])
    gathered = [torch.zeros_like(sig) for _ in range(dist.get_world_size(group))]
    dist.all_gather(gathered, sig, group=group)
    return all(torch.equal(g, gathered[0]) for g in gathered)


def shard_rows(X: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Rows of the global minibatch owned by ``rank`` (contiguous blocks)."""
    n = X.shape[0] // world
    return X[rank * n:(rank + 1) * n]
