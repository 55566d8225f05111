"""Multi-process data-parallel host logic on CPU (gloo, world size 2 and 4).

Each rank computes its shard's gradient with the loss scaled by the GLOBAL
1/B (oracle restatement of the reference pullback), packs it into the
flat [W0, b0, W1, b1, ...] buffer (nn_train.py:99-103 order) with the
engine's bucket layout, and the bucketed all-reduce of
paper_1811_01457_b200.train.DataParallel must reproduce the full-batch
gradient.  The device kernels are covered by the GPU tests; this checks
sharding, scaling, bucketing and the collective itself.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dense as OD


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layout(sizes):
    """Same flat layout rule as ChainEngine (64-element aligned segments)."""
    ld = lambda d: (d + 7) // 8 * 8  # noqa: E731
    off, segs = 0, []
    for i in range(len(sizes) - 1):
        fi, fo = sizes[i], sizes[i + 1]
        wo = off
        off = (off + fo * ld(fi) + 63) // 64 * 64
        bo = off
        off = (off + fo + 63) // 64 * 64
        segs.append((wo, bo, fi, fo))
    return off, segs


def _pack(grads, sizes):
    n, segs = _layout(sizes)
    flat = np.zeros(n)
    for (dW, db), (wo, bo, fi, fo) in zip(grads, segs):
        ldi = (fi + 7) // 8 * 8
        flat[wo:wo + fo * ldi].reshape(fo, ldi)[:, :fi] = dW
        flat[bo:bo + fo] = db
    buckets = [(wo, (bo + fo + 63) // 64 * 64) for wo, bo, fi, fo in segs]
    return flat, buckets


def _shard_grads(params, X, Y, acts, loss, B_global):
    # loss of the shard with the global mean scale: scale the oracle's 1/n by n/B
    lv, grads, _ = OD.mlp_step(params, X, Y, acts, loss, mode="blas")
    f = X.shape[0] / B_global
    return lv * f, [(dW * f, db * f) for dW, db in grads]


def _worker(rank, world, port, q, sliced=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1811_01457_b200.dense import pullback_ready_order, slice_first_layer_buckets
        from paper_1811_01457_b200.train import DataParallel, shard_rows

        rng = np.random.default_rng(0)  # same data and params on every rank
        sizes, acts = ((20, 256, 7) if sliced else (20, 13, 7)), ("tanh", "identity")
        B = 16
        params = [(rng.uniform(-0.5, 0.5, (sizes[i + 1], sizes[i])), rng.uniform(-0.1, 0.1, sizes[i + 1]))
                  for i in range(2)]
        X = rng.uniform(0, 1, (B, sizes[0]))
        Y = rng.uniform(-1, 1, (B, sizes[-1]))
        lv, grads = _shard_grads(params, shard_rows(X, rank, world), shard_rows(Y, rank, world), acts, "mse", B)
        flat, buckets = _pack(grads, sizes)
        if sliced:  # layer 0's bucket as 4 row slices of W0 (the last through b0), ChainEngine's rule
            _, segs = _layout(sizes)
            whole = buckets
            buckets = slice_first_layer_buckets(buckets, segs[0][0], sizes[0], sizes[1], 4)
            assert len(buckets) == len(whole) + 3
            assert buckets[0][0] == whole[0][0] and buckets[3][1] == whole[0][1]
            assert all(a[1] == b[0] for a, b in zip(buckets[:3], buckets[1:4]))  # contiguous, no overlap
        G = torch.from_numpy(flat)
        dp = DataParallel(G, buckets)
        # the engine's own readying order: top layer first, then W0's slices ascending
        order = pullback_ready_order(len(acts), 4 if sliced else 1)
        assert sorted(order) == list(range(len(buckets)))
        for i in order:
            dp.ready(i)
        dp.finish()
        loss = torch.tensor([lv], dtype=torch.float64)
        dist.all_reduce(loss)
        full_lv, full_grads = _shard_grads(params, X, Y, acts, "mse", B)
        want, _ = _pack(full_grads, sizes)
        err = float(np.abs(G.numpy() - want).max())
        q.put((rank, err, abs(float(loss.item()) - full_lv)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,sliced", [(2, False), (4, False), (2, True)])
def test_bucketed_allreduce_reproduces_full_batch_gradient(world, sliced):
    """Bucketed all-reduce of shard gradients == full-batch gradient; with
    `sliced`, layer 0's bucket is split into W0 row slices as data-parallel
    ChainEngines do for large first layers (readied last, in pullback order)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, sliced)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = [q.get(timeout=10) for _ in range(world)]
    for p in procs:
        assert p.exitcode == 0
    for rank, err, lerr in results:
        assert err <= 1e-12, (rank, err)
        assert lerr <= 1e-12, (rank, lerr)


def test_layout_matches_engine_rule():
    n, segs = _layout((784, 32, 10))
    assert all(wo % 64 == 0 and bo % 64 == 0 for wo, bo, _, _ in segs)
    assert n % 64 == 0


def _id_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1811_01457_b200.train import nccl_unique_id

        q.put((rank, nccl_unique_id()))
    finally:
        dist.destroy_process_group()


def test_nccl_unique_id_rendezvous():
    """The NCCL communicator's rendezvous (train.nccl_unique_id): every rank
    receives rank 0's 128-byte id from sg_dp_unique_id (host-only path)."""
    from paper_1811_01457_b200 import runtime as rt

    try:
        if not rt.load_library().sg_dp_available():
            pytest.skip("libnccl.so.2 not found")
    except rt.RuntimeUnavailable:
        pytest.skip("library not built")
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    ids = dict(q.get(timeout=10) for _ in range(world))
    for p in procs:
        assert p.exitcode == 0
    assert len(ids[0]) == 128 and any(ids[0])
    assert ids[0] == ids[1] == ids[2]


def _replica_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1811_01457_b200.train import replicas_identical

        p = torch.linspace(-1, 1, 1000, dtype=torch.float32)
        same = replicas_identical(p)
        if rank == 1:
            p[17] = torch.nextafter(p[17], torch.tensor(2.0))  # one ulp on one rank
        q.put((rank, same, replicas_identical(p)))
    finally:
        dist.destroy_process_group()


def test_replica_check_detects_one_ulp_drift():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = [q.get(timeout=10) for _ in range(world)]
    for p in procs:
        assert p.exitcode == 0
    assert all(same for _, same, _ in res)
    assert not any(drift for _, _, drift in res)


def test_pullback_ready_order_maps_every_bucket_once():
    """Host-only: the bucket indices ChainEngine readies (top layer first,
    layer 0's W0 slices last and ascending) cover the sliced bucket list of
    slice_first_layer_buckets exactly once, and each bucket index holds the
    layer the pullback has just finished."""
    from paper_1811_01457_b200.dense import bucket_of_layer, pullback_ready_order, slice_first_layer_buckets

    for L in (1, 2, 4, 16):
        assert pullback_ready_order(L, 1) == list(range(L - 1, -1, -1))
        for S in (2, 4):
            order = pullback_ready_order(L, S)
            assert sorted(order) == list(range(L + S - 1))
            assert order[-S:] == list(range(S))          # W0 slices, ascending, last
            assert order[:L - 1] == [l + S - 1 for l in range(L - 1, 0, -1)]
            sizes = [64] + [256] * L
            _, segs = _layout(sizes)
            whole = [(wo, (bo + fo + 63) // 64 * 64) for wo, bo, fi, fo in segs]
            sliced = slice_first_layer_buckets(whole, segs[0][0], sizes[0], sizes[1], S)
            for l in range(1, L):  # a layer's bucket is its whole segment, shifted by S-1
                assert sliced[bucket_of_layer(l, S)] == whole[l]
            rows = sizes[1] // S
            ldi = (sizes[0] + 7) // 8 * 8
            for k in range(S):
                lo, hi = sliced[bucket_of_layer(0, S, k)]
                assert lo == segs[0][0] + k * rows * ldi
