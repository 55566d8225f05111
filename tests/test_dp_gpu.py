"""The real data-parallel training step with two ranks on one GPU.

Two processes share cuda:0 under a gloo process group; each holds half of
the global minibatch (contiguous row blocks, train.shard_rows) and runs the
device step through Trainer(dp=True, dp_backend="torch"): ChainEngine
forward / fused loss scaled by the GLOBAL 1/B (nn_train.py:226) / pullback,
with every gradient bucket all-reduced (SUM) as the pullback readies it, in
the flat [W0, b0, W1, b1, ...] order (nn_train.py:99-103).  The collective
is host-mediated gloo: no kernel of one rank waits on the other's.

Checked against a single-process full-batch step on the same GPU:
* gradients within fp32 summation-order tolerance (the row sums of dW / db
  are split in two halves instead of one pass), 1e-5 of each tensor's max;
* loss within 1e-6 (sum of the two shard losses vs the full-batch loss);
* after SGD steps the parameter replicas are bit-identical on both ranks
  (replicas_identical) and match the single-process parameters within the
  same tolerance;
* the same with layer 0's dW in 4 row slices, each its own bucket
  (SGB200_DP_L0_SLICE_MIN=0 forces slicing at this size).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

SIZES, ACTS, B = (256, 512, 512, 128), ("tanh", "tanh", "identity"), 1024


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _chain():
    from paper_1811_01457_b200.dense import Chain, Dense

    chain = Chain(*[Dense(SIZES[i], SIZES[i + 1], ACTS[i]) for i in range(len(ACTS))]).init_params(
        np.random.default_rng(9))
    for l in chain.layers:
        l.b = np.random.default_rng(10).uniform(-0.1, 0.1, l.fan_out).astype(np.float32)
    return chain


def _data():
    rng = np.random.default_rng(5)
    X = rng.uniform(0, 1, (B, SIZES[0])).astype(np.float32)
    Y = rng.uniform(-1, 1, (B, SIZES[-1])).astype(np.float32)
    return X, Y


def _worker(rank, world, port, q, sliced, precision):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if sliced:
        os.environ["SGB200_DP_L0_SLICE_MIN"] = "0"
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1811_01457_b200.train import DataParallel, Trainer, shard_rows

        X, Y = _data()
        Xs = torch.from_numpy(shard_rows(X, rank, world)).cuda()
        Ys = torch.from_numpy(shard_rows(Y, rank, world)).cuda()
        tr = Trainer(_chain(), B, loss="mse", lr=0.01, precision=precision, dp=True, dp_backend="torch")
        assert isinstance(tr.dp, DataParallel) and tr.local_batch == B // world
        assert len(tr.engine.bucket_bounds) == (len(ACTS) + 3 if sliced else len(ACTS))
        lv, grads = tr.gradient(Xs, Ys)
        lt = torch.tensor([lv], dtype=torch.float64)
        dist.all_reduce(lt)
        losses = [float(tr.step(Xs, Ys).item()) for _ in range(3)]
        torch.cuda.synchronize()
        same = tr.replicas_identical()
        params = tr.engine.get_params()
        tr.close()
        q.put((rank, float(lt.item()), grads, params, same, losses))
    except Exception as e:  # report, the parent asserts
        q.put((rank, repr(e), None, None, False, None))
        raise
    finally:
        dist.destroy_process_group()


def _single(precision):
    from paper_1811_01457_b200.train import Trainer

    X, Y = _data()
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    tr = Trainer(_chain(), B, loss="mse", lr=0.01, precision=precision, small=False)
    lv, grads = tr.gradient(Xd, Yd)
    for _ in range(3):
        tr.step(Xd, Yd)
    return lv, grads, tr.engine.get_params()


def nrel(got, want):
    return float(np.abs(np.asarray(got) - np.asarray(want)).max() / max(np.abs(want).max(), 1e-30))


@pytest.mark.parametrize("sliced", [False, True])
@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_two_rank_data_parallel_step_matches_full_batch(sliced, precision):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, sliced, precision)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lv1, g1, p1 = _single(precision)
    for rank, lv, grads, params, same, _ in res:
        assert grads is not None, lv
        assert same, rank
        assert abs(lv - lv1) <= 1e-6 * max(1.0, abs(lv1)), (lv, lv1)
        for (gW, gb), (wW, wb) in zip(grads, g1):
            assert nrel(gW, wW) <= 1e-5 and nrel(gb, wb) <= 1e-5
        for (W, b), (W1, b1), (W0, b0) in zip(params, p1, [(l.W, l.b) for l in _chain().layers]):
            assert nrel(W - W0, W1 - W0) <= 1e-3 and nrel(b - b0, b1 - b0) <= 1e-3
    # both ranks hold the same parameters, bit for bit
    for (Wa, ba), (Wb, bb) in zip(res[0][3], res[1][3]):
        assert np.array_equal(Wa, Wb) and np.array_equal(ba, bb)
