"""GPU parity of the Dense training step against the reference.

Golden vectors: the unmodified reference's `grad` through Dense-chain IR
(tests/golden/mlp_*.npz, dense_sigmoid.npz).  Larger shapes: the pinned
oracle (oracle/dense.py).  Tolerances, per tensor, relative to the
tensor's largest magnitude (norm-relative, stricter than the elementwise
rel metric for small gradients):
  bf16 tensor-core path   <= 1e-2  (north star, TF32/BF16 GEMMs)
  tf32 tensor-core path   <= 3e-3  (fp32 operands read as TF32: 2^-10 per operand)
  strict_fp32             <= 1e-5
  strict_fp64             <= 1e-12 (only exp/tanh libm ulps differ)
"""

import numpy as np
import pytest

from conftest import load_npz
from oracle import dense as OD

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1811_01457_b200.dense import Chain, ChainEngine, Dense, DenseLayer  # noqa: E402
from paper_1811_01457_b200.train import Trainer  # noqa: E402

TOL = {"bf16": 1e-2, "tf32": 3e-3, "strict_fp32": 1e-5, "strict_fp64": 1e-12}


def nrel(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-30))


def chain_from(z, acts):
    sizes = [int(s) for s in z["sizes"]]
    layers = [Dense(sizes[i], sizes[i + 1], acts[i], z[f"W{i}"].astype(np.float64),
                    z[f"b{i}"].astype(np.float64)) for i in range(len(acts))]
    return Chain(*layers)


@pytest.mark.parametrize("precision", ["bf16", "tf32", "strict_fp32", "strict_fp64"])
@pytest.mark.parametrize("name,acts,loss", [
    ("mlp_c1_b32.npz", ("sigmoid", "identity"), "softmax_xent"),
    ("mlp_mse.npz", ("tanh", "tanh", "identity"), "mse"),
    ("mlp_bce.npz", ("tanh", "identity"), "bce"),  # 19 of 48 predictions clamped
])
def test_chain_gradients_match_reference(precision, name, acts, loss):
    z = load_npz(name)
    chain = chain_from(z, acts)
    n = z["X"].shape[0]
    tr = Trainer(chain, n, loss=loss, precision=precision)
    dt = torch.float64 if precision == "strict_fp64" else torch.float32
    X = torch.from_numpy(z["X"]).to(dt).cuda()
    Y = torch.from_numpy(z["Y"]).to(dt).cuda()
    lv, grads = tr.gradient(X, Y)
    tol = TOL[precision]
    assert abs(lv - z["loss"][0]) <= tol * max(1.0, abs(z["loss"][0]))
    for k, (gW, gb) in enumerate(grads):
        assert nrel(gW, z[f"dW{k}"]) <= tol, (k, nrel(gW, z[f"dW{k}"]))
        assert nrel(gb, z[f"db{k}"]) <= tol, (k, nrel(gb, z[f"db{k}"]))


@pytest.mark.parametrize("precision", ["bf16", "tf32", "strict_fp64"])
def test_sgd_step_matches_oracle(precision):
    z = load_npz("mlp_c1_b32.npz")
    acts = ("sigmoid", "identity")
    chain = chain_from(z, acts)
    tr = Trainer(chain, 32, loss="softmax_xent", lr=0.05, precision=precision)
    dt = torch.float64 if precision == "strict_fp64" else torch.float32
    X = torch.from_numpy(z["X"]).to(dt).cuda()
    Y = torch.from_numpy(z["Y"]).to(dt).cuda()
    tr.step(X, Y)
    params = [(z[f"W{k}"].astype(np.float64), z[f"b{k}"].astype(np.float64)) for k in range(2)]
    _, _, new = OD.mlp_step(params, z["X"].astype(np.float64), z["Y"].astype(np.float64), acts,
                            "softmax_xent", lr=0.05, mode="exact")
    got = tr.engine.get_params()
    for (W, b), (Wn, bn), (W0, b0) in zip(got, new, params):
        # compare the update itself (p_new - p_old) against the oracle's
        assert nrel(W - W0, Wn - W0) <= TOL[precision] * 10
        assert nrel(b - b0, bn - b0) <= TOL[precision] * 10


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_dense_layer_pullback_matches_reference(precision):
    z = load_npz("dense_sigmoid.npz")
    W, b = z["W0"].astype(np.float64), z["b0"].astype(np.float64)
    X, Ybar = z["X"].astype(np.float64), z["Y"].astype(np.float64)
    layer = DenseLayer(X.shape[0], W.shape[1], W.shape[0], "sigmoid", precision=precision)
    layer.set_params(W, b)
    layer.forward(torch.from_numpy(X).to(layer.X.dtype).cuda())
    dX, dW, db = layer.pullback(torch.from_numpy(Ybar).float().cuda())
    torch.cuda.synchronize()
    tol = TOL[precision]
    assert nrel(dX.double().cpu(), z["dX"]) <= tol
    assert nrel(dW.double().cpu(), z["dW0"]) <= tol
    assert nrel(db.double().cpu(), z["db0"]) <= tol


@pytest.mark.parametrize("sizes,acts,loss,B", [
    ((784, 32, 10), ("sigmoid", "identity"), "softmax_xent", 128),       # c1 at full size
    ((256, 256, 256, 256, 256), ("tanh",) * 3 + ("identity",), "mse", 1024),  # c4/c5 shape, scaled
    ((1024, 1024, 1024), ("tanh", "identity"), "mse", 4096),
])
@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_chain_vs_oracle_at_size(sizes, acts, loss, B, precision):
    rng = np.random.default_rng(B)
    chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(len(acts))]).init_params(rng)
    for l in chain.layers:
        l.b = rng.uniform(-0.1, 0.1, l.fan_out).astype(np.float32)
    X = rng.uniform(0, 1, (B, sizes[0])).astype(np.float32)
    if loss == "softmax_xent":
        Y = np.zeros((B, sizes[-1]), np.float32)
        Y[np.arange(B), rng.integers(0, sizes[-1], B)] = 1
    else:
        Y = rng.uniform(-1, 1, (B, sizes[-1])).astype(np.float32)
    tr = Trainer(chain, B, loss=loss, precision=precision)
    lv, grads = tr.gradient(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda())
    # oracle on the same bf16-rounded operands the tensor cores see
    params = [(l.W.astype(np.float64), l.b.astype(np.float64)) for l in chain.layers]
    lo, go, _ = OD.mlp_step(params, X.astype(np.float64), Y.astype(np.float64), acts, loss, mode="blas")
    tol = TOL[precision]
    assert abs(lv - lo) <= tol * max(1.0, abs(lo))
    for (gW, gb), (oW, ob) in zip(grads, go):
        assert nrel(gW, oW) <= tol
        assert nrel(gb, ob) <= tol


def test_cuda_graph_replay_matches_eager_and_is_deterministic():
    rng = np.random.default_rng(7)
    sizes, acts = (256, 512, 512, 128), ("tanh", "tanh", "identity")
    B = 512
    X = torch.from_numpy(rng.uniform(0, 1, (B, sizes[0])).astype(np.float32)).cuda()
    Y = torch.from_numpy(rng.uniform(-1, 1, (B, sizes[-1])).astype(np.float32)).cuda()

    def run(graph):
        chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(3)]).init_params(
            np.random.default_rng(1))
        tr = Trainer(chain, B, loss="mse", lr=0.002, precision="bf16", graph=graph)
        losses = [float(tr.step(X, Y).item()) for _ in range(5)]
        return losses, tr.engine.P.clone()

    l1, p1 = run(False)
    l2, p2 = run(True)
    l3, p3 = run(True)
    assert l1 == l2 == l3
    assert torch.equal(p1, p2) and torch.equal(p2, p3)
    assert l1[-1] < l1[0]  # it trains


def test_data_parallel_trainer_over_nccl_world1():
    """The DP code path (NCCL process group, bucketed async all-reduce issued
    from inside the pullback, broadcast of initial params) on the one GPU a
    box has: with world size 1 it must reproduce the single-GPU step -- for
    both all-reduce backends (torch.distributed, and the library's own NCCL
    communicator sg_dp_*, eager and captured in a CUDA graph)."""
    import os
    import socket

    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(5)
        sizes, acts = (256, 512, 128), ("tanh", "identity")
        B = 1024
        X = torch.from_numpy(rng.uniform(0, 1, (B, sizes[0])).astype(np.float32)).cuda()
        Y = torch.from_numpy(rng.uniform(-1, 1, (B, sizes[-1])).astype(np.float32)).cuda()

        from paper_1811_01457_b200.train import NcclDataParallel

        def run(dp, backend=None, graph=False):
            chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(2)]).init_params(
                np.random.default_rng(9))
            tr = Trainer(chain, B, loss="mse", lr=0.002, precision="bf16", dp=dp, dp_backend=backend,
                         graph=graph)
            if backend == "sg":
                assert isinstance(tr.dp, NcclDataParallel)
                assert tr.use_graph == graph
            if dp:  # 2 layers: 2 buckets, or 5 with layer 0 in 4 slices
                sliced = os.environ.get("SGB200_DP_L0_SLICE_MIN") == "0"
                assert len(tr.engine.bucket_bounds) == (5 if sliced else 2)
            losses = [float(tr.step(X, Y).item()) for _ in range(3)]
            assert tr.replicas_identical()
            if tr.dp is not None and hasattr(tr.dp, "close"):
                torch.cuda.synchronize()
                tr.dp.close()
            return losses, tr.engine.P.clone()

        l0, p0 = run(False)
        for backend, graph in (("torch", False), ("sg", False), ("sg", True)):
            l1, p1 = run(True, backend, graph)
            assert l0 == l1, backend
            assert torch.equal(p0, p1), backend
        # layer 0's dW in 4 row slices, each its own bucket (forced on at this
        # small size): still bit-identical to the single-GPU step
        os.environ["SGB200_DP_L0_SLICE_MIN"] = "0"
        try:
            for backend, graph in (("torch", False), ("sg", True)):
                l1, p1 = run(True, backend, graph)
                assert l0 == l1, backend
                assert torch.equal(p0, p1), backend
        finally:
            del os.environ["SGB200_DP_L0_SLICE_MIN"]
    finally:
        dist.destroy_process_group()


def test_data_parallel_shards_sum_to_full_gradient():
    """Single-GPU check of the DP math: shard gradients scaled by the global
    1/B sum to the full-batch gradient (the all-reduce itself is covered by
    the gloo multi-process test on CPU)."""
    rng = np.random.default_rng(3)
    sizes, acts = (128, 256, 64), ("tanh", "identity")
    B, world = 512, 4
    chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(2)]).init_params(rng)
    X = rng.uniform(0, 1, (B, sizes[0])).astype(np.float32)
    Y = rng.uniform(-1, 1, (B, sizes[-1])).astype(np.float32)
    full = ChainEngine(chain, B, "mse", "strict_fp64")
    full.load_batch(torch.from_numpy(X).double().cuda(), torch.from_numpy(Y).double().cuda())
    full.forward(); full.loss_and_seed(); full.pullback()
    acc = torch.zeros_like(full.G)
    for r in range(world):
        e = ChainEngine(chain, B // world, "mse", "strict_fp64", global_batch=B)
        xs = X[r * B // world:(r + 1) * B // world]
        ys = Y[r * B // world:(r + 1) * B // world]
        e.load_batch(torch.from_numpy(xs).double().cuda(), torch.from_numpy(ys).double().cuda())
        e.forward(); e.loss_and_seed(); e.pullback()
        acc += e.G
    assert nrel(acc.cpu().numpy(), full.G.cpu().numpy()) <= 1e-12


@pytest.mark.parametrize("precision", ["bf16", "tf32", "strict_fp32"])
def test_dense_abi_backward_without_fused_partials(precision):
    """sg_dense_backward computing db itself (no producer-fused colsum), with
    the lower layer's act' fused into dX, vs a float64 restatement."""
    from paper_1811_01457_b200.dense import dense_backward, dense_desc, dense_forward

    rng = np.random.default_rng(5)
    B, fi, fo = 200, 72, 136
    dt = torch.bfloat16 if precision == "bf16" else torch.float32
    X = torch.from_numpy(rng.uniform(0.05, 0.95, (B, fi)).astype(np.float32)).to(dt).cuda()
    W = torch.from_numpy(rng.uniform(-0.3, 0.3, (fo, fi)).astype(np.float32)).to(dt).cuda()
    b = torch.from_numpy(rng.uniform(-0.1, 0.1, fo).astype(np.float32)).cuda()
    dZ = torch.from_numpy(rng.uniform(-1, 1, (B, fo)).astype(np.float32)).to(dt).cuda()
    d = dense_desc(X, W, b, "tanh", precision)
    H = torch.empty((B, fo), dtype=dt, device="cuda")
    dense_forward(d, H=H)
    dW = torch.empty((fo, fi), device="cuda")
    db = torch.empty(fo, device="cuda")
    dX = torch.empty((B, fi), dtype=dt, device="cuda")
    dense_backward(d, dZ, dW, db, dX=dX, act_prev="sigmoid")
    torch.cuda.synchronize()
    x, w, z = (t.double().cpu().numpy() for t in (X, W, dZ))
    tol = {"bf16": 1e-2, "tf32": 3e-3, "strict_fp32": 1e-5}[precision]
    assert nrel(H.double().cpu(), np.tanh(x @ w.T + b.double().cpu().numpy())) <= tol
    assert nrel(dW.double().cpu(), z.T @ x) <= tol
    assert nrel(db.double().cpu(), z.sum(axis=0)) <= 1e-5
    assert nrel(dX.double().cpu(), (z @ w) * x * (1 - x)) <= tol
    if precision == "strict_fp32":  # partial column sums are a tensor-core feature
        cs = torch.zeros(((B + 31) // 32, fo), device="cuda")
        with pytest.raises(ValueError, match="tensor-core"):
            dense_backward(d, dZ, dW, db, colsum_in=cs)


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_dense_layer_c3_full_size(precision):
    """BASELINE c3 at its full size (Dense 4096->4096, batch 8192, sigmoid):
    forward and pullback vs an fp64 evaluation of the same layer on the same
    (bf16-rounded / fp32) operands (torch, test-side only)."""
    M, D = 8192, 4096
    g = torch.Generator(device="cuda").manual_seed(7)
    layer = DenseLayer(M, D, D, "sigmoid", precision=precision)
    r = (6.0 / (2 * D)) ** 0.5
    W = (torch.rand((D, D), generator=g, device="cuda") * 2 - 1) * r
    b = (torch.rand(D, generator=g, device="cuda") * 2 - 1) * 0.01
    layer.set_params(W.cpu().numpy(), b.cpu().numpy())
    X = (torch.rand((M, D), generator=g, device="cuda") * 2 - 1).to(layer.X.dtype)
    ybar = torch.rand((M, D), generator=g, device="cuda") * 2 - 1
    H = layer.forward(X).double()
    dX, dW, db = (t.double() for t in layer.pullback(ybar))
    torch.cuda.synchronize()
    x64, w64 = X.double(), layer.Wb.double()
    s = torch.sigmoid(x64 @ w64.T + b.double())
    dz = ybar.double() * s * (1 - s)

    def nrel_t(u, v):
        return float((u - v).abs().max() / v.abs().max())

    tol = TOL[precision]
    assert nrel_t(H, s) <= tol
    assert nrel_t(dX, dz @ w64) <= tol
    assert nrel_t(dW, dz.T @ x64) <= tol
    assert nrel_t(db, dz.sum(0)) <= tol


_SMALL_OFF = pytest.mark.skipif(__import__("os").environ.get("SGB200_MLP_SMALL") == "0",
                                reason="one-launch small step disabled (SGB200_MLP_SMALL=0)")


@pytest.mark.parametrize("sizes,acts,loss,B", [
    ((784, 32, 10), ("sigmoid", "identity"), "softmax_xent", 128),   # c1 at full size
    ((784, 32, 10), ("sigmoid", "identity"), "softmax_xent", 129),   # last CTA holds one row
    ((64, 48, 40, 24, 8), ("tanh", "relu", "sigmoid", "identity"), "mse", 200),
    ((100, 30, 5), ("tanh", "sigmoid"), "mse", 7),                   # activated top layer, tiny batch
])
@_SMALL_OFF
def test_small_chain_one_launch_step_matches_oracle(sizes, acts, loss, B):
    """sg_mlp_small_step (the whole step in one cooperative launch, fp32):
    loss, gradients and the SGD update against the fp64 oracle, and bit-identical
    to itself across runs (fixed-order reductions)."""
    rng = np.random.default_rng(B)
    X = rng.uniform(0, 1, (B, sizes[0])).astype(np.float32)
    if loss == "softmax_xent":
        Y = np.zeros((B, sizes[-1]), np.float32)
        Y[np.arange(B), rng.integers(0, sizes[-1], B)] = 1
    else:
        Y = rng.uniform(-1, 1, (B, sizes[-1])).astype(np.float32)

    def run():
        chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(len(acts))]).init_params(
            np.random.default_rng(3))
        for l in chain.layers:
            l.b = np.random.default_rng(4).uniform(-0.1, 0.1, l.fan_out).astype(np.float32)
        tr = Trainer(chain, B, loss=loss, lr=0.05, precision="bf16")
        assert tr.engine.small is not None
        lv = float(tr.step(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()).item())
        return chain, lv, tr.engine.get_grads(), tr.engine.get_params(), tr.engine.P.clone()

    chain, lv, grads, new, P1 = run()
    _, lv2, _, _, P2 = run()
    assert lv == lv2 and torch.equal(P1, P2)
    params = [(l.W.astype(np.float64), l.b.astype(np.float64)) for l in chain.layers]
    lo, go, no = OD.mlp_step(params, X.astype(np.float64), Y.astype(np.float64), acts, loss, lr=0.05,
                             mode="blas")
    tol = 2e-5  # fp32 end to end
    assert abs(lv - lo) <= tol * max(1.0, abs(lo))
    for (gW, gb), (oW, ob) in zip(grads, go):
        assert nrel(gW, oW) <= tol
        assert nrel(gb, ob) <= tol
    for (W, b), (Wn, bn), (W0, b0) in zip(new, no, params):
        assert nrel(W - W0, Wn - W0) <= tol
        assert nrel(b - b0, bn - b0) <= tol


@_SMALL_OFF
def test_small_chain_step_equals_layer_path_and_trains():
    """The one-launch step and the layer-by-layer tensor-core path (SGB200
    small path off) train the c1 model to the same losses (within bf16), and
    the one-launch step keeps the bf16 shadow in sync with P."""
    rng = np.random.default_rng(0)
    sizes, acts, B = (784, 32, 10), ("sigmoid", "identity"), 128
    X = torch.from_numpy(rng.uniform(0, 1, (B, 784)).astype(np.float32)).cuda()
    Y = torch.zeros((B, 10), device="cuda")
    Y[torch.arange(B), torch.from_numpy(rng.integers(0, 10, B)).cuda()] = 1

    def run(small):
        chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(2)]).init_params(
            np.random.default_rng(1))
        tr = Trainer(chain, B, loss="softmax_xent", lr=0.5, precision="bf16", small=small, graph=not small)
        assert (tr.engine.small is not None) == small
        assert tr.compute_precision == ("fp32" if small else "bf16")  # the API says what runs
        return [float(tr.step(X, Y).item()) for _ in range(20)], tr

    ls, trs = run(True)
    ll, _ = run(False)
    # the same one-launch steps replayed from a CUDA graph: bit-identical
    chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(2)]).init_params(np.random.default_rng(1))
    trg = Trainer(chain, B, loss="softmax_xent", lr=0.5, precision="bf16", small=True, graph=True)
    lg = [float(trg.step(X, Y).item()) for _ in range(20)]
    assert trg._small_graph is not None
    assert lg == ls and torch.equal(trg.engine.P, trs.engine.P)
    assert ls[-1] < ls[0] - 0.1
    for a, b in zip(ls, ll):
        assert abs(a - b) <= 1e-2 * max(1.0, abs(b))
    e = trs.engine
    assert torch.equal(e.S, e.P.to(torch.bfloat16))


def _domain_cases():
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "domain.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _domain_cases(), ids=lambda c: c["name"])
@pytest.mark.parametrize("precision", ["bf16", "tf32", "strict_fp32", "strict_fp64"])
def test_domain_errors_match_reference(case, precision):
    """Extreme logits / pre-activations (tests/golden/domain.json, produced by
    the unmodified reference): where the reference raises -- OverflowError
    from math.exp (sigmoid activation, softmax exp, BCE head), EvalError
    wrapping DomainError from div (row sum 0) or log (p == 0, also when the
    row sum overflows) -- Trainer.gradient raises the same exception type and
    message; where it does not, the stable device loss matches its value and
    no error is raised (gradients compared where the reference's own are finite;
    where the reference's float64 pullback itself overflows -- s*s in div's
    adjoint, 1/p of a subnormal p -- the stable gradients are checked against
    the exact softmax-CE gradient instead)."""
    from paper_1811_01457_b200.fused import EvalError

    acts = tuple(case["acts"])
    (W0, b0), (W1, b1) = [(np.array(w, dtype=np.float64), np.array(b, dtype=np.float64)) for w, b in case["params"]]
    chain = Chain(Dense(W0.shape[1], W0.shape[0], acts[0], W0, b0), Dense(W1.shape[1], W1.shape[0], acts[1], W1, b1))
    X = np.array(case["X"])
    Y = np.array(case["Y"])
    n = X.shape[0]
    tr = Trainer(chain, n, loss=case["loss_kind"], precision=precision)
    dt = torch.float64 if precision == "strict_fp64" else torch.float32
    Xd, Yd = torch.from_numpy(X).to(dt).cuda(), torch.from_numpy(Y).to(dt).cuda()
    if case["raises"] == "OverflowError":
        with pytest.raises(OverflowError, match="^math range error$"):
            tr.gradient(Xd, Yd)
    elif case["raises"] == "EvalError":
        with pytest.raises(EvalError) as ei:
            tr.gradient(Xd, Yd)
        assert ei.value.message == case["message"]
        assert type(ei.value.__cause__).__name__ == case["cause"] == "DomainError"
    else:
        lv, grads = tr.gradient(Xd, Yd)
        tol = TOL[precision]
        # log of a subnormal p keeps fewer than 53 bits in the reference (its
        # loss is off by up to ~1e-5 relative); the stable z - lse is exact
        ltol = max(tol, 1e-5) if case["p_subnormal"] else tol
        assert abs(lv - case["loss"]) <= ltol * max(1.0, abs(case["loss"]))
        for (gW, gb), (rW, rb) in zip(grads, case["grads"]):
            assert np.isfinite(gW).all() and np.isfinite(gb).all()
            if not case["pullback_overflow"]:
                assert nrel(gW, np.array(rW)) <= tol and nrel(gb, np.array(rb)) <= tol
        if case["pullback_overflow"]:
            # the reference's float64 pullback overflowed (s*s in div's adjoint,
            # 1/p of a subnormal p), so its gradients are not the derivative:
            # check the stable ones against the exact softmax-CE gradient instead
            _, go, _ = OD.mlp_step([(W0, b0), (W1, b1)], X, Y, acts, case["loss_kind"], mode="blas")
            for (gW, gb), (oW, ob) in zip(grads, go):
                assert nrel(gW, oW) <= tol and nrel(gb, ob) <= tol
    tr.check()  # the flags were consumed by the raise: a clean state for the next step
    # the one-launch small step (softmax heads, tensor-core precisions) flags the same conditions
    if tr.engine.small is not None and case["loss_kind"] == "softmax_xent":
        tr.step(Xd, Yd)
        if case["raises"] == "OverflowError":
            with pytest.raises(OverflowError):
                tr.check()
        elif case["raises"] == "EvalError":
            with pytest.raises(EvalError, match=case["message"]):
                tr.check()
        else:
            tr.check()


@pytest.mark.parametrize("knobs", [
    {"SGB200_GEMM_SPLIT_FIXUP": "1"}, {"SGB200_DENSE_FUSED_DB": "1"}, {"SGB200_GEMM_WIDE": "1"},
])
def test_opt_in_gemm_variants_are_bit_identical(knobs):
    """The opt-in kernel variants -- in-kernel split-K fix-up, bias-gradient
    finalize fused into the dW GEMM, wide epilogue slots -- compute the same
    tiles in the same order: a training step is bit-identical to the default
    path.  (Run in a subprocess: the knobs are read once per process.)"""
    import os
    import subprocess
    import sys

    code = """
import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1811_01457_b200.dense import Chain, ChainEngine, Dense
rng = np.random.default_rng(2)
sizes, acts, B = (512, 768, 512, 256), ('tanh', 'sigmoid', 'identity'), 2048
chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(3)]).init_params(rng)
e = ChainEngine(chain, B, 'mse', 'bf16', small=False)
X = torch.from_numpy(rng.uniform(0, 1, (B, sizes[0])).astype(np.float32)).cuda()
Y = torch.from_numpy(rng.uniform(-1, 1, (B, sizes[-1])).astype(np.float32)).cuda()
e.load_batch(X, Y); e.forward(); e.loss_and_seed(); e.pullback()
torch.cuda.synchronize()
np.save(sys.argv[1], np.concatenate([e.G.double().cpu().numpy(), e.loss.cpu().numpy()]))
"""
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        outs = []
        for env in ({}, knobs):
            f = os.path.join(d, f"g{len(outs)}.npy")
            subprocess.run([sys.executable, "-c", code, f], check=True, env={**os.environ, **env},
                           cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
            outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
@pytest.mark.parametrize("M,D", [(8192, 4096), (1000, 520), (777, 522), (100, 72), (200, 40)])
def test_value_and_pullback_fuses_the_seed(M, D, precision):
    """DenseLayer.value_and_pullback (the forward GEMM's epilogue also forms
    dZ = ybar .* act'(H) and its column sums) against the same layer's
    forward + separate act' + pullback and an fp64 evaluation: c3 at full size
    and a ragged shape."""
    g = torch.Generator(device="cuda").manual_seed(M)
    W = ((torch.rand((D, D), generator=g, device="cuda") * 2 - 1) * (6.0 / (2 * D)) ** 0.5)
    b = (torch.rand(D, generator=g, device="cuda") * 2 - 1) * 0.01
    X = (torch.rand((M, D), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    ybar = torch.rand((M, D), generator=g, device="cuda") * 2 - 1
    outs = []
    for fused in (False, True):
        layer = DenseLayer(M, D, D, "sigmoid", precision=precision)
        layer.set_params(W.cpu().numpy(), b.cpu().numpy())
        if fused:
            H, dX, dW, db = layer.value_and_pullback(ybar, X)
        else:
            H = layer.forward(X)
            dX, dW, db = layer.pullback(ybar)
        torch.cuda.synchronize()
        outs.append((H.clone(), layer.dZ.clone(), dX.clone(), dW.clone(), db.clone()))
    (H0, Z0, X0, W0, b0), (H1, Z1, X1, W1, b1) = outs
    assert torch.equal(H0, H1)
    assert torch.equal(Z0, Z1)  # dZ from the same bf16 H: identical values
    x64, w64 = X.double(), layer.Wb.double()
    s = torch.sigmoid(x64 @ w64.T + b.double())
    dz = ybar.double() * s * (1 - s)

    def nrel_t(u, v):
        return float((u.double() - v).abs().max() / v.abs().max())

    assert nrel_t(X1, dz @ w64) <= 1e-2
    assert nrel_t(W1, dz.T @ x64) <= 1e-2
    assert nrel_t(b1, dz.sum(0)) <= 1e-2
    assert nrel_t(b1, b0.double()) <= 1e-5  # db: partial sums in another order only


@pytest.mark.parametrize("sizes,B", [((512, 768, 256), 2048), ((300, 200, 10), 1000), ((64, 96, 33), 70)])
def test_fused_mse_loss_matches_separate_loss_kernel(sizes, B):
    """forward(fuse_loss=True) (the MSE loss and its seed dz formed in the
    top GEMM's epilogue, SG_EPI_BIAS_MSE) against forward() + the separate
    loss kernel on the same engine and batch: dz is the same arithmetic on the
    same fp32 z (bit-identical), the loss differs only in its summation order
    (f64 partials), the bias gradient in the order of its per-32-row column
    sums.  Ragged widths and batches included."""
    rng = np.random.default_rng(B)
    L = len(sizes) - 1
    chain = Chain(*[Dense(sizes[i], sizes[i + 1], "tanh" if i < L - 1 else "identity")
                    for i in range(L)]).init_params(rng)
    e = ChainEngine(chain, B, "mse", "bf16", small=False)
    assert e.fused_mse
    X = torch.from_numpy(rng.uniform(0, 1, (B, sizes[0])).astype(np.float32)).cuda()
    Y = torch.from_numpy(rng.uniform(-1, 1, (B, sizes[-1])).astype(np.float32)).cuda()
    outs = []
    for fuse in (False, True):
        e.G.zero_()
        e.load_batch(X, Y)
        z = e.forward(fuse_loss=fuse)
        assert (z is None) == fuse
        e.loss_and_seed()
        dz = e.dz_of(L - 1).clone()
        e.pullback()
        torch.cuda.synchronize()
        outs.append((float(e.loss.item()), dz, e.G.clone(), [g.clone() for g in e.gb]))
    (l0, dz0, G0, gb0), (l1, dz1, G1, gb1) = outs
    assert torch.equal(dz0, dz1)
    assert abs(l1 - l0) <= 1e-6 * abs(l0)  # fp32 sums of 8 squares, fp64 beyond: summation order only
    if sizes[-1] % 8 == 0:  # k_mse_v8 folds its loss partials exactly like the epilogue
        assert l1 == l0
    for a, b in zip(gb0, gb1):
        assert float((a - b).abs().max()) <= 1e-5 * max(1e-30, float(a.abs().max()))
    # the weight gradients only see dz: identical
    for l in range(L):
        wo, bo = e.seg[l]
        assert torch.equal(G0[wo:bo], G1[wo:bo])


@pytest.mark.parametrize("sizes", [(256, 384, 256, 128), (300, 333, 130, 72), (96, 48, 40, 24)])
def test_deferred_splitk_is_bit_identical(sizes):
    """Deferred split-K (a dW GEMM's partials left in its own buffer, every
    layer's reduced in one sg_splitk_reduce_multi launch after the pullback)
    against the per-GEMM reduce: identical dW and db, and the split actually
    happens for these narrow layers (K = batch >> M = N); ragged widths too."""
    import os

    from paper_1811_01457_b200.gemm import gemm, gemm_splits, gemm_desc, splitk_reduce

    rng = np.random.default_rng(11)
    acts, B = ("tanh", "tanh", "identity"), 16384
    chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(3)]).init_params(rng)
    X = torch.from_numpy(rng.uniform(0, 1, (B, sizes[0])).astype(np.float32)).cuda()
    Y = torch.from_numpy(rng.uniform(-1, 1, (B, sizes[-1])).astype(np.float32)).cuda()
    grads = []
    for defer in ("0", "1"):
        os.environ["SGB200_DEFER_SPLITK"] = defer
        try:
            e = ChainEngine(chain, B, "mse", "bf16", small=False)
            e._dw_split_plan()  # planned while the knob is set
        finally:
            del os.environ["SGB200_DEFER_SPLITK"]
        e.load_batch(X, Y)
        e.forward(fuse_loss=True)
        e.loss_and_seed()
        e.pullback()
        torch.cuda.synchronize()
        assert (sum(sp is not None for sp in e.dw_split) > 0) == (defer == "1")
        grads.append(e.G.clone())
    assert torch.equal(grads[0], grads[1])
    # the binding alone: partials + one multi-job reduce == the GEMM's own reduce
    A = (torch.rand((B, 320), device="cuda") - 0.5).to(torch.bfloat16)
    Bm = (torch.rand((B, 192), device="cuda") - 0.5).to(torch.bfloat16)
    ref = torch.empty((320, 192), device="cuda")
    gemm(A, Bm, a_mn=True, b_mn=True, out=ref)
    splits, ld = gemm_splits(gemm_desc(A, Bm, a_mn=True, b_mn=True, out=ref))
    assert splits > 1
    part = torch.empty(splits * 320 * ld, device="cuda")
    out = torch.full((320, 192), float("nan"), device="cuda")
    gemm(A, Bm, a_mn=True, b_mn=True, out=out, split_part=part)
    splitk_reduce([(part, splits, 320, 192, ld, out)])
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    with pytest.raises(Exception):
        gemm(A, Bm, a_mn=True, b_mn=True, out=out, split_part=part[:10])


def _bf16(x):
    """Round to bfloat16 (nearest even), back to float64."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32).astype(np.float64)


@pytest.mark.parametrize("B", [1, 3])
def test_tiny_batches_bf16_layer_path_matches_bf16_arithmetic(B):
    """One and three rows through the bf16 layer-by-layer path (a layer too
    wide for the one-launch step): the 1-SM GEMM kernels at M = 1 / 3 and
    the memory-bound kernels' tail blocks, against a numpy restatement that
    rounds exactly where the bf16 path stores (X, W, the activations, the
    seeds dz the GEMMs read; the bias gradients sum the fp32 seeds) and
    accumulates in fp64.  With U(-1, 1) targets the MSE seed
    z - y of a single row cancels most of z's digits: against pure fp64 the
    bf16 path is 9 % off on dW here -- and so is this restatement, so the
    kernels are checked against the arithmetic they implement (1e-3)."""
    rng = np.random.default_rng(40 + B)
    sizes = (33, 1100, 7)
    chain = Chain(Dense(33, 1100, "relu"), Dense(1100, 7, "identity")).init_params(rng)
    for l in chain.layers:
        l.b = rng.uniform(-0.1, 0.1, l.fan_out).astype(np.float32)
    X = rng.uniform(0, 1, (B, 33)).astype(np.float32)
    Y = rng.uniform(-1, 1, (B, 7)).astype(np.float32)
    tr = Trainer(chain, B, loss="mse", precision="bf16")
    assert tr.engine.small is None
    lv, ((gW0, gb0), (gW1, gb1)) = tr.gradient(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda())
    (W0, b0), (W1, b1) = [(l.W.astype(np.float64), l.b.astype(np.float64)) for l in chain.layers]
    x, w0, w1 = _bf16(X), _bf16(W0), _bf16(W1)
    z0 = x @ w0.T + b0
    h1 = _bf16(np.maximum(z0, 0.0))
    z = h1 @ w1.T + b1
    d = z - Y
    dzf = 2.0 * d / B                      # the seed in fp32: its column sums are db (epilogue)
    dz = _bf16(dzf)                        # stored bf16: what the dW / dX GEMMs read
    dz0f = (dz @ w1) * (z0 > 0)
    dz0 = _bf16(dz0f)
    want = {"loss": float((d * d).sum() / B), "gW1": dz.T @ h1, "gb1": dzf.sum(0), "gW0": dz0.T @ x,
            "gb0": dz0f.sum(0)}
    assert abs(lv - want["loss"]) <= 1e-3 * max(1.0, abs(want["loss"]))
    for name, got in (("gW1", gW1), ("gb1", gb1), ("gW0", gW0), ("gb0", gb0)):
        assert nrel(got, want[name]) <= 1e-3, name


@pytest.mark.parametrize("sizes,acts,loss,B", [
    ((33, 1100, 7), ("relu", "identity"), "mse", 1),
    ((33, 1100, 7), ("relu", "identity"), "mse", 3),
    ((40, 24, 24, 24, 24, 24, 3), ("tanh",) * 5 + ("identity",), "softmax_xent", 3),
])
def test_tiny_batches_tf32_layer_path_vs_oracle(sizes, acts, loss, B):
    """The same tiny batches in TF32 (fp32 activations) against the fp64
    oracle, at the north star's 1e-2: with one to three rows nothing
    averages the operands' 2^-11 roundings over six layers."""
    rng = np.random.default_rng(B + len(sizes))
    chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(len(acts))]).init_params(rng)
    for l in chain.layers:
        l.b = rng.uniform(-0.1, 0.1, l.fan_out).astype(np.float32)
    X = rng.uniform(0, 1, (B, sizes[0])).astype(np.float32)
    if loss == "softmax_xent":
        Y = np.zeros((B, sizes[-1]), np.float32)
        Y[np.arange(B), rng.integers(0, sizes[-1], B)] = 1
    else:
        Y = rng.uniform(-1, 1, (B, sizes[-1])).astype(np.float32)
    tr = Trainer(chain, B, loss=loss, precision="tf32")
    assert tr.engine.small is None  # the layer-by-layer path
    lv, grads = tr.gradient(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda())
    params = [(l.W.astype(np.float64), l.b.astype(np.float64)) for l in chain.layers]
    lo, go, _ = OD.mlp_step(params, X.astype(np.float64), Y.astype(np.float64), acts, loss, mode="blas")
    assert abs(lv - lo) <= 1e-2 * max(1.0, abs(lo))
    for (gW, gb), (oW, ob) in zip(grads, go):
        assert nrel(gW, oW) <= 1e-2
        assert nrel(gb, ob) <= 1e-2


def test_trainer_accepts_batch_dtypes_and_layouts():
    """Trainer.step on the same batch given as fp32, fp64 and bf16-exact
    values, with Y contiguous, row-padded (a strided slice) or fp64: the
    minibatch load casts with sg_cast_2d and the loss reads unit-stride rows
    in place, so every form trains to the same bits; host tensors are refused
    with a ValueError (no silent copy inside a captured step)."""
    rng = np.random.default_rng(21)
    sizes, acts, B = (64, 96, 48), ("tanh", "identity"), 640
    Xb = torch.from_numpy(rng.uniform(0, 1, (B, 64)).astype(np.float32)).to(torch.bfloat16).float().cuda()
    Y = torch.from_numpy(rng.uniform(-1, 1, (B, 48)).astype(np.float32)).cuda()
    Ypad = torch.zeros((B, 56), device="cuda")
    Ypad[:, :48] = Y
    variants = {"f32": (Xb, Y), "f64": (Xb.double(), Y.double()), "bf16 X": (Xb.to(torch.bfloat16), Y),
                "padded Y": (Xb, Ypad[:, :48])}
    out = {}
    for name, (X, Yv) in variants.items():
        chain = Chain(Dense(64, 96, "tanh"), Dense(96, 48, "identity")).init_params(np.random.default_rng(2))
        tr = Trainer(chain, B, loss="mse", lr=1e-2, precision="bf16", small=False)
        losses = [float(tr.step(X, Yv).item()) for _ in range(3)]
        out[name] = (losses, tr.engine.P.clone())
    ref = out["f32"]
    for name, (losses, P) in out.items():
        assert losses == ref[0], name
        assert torch.equal(P, ref[1]), name
    chain = Chain(Dense(64, 96, "tanh"), Dense(96, 48, "identity")).init_params(np.random.default_rng(2))
    tr = Trainer(chain, B, loss="mse", precision="bf16", small=False)
    with pytest.raises(ValueError, match="device tensor"):
        tr.step(Xb.cpu(), Y)


def test_graph_replay_with_alternating_batches():
    """A loader that alternates two minibatch buffers: each (X, Y) pair is
    captured on its second step (not only on back-to-back repeats) and
    replayed after; the losses and parameters equal the eager run's bit for bit."""
    rng = np.random.default_rng(17)
    sizes, acts, B = (128, 256, 64), ("tanh", "identity"), 512
    pairs = [(torch.from_numpy(rng.uniform(0, 1, (B, 128)).astype(np.float32)).cuda(),
              torch.from_numpy(rng.uniform(-1, 1, (B, 64)).astype(np.float32)).cuda()) for _ in range(2)]
    runs = {}
    for graph in (False, True):
        chain = Chain(Dense(128, 256, "tanh"), Dense(256, 64, "identity")).init_params(np.random.default_rng(3))
        tr = Trainer(chain, B, loss="mse", lr=1e-2, precision="bf16", graph=graph, small=False)
        losses = [float(tr.step(*pairs[i % 2]).item()) for i in range(8)]
        runs[graph] = (losses, tr.engine.P.clone(), len(tr._graphs))
    assert runs[True][2] == 2  # both pairs captured
    assert runs[False][0] == runs[True][0]
    assert torch.equal(runs[False][1], runs[True][1])


@pytest.mark.parametrize("N", [1, 2, 127, 128, 129, 1000, 1024])
@pytest.mark.parametrize("precision", ["tf32", "strict_fp64"])
def test_softmax_xent_class_counts(N, precision):
    """The softmax cross-entropy loss kernel across its two layouts (rows of
    <= 128 classes per warp group, wider rows per block) and their edges, up
    to its 1024-class limit: loss and gradients against the oracle; 1025
    classes are refused with a ValueError."""
    rng = np.random.default_rng(N)
    B = 300
    chain = Chain(Dense(16, N, "identity")).init_params(rng)
    chain.layers[0].b = rng.uniform(-0.5, 0.5, N).astype(np.float32)
    X = rng.uniform(-1, 1, (B, 16)).astype(np.float32)
    Y = np.zeros((B, N), np.float32)
    Y[np.arange(B), rng.integers(0, N, B)] = 1
    tr = Trainer(chain, B, loss="softmax_xent", precision=precision, small=False)
    lv, ((gW, gb),) = tr.gradient(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda())
    params = [(chain.layers[0].W.astype(np.float64), chain.layers[0].b.astype(np.float64))]
    lo, ((oW, ob),), _ = OD.mlp_step(params, X.astype(np.float64), Y.astype(np.float64), ("identity",),
                                     "softmax_xent", mode="blas")
    tol = TOL[precision]
    assert abs(lv - lo) <= tol * max(1.0, abs(lo))
    assert nrel(gW, oW) <= tol and nrel(gb, ob) <= tol


def test_softmax_xent_refuses_too_many_classes():
    chain = Chain(Dense(16, 1025, "identity")).init_params(np.random.default_rng(0))
    tr = Trainer(chain, 64, loss="softmax_xent", precision="tf32", small=False)
    X = torch.zeros((64, 16), device="cuda")
    Y = torch.zeros((64, 1025), device="cuda")
    with pytest.raises(ValueError, match="1024 classes"):
        tr.gradient(X, Y)


@pytest.mark.parametrize("M,N,K", [(2048, 1024, 512), (1000, 520, 200), (100, 72, 64)])
def test_tf32_seeded_forward_matches_separate_act_grad(M, N, K):
    """TF32 BIAS_ACT_SEED (h and dz = seed .* act'(h) in fp32 from one GEMM
    epilogue, with the bias-gradient partials) against the TF32 forward plus
    the separate sg_act_grad kernel: h and dz bit-identical (the same fp32
    arithmetic), the column sums equal up to their summation order."""
    from paper_1811_01457_b200 import runtime as rt
    from paper_1811_01457_b200.dense import ACT, _dt, _lib, _p
    from paper_1811_01457_b200.gemm import gemm

    g = torch.Generator(device="cuda").manual_seed(M + N)
    X = torch.rand((M, K), generator=g, device="cuda") * 2 - 1
    W = (torch.rand((N, K), generator=g, device="cuda") * 2 - 1) * K ** -0.5
    b = (torch.rand(N, generator=g, device="cuda") * 2 - 1) * 0.1
    seed = torch.rand((M, N), generator=g, device="cuda") * 2 - 1
    G = (M + 31) // 32
    h1, dz1, cs1 = torch.empty((M, N), device="cuda"), torch.empty((M, N), device="cuda"), torch.zeros((G, N), device="cuda")
    gemm(X, W, precision="tf32", epilogue="bias_act_seed", act="sigmoid", bias=b, seed=seed, out=h1, out2_lp=dz1,
         colsum=cs1)
    h0, dz0, cs0 = torch.empty_like(h1), torch.empty_like(dz1), torch.zeros_like(cs1)
    gemm(X, W, precision="tf32", epilogue="bias_act", act="sigmoid", bias=b, out=h0)
    lib = _lib()
    rt.check(lib.sg_act_grad(rt.context(), _p(seed), _dt(seed), seed.stride(0), _p(h0), _dt(h0), h0.stride(0), M, N,
                             ACT["sigmoid"], _p(dz0), _dt(dz0), dz0.stride(0), None, 0, 0, _p(cs0), cs0.stride(0),
                             rt.stream_ptr()), "sg_act_grad")
    torch.cuda.synchronize()
    assert torch.equal(h1, h0)
    assert torch.equal(dz1, dz0)
    assert float((cs1.double().sum(0) - cs0.double().sum(0)).abs().max()) <= 1e-5 * float(cs0.abs().sum(0).max())


def test_repeated_steps_and_split_gemms_do_not_grow_device_memory():
    """Training steps (eager and graph-replayed) and split-K GEMMs with their
    stream-ordered partial buffers: device memory stays flat over many calls."""
    from paper_1811_01457_b200.gemm import gemm

    rng = np.random.default_rng(4)
    B = 4096
    X = torch.from_numpy(rng.uniform(0, 1, (B, 256)).astype(np.float32)).cuda()
    Y = torch.from_numpy(rng.uniform(-1, 1, (B, 128)).astype(np.float32)).cuda()
    trs = [Trainer(Chain(Dense(256, 384, "tanh"), Dense(384, 128, "identity")).init_params(np.random.default_rng(1)),
                   B, loss="mse", lr=1e-3, precision="bf16", graph=g, small=False) for g in (False, True)]
    A = (torch.rand((16384, 256), device="cuda") - 0.5).to(torch.bfloat16)
    out = torch.empty((256, 256), device="cuda")

    def run():
        for tr in trs:
            tr.step(X, Y)
        gemm(A, A, a_mn=True, b_mn=True, out=out)  # K = 16384 over 1 tile: split-K with its own partials

    for _ in range(5):
        run()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(100):
        run()
    torch.cuda.synchronize()
    assert free0 - torch.cuda.mem_get_info()[0] <= 8 << 20
