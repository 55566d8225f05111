"""Persistent GEMM chains (sg_chain_*) against the layer-by-layer path.

A chain runs the same GEMMs -- the same 256 x 256 pair tiles, k order,
fused epilogues and split-K summation order -- as issuing them one by one,
only in one persistent launch with row-block dependencies between them, so
the results must be BIT-identical:
* GemmChain of GEMMs with "rows", "krows" and "all" dependencies vs the same
  gemm() calls in stream order;
* a Dense chain's forward + loss + pullback (chained) vs the per-layer path,
  for widths and batches that are and are not multiples of the 256-row tile;
* a CUDA-graph training run: every step's loss and the final parameters.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1811_01457_b200.dense import Chain, ChainEngine, Dense, _pair_splits  # noqa: E402
from paper_1811_01457_b200.gemm import GemmChain, gemm, gemm_desc  # noqa: E402
from paper_1811_01457_b200.train import Trainer  # noqa: E402

bf = torch.bfloat16


def _t(rows, cols, scale, g, dtype=bf):
    ld = (cols + 7) // 8 * 8
    buf = torch.zeros((rows, ld), dtype=dtype, device="cuda")
    buf[:, :cols] = ((torch.rand((rows, cols), generator=g, device="cuda") * 2 - 1) * scale).to(dtype)
    return buf[:, :cols]


@pytest.mark.parametrize("M,D", [(1024, 512), (1000, 300), (2048, 1024)])
def test_gemm_chain_dependencies_match_sequential_gemms(M, D):
    """x1 = tanh(x0 W0^T + b)  ->  x2 = sigmoid(x1 W1^T)  (rows on 0)
    -> dW-like x1^T x2 split-K (krows on 1) -> x3 = x2 W1 (all on 1)."""
    g = torch.Generator(device="cuda").manual_seed(M + D)
    x0, W0, W1 = _t(M, D, 1.0, g), _t(D, D, 0.05, g), _t(D, D, 0.05, g)
    b = (torch.rand(D, generator=g, device="cuda") - 0.5) * 0.1
    outs = {}
    for mode in ("seq", "chain"):
        x1, x2 = _t(M, D, 0.0, g), _t(M, D, 0.0, g)
        gw = torch.zeros((D, D), device="cuda")
        x3 = torch.zeros((M, D), device="cuda")
        cs = torch.zeros(((M + 31) // 32, D), device="cuda")
        specs = [
            (dict(A=x0, B=W0, epilogue="bias_act", act="tanh", bias=b, out_lp=x1), 1, []),
            (dict(A=x1, B=W1, epilogue="bias_act", act="sigmoid", out_lp=x2, colsum=cs), 1, [("rows", 0)]),
            (dict(A=x1, B=x2, a_mn=True, b_mn=True, out=gw), _pair_splits(D, D, M, 74), [("krows", 1)]),
            (dict(A=x2, B=W1, b_mn=True, out=x3), _pair_splits(M, D, D, 74), [("all", 1)]),
        ]
        if mode == "seq":
            for kw, _, _ in specs:
                A, B = kw.pop("A"), kw.pop("B")
                gemm(A, B, **kw)
        else:
            ch = GemmChain([(gemm_desc(kw.pop("A"), kw.pop("B"), **kw), s, deps) for kw, s, deps in specs])
            ch.run()
            ch.run()  # replays: counters are reset in-kernel between launches
        torch.cuda.synchronize()
        outs[mode] = [x1.clone(), x2.clone(), gw.clone(), x3.clone(), cs.clone()]
        if mode == "chain":
            ch.close()
    for k, (a, c) in enumerate(zip(outs["seq"], outs["chain"])):
        assert torch.equal(a, c), k


@pytest.mark.parametrize("sizes,acts,B", [
    ((512, 512, 384, 300), ("tanh", "sigmoid", "identity"), 1024),
    ((300, 520, 264, 72), ("relu", "tanh", "identity"), 1000),       # ragged widths and batch
    ((1024,) * 6, ("tanh",) * 4 + ("identity",), 2048),
])
def test_chained_step_is_bit_identical_to_layer_path(sizes, acts, B):
    rng = np.random.default_rng(B)
    chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(len(acts))]).init_params(rng)
    for l in chain.layers:
        l.b = rng.uniform(-0.1, 0.1, l.fan_out).astype(np.float32)
    X = torch.from_numpy(rng.uniform(0, 1, (B, sizes[0])).astype(np.float32)).cuda()
    Y = torch.from_numpy(rng.uniform(-1, 1, (B, sizes[-1])).astype(np.float32)).cuda()
    res = {}
    for use in (False, "full", "pairwise"):
        e = ChainEngine(chain, B, "mse", "bf16", small=False, gemm_chain=use)
        for _ in range(2):  # twice: the chain replays from reset counters
            e.load_batch(X, Y)
            e.forward()
            e.loss_and_seed()
            e.pullback()
        torch.cuda.synchronize()
        assert (e.chains is not None) == bool(use)
        res[use] = (e.loss.clone(), e.G.clone(), e.Zt.clone(), [h.clone() for h in e.H])
    l0, g0, z0, h0 = res[False]
    for mode in ("full", "pairwise"):
        l1, g1, z1, h1 = res[mode]
        assert torch.equal(z0, z1), mode
        assert all(torch.equal(a, b) for a, b in zip(h0, h1)), mode
        assert torch.equal(l0, l1), mode
        assert torch.equal(g0, g1), mode


def test_chained_training_run_matches_layer_path():
    """CUDA-graph training (minibatch load, chained forward, loss, chained
    pullback, batched bias-gradient finalize, SGD): identical losses and
    parameters to the per-layer path, step by step.  Both arms take the
    separate loss kernel (SGB200_FUSED_LOSS=0): the chained forward has no
    loss-fused epilogue, and the fused one sums the bias-gradient partials in
    another order (tests/test_dense_gpu.py::test_fused_mse_loss_matches_separate_loss_kernel)."""
    rng = np.random.default_rng(3)
    sizes, acts, B = (512,) * 5, ("tanh",) * 3 + ("identity",), 2048
    X = torch.from_numpy(rng.uniform(0, 1, (B, sizes[0])).astype(np.float32)).cuda()
    Y = torch.from_numpy(rng.uniform(-1, 1, (B, sizes[-1])).astype(np.float32)).cuda()
    runs = {}
    for use in (False, True):
        import os

        os.environ["SGB200_CHAIN"] = "1" if use else "0"
        os.environ["SGB200_FUSED_LOSS"] = "0"
        try:
            chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(4)]).init_params(
                np.random.default_rng(1))
            tr = Trainer(chain, B, loss="mse", lr=1e-3, precision="bf16", graph=True)
            assert tr.engine.chainable == use  # SGB200_CHAIN=1 opts in
            losses = [float(tr.step(X, Y).item()) for _ in range(6)]
            runs[use] = (losses, tr.engine.P.clone())
        finally:
            del os.environ["SGB200_CHAIN"]
            del os.environ["SGB200_FUSED_LOSS"]
    assert runs[False][0] == runs[True][0]
    assert torch.equal(runs[False][1], runs[True][1])
    assert runs[True][0][-1] < runs[True][0][0]


def test_forward_chain_mode_matches_layer_path():
    """SGB200_CHAIN=3: the forward GEMMs below the top layer as ONE chain, the
    top layer (fused MSE) and the pullback layer by layer -- the same kernels'
    arithmetic, so losses and parameters equal the per-layer path's."""
    import os

    rng = np.random.default_rng(5)
    sizes, acts, B = (384, 512, 512, 640, 256), ("tanh", "relu", "tanh", "identity"), 3000
    X = torch.from_numpy(rng.uniform(0, 1, (B, sizes[0])).astype(np.float32)).cuda()
    Y = torch.from_numpy(rng.uniform(-1, 1, (B, sizes[-1])).astype(np.float32)).cuda()
    runs = {}
    for mode in ("0", "3"):
        os.environ["SGB200_CHAIN"] = mode
        try:
            chain = Chain(*[Dense(sizes[i], sizes[i + 1], acts[i]) for i in range(4)]).init_params(
                np.random.default_rng(1))
            tr = Trainer(chain, B, loss="mse", lr=1e-3, precision="bf16", graph=True)
            assert tr.engine.chain_mode == (None if mode == "0" else "forward")
            losses = [float(tr.step(X, Y).item()) for _ in range(5)]
            runs[mode] = (losses, tr.engine.P.clone())
        finally:
            del os.environ["SGB200_CHAIN"]
    assert runs["0"][0] == runs["3"][0]
    assert torch.equal(runs["0"][1], runs["3"][1])
