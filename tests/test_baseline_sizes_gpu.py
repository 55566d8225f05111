"""Parity of the BASELINE training-step configurations at their full sizes
and at their 8-GPU shard sizes (BASELINE.json configs[3], configs[4]).

c4: 4 x Dense 4096 (tanh, tanh, tanh, identity), MSE, batch 65536;
    8-GPU shard: batch 8192 of the global 65536 (loss scaled by the global
    1/B) with layer 0's dW in 4 row slices, as the data-parallel engine runs it.
c5: 16 x Dense 1024 (15 tanh, identity), MSE, batch 32768; shard: 4096.

The bf16 tensor-core step (tcgen05 GEMMs, fused epilogues, fused loss) is
compared against a float64 restatement of the reference's Dense IR and its
pullback evaluated on the device with torch (test-side only):
z = h . W^T + b (tensor.py:351-361, 179-182), tanh (tensor.py:245-250),
MSE = sum((z - y)^2) / n, and the adjoints of rules.py:45-46 (add ->
reduce_like column sums), 82-84 (tanh), 113-115 (matmul), 123-124
(transpose).  The reference's operands are the fp32 master weights and
inputs; the tensor cores see them rounded to bf16 and the activations are
stored in bf16, so the tolerance is north_star's BF16 bound: <= 1e-2
relative to each tensor's largest magnitude, on the loss and on every
layer's dW and db.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1811_01457_b200.dense import Chain, ChainEngine, Dense  # noqa: E402

TOL = 1e-2


def reference_step_fp64(Ws, bs, X, Y, acts, scale):
    """float64 loss and gradients of the reference's MSE Dense-chain IR (device, torch)."""
    hs = [X.double()]
    for W, b, act in zip(Ws, bs, acts):
        zb = hs[-1] @ W.double().T + b.double()
        hs.append(torch.tanh(zb) if act == "tanh" else zb)
    d = hs[-1] - Y.double()
    loss = float((d * d).sum() * scale)
    gbar = d * scale + d * scale  # rules.py:53-58 on mul(d, d)
    grads = [None] * len(Ws)
    for l in range(len(Ws) - 1, -1, -1):
        dz = gbar * (1.0 - hs[l + 1] * hs[l + 1]) if acts[l] == "tanh" else gbar
        grads[l] = (dz.T @ hs[l], dz.sum(0))
        if l > 0:
            gbar = dz @ Ws[l].double()
        del dz
    return loss, grads


def nrel(got, want):
    return float((got.double() - want).abs().max() / want.abs().max().clamp_min(1e-300))


def run_case(width, layers, batch, global_batch, slices, seed):
    sizes = (width,) * (layers + 1)
    acts = ("tanh",) * (layers - 1) + ("identity",)
    rng = np.random.default_rng(seed)
    chain = Chain(*[Dense(width, width, a) for a in acts]).init_params(rng)
    for l in chain.layers:  # nonzero biases so the bias path is exercised
        l.b = rng.uniform(-0.1, 0.1, width).astype(np.float32)
    eng = ChainEngine(chain, batch, "mse", "bf16", global_batch=global_batch)
    if slices > 1:
        assert eng.enable_first_layer_slices(slices, min_params=0)
    g = torch.Generator(device="cuda").manual_seed(seed)
    X = torch.rand((batch, width), generator=g, device="cuda")
    Y = torch.rand((batch, width), generator=g, device="cuda") * 2 - 1
    ready = []
    eng.grad_ready = ready.append
    eng.load_batch(X, Y)
    eng.forward()
    eng.loss_and_seed()
    eng.pullback()
    torch.cuda.synchronize()
    from paper_1811_01457_b200.dense import pullback_ready_order

    assert ready == pullback_ready_order(layers, slices)  # every bucket readied once, in the engine's order
    loss = float(eng.loss.item())
    Ws = [eng.W[l] for l in range(layers)]
    bs = [eng.b[l] for l in range(layers)]
    want_loss, want = reference_step_fp64(Ws, bs, X, Y, acts, 1.0 / global_batch)
    assert abs(loss - want_loss) <= TOL * abs(want_loss), (loss, want_loss)
    worst = 0.0
    for l, (gW, gb) in enumerate(want):
        eW, eb = nrel(eng.gW[l], gW), nrel(eng.gb[l], gb)
        worst = max(worst, eW, eb)
        assert eW <= TOL and eb <= TOL, (l, eW, eb)
    del want
    torch.cuda.empty_cache()
    return worst


@pytest.mark.parametrize("name,width,layers,batch,global_batch,slices", [
    ("c4", 4096, 4, 65536, 65536, 1),
    ("c4_shard8_sliced", 4096, 4, 8192, 65536, 4),
    ("c5", 1024, 16, 32768, 32768, 1),
    ("c5_shard8", 1024, 16, 4096, 32768, 1),
])
def test_baseline_step_parity_at_size(name, width, layers, batch, global_batch, slices):
    worst = run_case(width, layers, batch, global_batch, slices, seed=11)
    print(f"{name}: worst gradient nrel {worst:.2e}")
