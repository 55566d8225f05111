"""Small device cases with guard bands: out-of-bounds write checks without compute-sanitizer.

compute-sanitizer is closed on this GPU pool (it prints "compute-sanitizer is
closed on this pool ...": runs under it have left GPUs needing a reset), so
every output here lives inside a guarded allocation -- sentinel bands before
and after it and in the padding columns between its width and its row
stride -- and each case checks that no kernel wrote outside its tensor, that
the result is right (loose tolerance), and that a second run is bit-identical.

  python tools/sanitize_cases.py [case ...]

Cases: fused (K1 + K2 + pack of sigma(a*x+b)), gemm1 (1-SM tcgen05 tiles),
pair (CTA-pair tiles), splitk (pair split-K + reduce), tail (split tail with
TMA reduce-add), actgrad (ACT_GRAD epilogue with TMA-streamed aux + colsum),
small (the one-launch small-chain step with its grid barrier), chain (a
persistent GEMM chain with row / K-row dependencies and in-kernel split-K),
step (a Dense-chain training step, layer path), loss (fused losses).
Each case checks its result loosely so a silent corruption also shows.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1811_01457_b200 import fused as F  # noqa: E402
from paper_1811_01457_b200.dense import Chain, ChainEngine, Dense  # noqa: E402
from paper_1811_01457_b200.gemm import GemmChain, gemm, gemm_desc  # noqa: E402
from paper_1811_01457_b200.irtext import parse_ir  # noqa: E402
from paper_1811_01457_b200.train import Trainer  # noqa: E402

bf = torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
GUARDS = []
SENTINEL = {torch.float32: float("nan"), bf: float("nan"), torch.float64: float("nan")}


def guarded(rows, cols, dtype=torch.float32, ld=None, band=4096):
    """A [rows, cols] tensor of row stride ld (default: cols rounded up to 8, +8)
    inside sentinel bands; registered for check_guards()."""
    ld = ld or ((cols + 7) // 8 * 8 + 8)
    buf = torch.full((band + rows * ld + band,), 12345.0, dtype=dtype, device="cuda")
    body = buf[band:band + rows * ld].view(rows, ld)
    body[:, :cols].fill_(0)
    view = body[:, :cols]
    GUARDS.append((buf, band, rows, ld, cols))
    return view


def check_guards():
    for k, (buf, band, rows, ld, cols) in enumerate(GUARDS):
        sentinel = torch.tensor(12345.0, dtype=buf.dtype, device="cuda")
        what = f"guarded tensor #{k} ({rows} x {cols}, ld {ld}, {buf.dtype})"
        assert bool((buf[:band] == sentinel).all()), f"write before {what}"
        assert bool((buf[band + rows * ld:] == sentinel).all()), f"write after {what}"
        if ld > cols:
            pad = buf[band:band + rows * ld].view(rows, ld)[:, cols:]
            bad = (pad != sentinel).nonzero()
            assert len(bad) == 0, f"write into the row padding of {what}: {len(bad)} elements, first {bad[:4].tolist()}"
    GUARDS.clear()


def rnd(*shape, dtype=torch.float32, scale=1.0):
    return ((torch.rand(shape, generator=g, device="cuda") * 2 - 1) * scale).to(dtype)


def check_gemm(M, N, K, a_mn=False, b_mn=False):
    A = rnd(K, M, dtype=bf) if a_mn else rnd(M, K, dtype=bf)
    B = rnd(K, N, dtype=bf) if b_mn else rnd(N, K, dtype=bf)
    out = guarded(M, N)
    gemm(A, B, a_mn=a_mn, b_mn=b_mn, out=out)
    first = out.clone()
    gemm(A, B, a_mn=a_mn, b_mn=b_mn, out=out)
    assert torch.equal(first, out), "not deterministic"
    a = A.double().T if a_mn else A.double()
    b = B.double() if b_mn else B.double().T
    err = float((out.double() - a @ b).abs().max())
    assert err < 1e-2 * K ** 0.5, err


def case_fused():
    m = parse_ir("""
func @affsig(%a: f64, %x: f64, %b: f64) -> f64 {
^entry:
  %m = mul %a, %x
  %s = add %m, %b
  %y = sigmoid %s
  ret %y
}
""")
    x, a, b = rnd(64, 200), rnd(200), rnd(200)
    y = F.fused_map(m, "affsig", [a, x, b])
    yb = rnd(64, 200)
    F.fused_map_grad(m, "affsig", [a, x, b], yb)
    F.fused_map_with_partials(m, "affsig", [a, x, b])
    assert float((y - torch.sigmoid(a * x + b)).abs().max()) < 1e-5


def case_gemm1():
    check_gemm(200, 120, 136)
    check_gemm(130, 64, 72, b_mn=True)


def case_pair():
    check_gemm(520, 300, 200)
    check_gemm(512, 512, 256, a_mn=True, b_mn=True)


def case_splitk():
    check_gemm(256, 256, 8192, a_mn=True, b_mn=True)


def case_tail():
    check_gemm(4096, 4096, 512, a_mn=True, b_mn=True)  # 256 pair tiles: last wave split in K halves


def case_actgrad():
    M, N, K = 512, 384, 256
    dZ, W, H = rnd(M, N, dtype=bf), rnd(N, K, dtype=bf, scale=0.1), (torch.rand((M, K), device="cuda")).to(bf)
    lp = guarded(M, K, bf)
    cs = guarded((M + 31) // 32, K)
    gemm(dZ, W, b_mn=True, epilogue="act_grad", act="tanh", aux=H, out_lp=lp, colsum=cs)
    want = (dZ.double() @ W.double()) * (1 - H.double() ** 2)
    assert float((lp.double() - want).abs().max()) < 5e-2


def case_small():
    chain = Chain(Dense(784, 32, "sigmoid"), Dense(32, 10, "identity")).init_params(np.random.default_rng(0))
    tr = Trainer(chain, 128, loss="softmax_xent", lr=0.05)
    assert tr.engine.small is not None
    X = torch.rand((128, 784), device="cuda")
    Y = torch.zeros((128, 10), device="cuda")
    Y[torch.arange(128), torch.randint(0, 10, (128,), device="cuda")] = 1
    for _ in range(3):
        tr.step(X, Y)
    tr.check()


def case_chain():
    M, D = 1000, 300
    x0, W0, W1 = guarded(M, D, bf), guarded(D, D, bf), guarded(D, D, bf)
    x0.copy_(rnd(M, D, dtype=bf))
    W0.copy_(rnd(D, D, dtype=bf, scale=0.05))
    W1.copy_(rnd(D, D, dtype=bf, scale=0.05))
    x1, x2 = guarded(M, D, bf), guarded(M, D, bf)
    gw = guarded(D, D)
    ch = GemmChain([
        (gemm_desc(x0, W0, epilogue="bias_act", act="tanh", out_lp=x1), 1, []),
        (gemm_desc(x1, W1, epilogue="bias_act", act="sigmoid", out_lp=x2), 1, [("rows", 0)]),
        (gemm_desc(x1, x2, a_mn=True, b_mn=True, out=gw), 4, [("krows", 1)]),
    ])
    ch.run()
    ch.run()
    torch.cuda.synchronize()
    want = x1.double().T @ x2.double()
    assert float((gw.double() - want).abs().max()) < 1e-2 * M ** 0.5
    ch.close()


def case_step():
    for use_chain in (False, True):
        chain = Chain(*[Dense(256, 256, "tanh"), Dense(256, 512, "relu"), Dense(512, 64, "identity")]).init_params(
            np.random.default_rng(1))
        e = ChainEngine(chain, 520, "mse", "bf16", small=False, gemm_chain=use_chain)
        e.load_batch(torch.rand((520, 256), device="cuda"), torch.rand((520, 64), device="cuda"))
        e.forward()
        e.loss_and_seed()
        e.pullback()
        e.sgd(0.01)


def case_loss():
    for loss, n_out in (("softmax_xent", 10), ("mse", 24), ("bce", 1)):
        chain = Chain(Dense(40, 24, "tanh"), Dense(24, n_out, "identity")).init_params(np.random.default_rng(2))
        for prec in ("bf16", "tf32", "strict_fp32"):
            tr = Trainer(chain, 96, loss=loss, precision=prec, small=False)
            X = torch.rand((96, 40), device="cuda")
            Y = (torch.rand((96, n_out), device="cuda") > 0.5).float()
            tr.gradient(X, Y)


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}
if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        torch.cuda.synchronize()
        check_guards()
        print("case", n, "ok (result, determinism, guard bands)", flush=True)
