import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
from oracle import dense as OD
from paper_1811_01457_b200.dense import Chain, Dense
from paper_1811_01457_b200.train import Trainer
rng = np.random.default_rng(0)
sizes, acts, B = (64, 48, 10), ("sigmoid", "identity"), 32
chain = Chain(Dense(64, 48, "sigmoid"), Dense(48, 10)).init_params(rng)
X = rng.uniform(0, 1, (B, 64)).astype(np.float32)
Y = np.zeros((B, 10), np.float32); Y[np.arange(B), rng.integers(0, 10, B)] = 1
tr = Trainer(chain, B, loss="softmax_xent", lr=0.05, precision="bf16")
lv, grads = tr.gradient(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda())
params = [(l.W.astype(np.float64), l.b.astype(np.float64)) for l in chain.layers]
lo, go, _ = OD.mlp_step(params, X.astype(np.float64), Y.astype(np.float64), acts, "softmax_xent")
print("lv", lv, "lo", lo)
print("Zt", tr.engine.Zt[:2].cpu().numpy())
print("loss_part", tr.engine.loss_part[:4].cpu().numpy())
