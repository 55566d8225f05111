"""Generate golden vectors by running the UNMODIFIED reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (pure Python + numpy) is importable here but does not travel
to the GPU box, so its outputs are frozen into the small fixtures next to
this script.  Everything is seeded; re-running reproduces the files
bit for bit.  Inputs are float32-representable so the same fixtures serve
the f32 and f64 device paths.

Reference entry points exercised (all under /root/reference/pkg/src/ssagrad):
  forward_ad.fused_map_with_partials / fused_map_pullback (forward_ad.py:194-235)
  interp.Machine fused_map and EvalError sites (interp.py:95-138, 322-332)
  reverse_ad.grad through fused_map and Dense IR (reverse_ad.py:633-663)
  tensor.matmul / reduce_to (tensor.py:327-361)
  nn_train-style Dense chains built with SEmitter (nn_train.py:189-227)
"""

from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from ssagrad import DenseTensor, Machine, Module, grad, parse_ir  # noqa: E402
from ssagrad import tensor as T  # noqa: E402
from ssagrad.forward_ad import fused_map_pullback, fused_map_with_partials  # noqa: E402
from ssagrad.interp import EvalError  # noqa: E402
from ssagrad.ir import F64, tensor_type  # noqa: E402
from ssagrad.structure import SEmitter, flatten  # noqa: E402
from ssagrad import nn_train  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from fused_src import FUSED_SRC  # noqa: E402
sys.path.insert(0, HERE)


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def dt(shape, rng, lo=-2.0, hi=2.0):
    return DenseTensor(f32(rng.uniform(lo, hi, size=shape)))


def enc(v):
    if isinstance(v, DenseTensor):
        return {"shape": list(v.shape), "data": v.flat()}
    return float(v)


# ------------------------------------------------------------------ fused
def fused_cases():
    m = parse_ir(FUSED_SRC)
    rng = np.random.default_rng(11)
    cases = []
    plans = [
        ("two", [(4,), ()]), ("two", [(2, 3), (2, 3)]), ("two", [(2, 1), (3,)]),
        ("two", [(), ()]), ("sgau", [(3, 3), ()]), ("sgau", [(6,), (6,)]),
        ("poly", [(5,)]), ("branchy", [(9,)]), ("gauss", [(4,), ()]),
        ("affsig", [(3,), (5, 3), (3,)]), ("affsig", [(), (4, 6), ()]),
        ("affsig", [(4, 1), (4, 6), (1, 6)]), ("affsig", [(2, 1, 3), (2, 4, 3), (4, 1)]),
        ("cubeloop", [(7,)]), ("powloop3", [(2, 5)]), ("relusq", [(8,)]),
        ("pick", [(6,), (6,)]), ("callin", [(5,)]), ("divy", [(4,), (4,)]),
        ("mixed", [(3, 4), (4,), ()]), ("logp", [(6,)]),
    ]
    for name, shapes in plans:
        args = []
        for s in shapes:
            if s == ():
                args.append(float(f32(rng.uniform(-2, 2))))
            else:
                lo = 0.1 if name == "logp" else -2.0
                args.append(dt(s, rng, lo=lo))
        if name == "branchy":  # keep clear of the branch point
            a = args[0].data.copy()
            a[np.abs(a) < 0.05] = 0.5
            args[0] = DenseTensor(a)
        primal, parts = fused_map_with_partials(m, name, tuple(args))
        shp = primal.shape if isinstance(primal, DenseTensor) else ()
        ybar = dt(shp, rng, -1, 1) if shp else None
        types = [tensor_type(*a.shape) if isinstance(a, DenseTensor) else F64 for a in args]
        pb = fused_map_pullback(parts, types, ybar) if ybar is not None else None
        cases.append({
            "fn": name,
            "args": [enc(a) for a in args],
            "primal": enc(primal),
            "partials": [enc(p) for p in parts],
            "ybar": enc(ybar) if ybar is not None else None,
            "pullback": [enc(c) for c in pb] if pb is not None else None,
        })
    # reverse mode through fused_map (test_forward_ad.py:164-172 analogue)
    x = DenseTensor(f32([0.2, -0.9, 1.4, 0.05]))
    g = grad(m, "mapped", (x, 0.7))
    mfn = m.get("mapped")
    grads = {"x": enc(g[mfn.params[0][0]]), "b": enc(g[mfn.params[1][0]])}
    # domain errors: reference EvalError location of the first failing element
    errors = []
    for name, vals in (("logp", [0.5, 2.0, -1.0, 3.0, -2.0]), ("divy", None)):
        if name == "logp":
            args = (DenseTensor(f32(vals)),)
        else:
            args = (DenseTensor(f32([1.0, 2.0, 3.0])), DenseTensor(f32([1.0, 0.0, 2.0])))
        try:
            fused_map_with_partials(m, name, args)
            raise AssertionError("expected EvalError")
        except EvalError as e:
            errors.append({"fn": name, "args": [enc(a) for a in args], "function": e.function,
                           "block": e.block, "index": e.index, "message": e.message})
    return {"cases": cases, "grad_mapped": grads, "errors": errors}


def fuzz_cases(n_programs=60, width=16):
    """Random scalar sub-functions fused over vectors, reference partials."""
    from ssagrad import print_ir
    from ssagrad.progen import random_program

    rng = random.Random(7)
    m = Module()
    out = []
    k = 0
    while len(out) < n_programs and k < 10 * n_programs:
        name = f"fz{k}"
        k += 1
        fn = random_program(m, rng, name, scalar_only=True)
        if any(ty.kind != "f64" for _, ty in fn.params):
            continue
        args = tuple(DenseTensor(f32([rng.uniform(-2, 2) for _ in range(width)])) for _ in fn.params)
        try:
            primal, parts = fused_map_with_partials(m, name, args)
        except (EvalError, OverflowError, ZeroDivisionError):
            continue
        if not all(np.isfinite(p.data).all() for p in [primal] + list(parts)):
            continue
        out.append({"fn": name, "args": [enc(a) for a in args], "primal": enc(primal),
                    "partials": [enc(p) for p in parts]})
    return {"ir": print_ir(m), "cases": out}


# ----------------------------------------------------------------- tensor
def tensor_cases():
    rng = np.random.default_rng(5)
    out = {}
    for i, (m_, k_, n_) in enumerate([(7, 13, 5), (33, 64, 17), (16, 100, 24)]):
        a = f32(rng.uniform(-1, 1, (m_, k_)))
        b = f32(rng.uniform(-1, 1, (k_, n_)))
        out[f"mm{i}_a"], out[f"mm{i}_b"] = a, b
        out[f"mm{i}_c"] = T.matmul(DenseTensor(a), DenseTensor(b)).data
    x = f32(rng.uniform(-1, 1, (6, 4, 5)))
    out["rt_x"] = x
    out["rt_to_5"] = T.reduce_to(DenseTensor(x), (5,)).data
    out["rt_to_415"] = T.reduce_to(DenseTensor(x), (4, 1)).data
    out["rt_to_145"] = T.reduce_to(DenseTensor(x), (1, 4, 5)).data
    out["rt_to_all"] = np.array([T.reduce_to(DenseTensor(x), ())])
    return out


# ------------------------------------------------------------ dense chains
def build_chain_loss(module, name, sizes, acts, n, loss):
    """Emit the loss of a Dense chain exactly as nn_train builds layers."""
    em = SEmitter(name, (F64,), module)
    pairs = []
    for k in range(len(sizes) - 1):
        w = em.param(f"W{k}", tensor_type(sizes[k + 1], sizes[k]))
        b = em.param(f"b{k}", tensor_type(sizes[k + 1]))
        pairs.append((w, b))
    x = em.param("X", tensor_type(n, sizes[0]))
    y = em.param("Y", tensor_type(n) if loss == "bce" else tensor_type(n, sizes[-1]))
    h = x
    for (w, b), act in zip(pairs, acts):  # nn_train.py:189-196
        wt = em.emit("transpose", (w,), None, "wt")
        z = em.emit("matmul", (h, wt), None, "z")
        zb = em.emit("add", (z, b), None, "zb")
        h = zb if act == "identity" else em.emit(act, (zb,), None, "h")
    if loss == "softmax_xent":  # SURVEY §8(d) c1 loss IR
        e = em.emit("exp", (h,), None, "e")
        s = em.emit("reduce_sum", (e,), {"axis": 1}, "s")
        s2 = em.emit("reshape", (s,), {"shape": (n, 1)}, "s2")
        p = em.emit("div", (e, s2), None, "p")
        lp = em.emit("log", (p,), None, "lp")
        t = em.emit("mul", (y, lp), None, "t")
        tot = em.emit("reduce_sum", (t,), {"axis": "all"}, "tot")
        sc = em.const_f64(-1.0 / n, "sc")
    elif loss == "mse":
        d = em.emit("sub", (h, y), None, "d")
        sq = em.emit("mul", (d, d), None, "sq")
        tot = em.emit("reduce_sum", (sq,), {"axis": "all"}, "tot")
        sc = em.const_f64(1.0 / n, "sc")
    elif loss == "bce":  # one-logit head + clamped mean BCE, emitted by the reference itself
        flatz = em.emit("reshape", (h,), {"shape": (n,)}, "logit")  # _batch_head, nn_train.py:209-210
        p = em.emit("sigmoid", (flatz,), None, "hat")
        lob = em.emit("bcast", (em.const_f64(1e-7, "lo"),), {"shape": (n,)}, "lob")
        hib = em.emit("bcast", (em.const_f64(1.0 - 1e-7, "hi"),), {"shape": (n,)}, "hib")
        ones = em.emit("bcast", (em.const_f64(1.0, "one"),), {"shape": (n,)}, "ones")
        l = nn_train._bce_mean(em, p, y, n, lob, hib, ones, "c")  # nn_train.py:213-227
        module.add(flatten(em.finish((l,))))
        return
    else:  # "dot": loss = sum(h * Y), i.e. pull back the seed Y through the chain
        t = em.emit("mul", (h, y), None, "t")
        tot = em.emit("reduce_sum", (t,), {"axis": "all"}, "tot")
        sc = em.const_f64(1.0, "sc")
    l = em.emit("mul", (tot, sc), None, "loss")
    module.add(flatten(em.finish((l,))))


def chain_case(sizes, acts, n, loss, seed, lr=0.05, y_kind="onehot", last_scale=1.0):
    rng = np.random.default_rng(seed)
    module = Module()
    build_chain_loss(module, "chain", sizes, acts, n, loss)
    params = []
    for k in range(len(sizes) - 1):
        fi, fo = sizes[k], sizes[k + 1]
        r = np.sqrt(6.0 / (fi + fo))  # init_params, nn_train.py:130-140
        W = f32(rng.uniform(-r, r, (fo, fi)) * (last_scale if k == len(sizes) - 2 else 1.0))
        b = f32(rng.uniform(-0.1, 0.1, fo))
        params.append((W, b))
    X = f32(rng.uniform(0, 1, (n, sizes[0])))
    if y_kind == "binary":
        Y = rng.integers(0, 2, n).astype(np.float64)
    elif y_kind == "onehot":
        Y = np.zeros((n, sizes[-1]))
        Y[np.arange(n), rng.integers(0, sizes[-1], n)] = 1.0
    else:
        Y = f32(rng.uniform(-1, 1, (n, sizes[-1])))
    args = []
    for W, b in params:
        args += [DenseTensor(W), DenseTensor(b)]
    args += [DenseTensor(X), DenseTensor(Y)]
    loss_v = Machine(module).call("chain", tuple(args))[0]
    g = grad(module, "chain", tuple(args))
    fn = module.get("chain")
    # inputs are float32-representable: store them as float32 (exact)
    out = {"X": X.astype(np.float32), "Y": Y.reshape(n, -1).astype(np.float32), "loss": np.array([loss_v]),
           "sizes": np.array(sizes), "lr": np.array([lr])}
    for k, (W, b) in enumerate(params):
        out[f"W{k}"], out[f"b{k}"] = W.astype(np.float32), b.astype(np.float32)
        gW = g[fn.params[2 * k][0]].data
        gb = g[fn.params[2 * k + 1][0]].data
        out[f"dW{k}"], out[f"db{k}"] = gW, gb
    out["dX"] = g[fn.params[2 * len(params)][0]].data
    return out


# ----------------------------------------------- augmented IR (GpuMachine)
def machine_cases():
    """Augmented forward/pullback pairs printed by the reference, with inputs
    and the reference's own cotangents, so the GPU machine can run the same
    IR on a box without the reference."""
    from ssagrad import augment, print_ir, generate_suite
    from ssagrad.nn_train import (DANConfig, _batch_tensors, _weight_args, build_loss_ir,
                                  dan_step, init_params, make_synthetic)
    from conftest_ref import ANALYTIC_SRC

    out = {}
    # analytic: tensor matmul/tanh/reduce (@net) and fused_map through a pack (@mapped)
    m = parse_ir(ANALYTIC_SRC)
    for name in ("net", "mapped", "cube", "absval", "callin"):
        augment(m, name)
    w = DenseTensor(f32([[0.3, -0.5, 0.8], [1.1, 0.2, -0.4]]))
    v = DenseTensor(f32([[0.5], [-1.2], [0.9]]))
    x = DenseTensor(f32([0.2, -0.9, 1.4, 0.05]))
    cases = {"net": (w, v), "mapped": (x, 0.7), "cube": (1.3,), "absval": (-2.5,), "callin": (1.3,)}
    analytic = {"ir": print_ir(m), "cases": []}
    for name, args in cases.items():
        fn = m.get(name)
        g = grad(m, name, args)
        analytic["cases"].append({"fn": name, "args": [enc(a) for a in args],
                                  "grads": [enc(g[pv]) for pv, ty in fn.params if ty.is_differentiable]})
    out["analytic"] = analytic

    # generated programs with branches/loops over tensors (test corpus seed)
    gm = Module()
    suite = generate_suite(gm, random.Random(20260822), 40, inputs_per=2)
    picked = []
    for name, inputs in suite:
        fn = gm.get(name)
        if any(ty.is_tensor for _, ty in fn.params) and len(picked) < 8:
            picked.append((name, inputs))
    corpus = {"cases": []}
    for name, inputs in picked:
        augment(gm, name)
        fn = gm.get(name)
        for args in inputs:
            g = grad(gm, name, args)
            corpus["cases"].append({"fn": name, "args": [enc(a) if not isinstance(a, int) else {"i64": a}
                                                         for a in args],
                                    "grads": [enc(g[pv]) for pv, ty in fn.params if ty.is_differentiable]})
    corpus["ir"] = print_ir(gm)
    out["corpus"] = corpus

    # the DAN two-head step (nn_train.py:337-375) at the test-suite SMALL config
    cfg = DANConfig(dim=6, trunk_sizes=(6, 4), head_sizes=(4, 1), n_samples=48, batch_size=8, epochs=2)
    sizes = (cfg.trunk_sizes, cfg.head_sizes, cfg.head_sizes)
    dm = Module()
    loss_fn = build_loss_ir(dm, sizes, cfg.batch_size)
    augment(dm, loss_fn.name)
    params = init_params(sizes, random.Random(2))
    batch = make_synthetic(cfg)[:cfg.batch_size]
    X, Yc, Yd = _batch_tensors(batch)
    args = _weight_args(params) + (X, Yc, Yd, cfg.lam)
    g_c = grad(dm, loss_fn.name, args, (1.0, 0.0))
    g_d = grad(dm, loss_fn.name, args, (0.0, 1.0))
    new, losses = dan_step(dm, params, batch, cfg)
    out["dan"] = {
        "ir": print_ir(dm), "fn": loss_fn.name, "lr": cfg.lr, "lam": cfg.lam,
        "args": [enc(a) for a in args],
        "g_c": [enc(g_c[pv]) for pv, ty in loss_fn.params if ty.is_differentiable],
        "g_d": [enc(g_d[pv]) for pv, ty in loss_fn.params if ty.is_differentiable],
        "new_params": [enc(t) for l in new.layers() for t in (l.W, l.b)],
        "losses": [losses["c_loss"], losses["d_loss"]],
    }
    return out


def spmd_cases():
    """Vectorised (SPMD lane) aug/pb programs printed by the reference and
    its batched_grad cotangents (spmd_batch.py:718-745): per-lane traces,
    lane-divergent loops, and matmul -> bmm for lanes that carry weights."""
    from ssagrad import augment, batched_grad, print_ir, stack_lanes, vectorize
    from ssagrad.ir import tensor_type
    from conftest_ref import ANALYTIC_SRC

    m = parse_ir(ANALYTIC_SRC)
    rng = np.random.default_rng(17)
    lanes = 4
    cases = []
    for name in ("net", "prod", "cube", "absval", "powloop"):
        fn = m.get(name)
        a, p = augment(m, name)
        vectorize(m, a.name, lanes)
        vectorize(m, p.name, lanes)
        per_lane = []
        for _ in range(lanes):
            args = []
            for _, ty in fn.params:
                if ty.kind == "tensor":
                    args.append(DenseTensor(f32(rng.uniform(-1.5, 1.5, ty.shape))))
                elif ty.kind == "i64":
                    args.append(int(rng.integers(0, 6)))
                else:
                    args.append(float(f32(rng.uniform(-2, 2, ()))))
            per_lane.append(args)
        stacked = tuple(stack_lanes(ty, [la[i] for la in per_lane]) for i, (_, ty) in enumerate(fn.params))
        seeds = tuple(stack_lanes(ty, [1.0] * lanes) for ty in fn.results)
        bg = batched_grad(m, name, lanes, stacked, seeds)
        cases.append({"fn": name, "lanes": lanes,
                      "args": [enc(v) for v in stacked], "seeds": [enc(v) for v in seeds],
                      "grads": [enc(bg[pv]) for pv, ty in fn.params if ty.is_differentiable]})
    return {"ir": print_ir(m), "cases": cases}


def dan_train_case():
    """Everything the reference's DAN `train` (nn_train.py:418-450) needs,
    frozen: augmented loss IR (batch 32), eval IR (n = 320), the synthetic
    data and initial parameters, and the reference's own epoch records for
    lam = 0 and lam = 1 (the acceptance criterion 7 configuration)."""
    from dataclasses import replace

    from ssagrad import augment, print_ir, train
    from ssagrad.nn_train import DANConfig, build_eval_ir, build_loss_ir, init_params, make_synthetic

    cfg = DANConfig()
    sizes = (cfg.trunk_sizes, cfg.head_sizes, cfg.head_sizes)
    m = Module()
    loss_fn = build_loss_ir(m, sizes, cfg.batch_size)
    augment(m, loss_fn.name)
    data = make_synthetic(cfg)
    eval_fn = build_eval_ir(m, sizes, len(data))
    params = init_params(sizes, random.Random(cfg.seed + 1))
    hist = {}
    for lam in (0.0, 1.0):
        hist[str(lam)] = train(replace(cfg, lam=lam)).records
    return {
        "ir": print_ir(m), "loss_fn": loss_fn.name, "eval_fn": eval_fn.name,
        "cfg": {"lr": cfg.lr, "epochs": cfg.epochs, "batch_size": cfg.batch_size, "seed": cfg.seed},
        "X": [s.x.flat() for s in data], "yc": [s.y_c for s in data], "yd": [s.y_d for s in data],
        "params": [enc(t) for l in params.layers() for t in (l.W, l.b)],
        "n_trunk": len(params.trunk), "n_head": len(params.class_head),
        "history": hist,
    }


def save_spmd():
    with open(os.path.join(HERE, "spmd.json"), "w") as f:
        json.dump(spmd_cases(), f, indent=0)


def save_bce():
    # binary classifier with the DAN head/loss recipe; large first-layer weights
    # push some predictions into the clamp range (select gradients = 0)
    np.savez_compressed(os.path.join(HERE, "mlp_bce.npz"),
                        **chain_case((12, 16, 1), ("tanh", "identity"), 48, "bce", 4, y_kind="binary",
                                     last_scale=24.0))


def domain_cases():
    """Dense chains whose float64 evaluation hits the reference's domain
    conditions: the c1 softmax loss IR (exp / reduce_sum / div / log) and the
    BCE head, run through the UNMODIFIED reference (Machine.call + grad).  The
    outcome is what it raises -- OverflowError from math.exp (scalar_sigmoid or
    the loss's exp), EvalError wrapping DomainError from div / log -- or the
    loss and gradients when nothing is undefined (extreme but finite logits)."""
    cases = []
    rng = np.random.default_rng(21)
    n, d0, d1, d2 = 6, 4, 3, 2
    X = f32(rng.uniform(0, 1, (n, d0)))
    W0 = f32(rng.uniform(-0.5, 0.5, (d1, d0)))
    b0 = f32(rng.uniform(-0.1, 0.1, d1))
    zeroW1 = np.zeros((d2, d1))
    plans = [  # (name, loss, hidden act, W0, b0, W1, b1)
        ("exp_overflow", "softmax_xent", "sigmoid", W0, b0, zeroW1, [800.0, 0.0]),
        ("div_zero", "softmax_xent", "sigmoid", W0, b0, zeroW1, [-800.0, -900.0]),
        ("log_zero", "softmax_xent", "sigmoid", W0, b0, zeroW1, [0.0, -800.0]),
        ("sum_overflow", "softmax_xent", "sigmoid", W0, b0, zeroW1, [709.5, 709.625]),
        ("sigmoid_overflow", "softmax_xent", "sigmoid", np.full((d1, d0), -800.0), b0, zeroW1, [0.5, -0.5]),
        ("extreme_finite", "softmax_xent", "sigmoid", W0, b0, zeroW1, [700.0, 0.0]),
        ("subnormal_p", "softmax_xent", "tanh", W0, b0, zeroW1, [0.0, -740.0]),
        ("bce_sigmoid_overflow", "bce", "tanh", W0, b0, np.zeros((1, d1)), [-720.0]),
        ("bce_saturated_ok", "bce", "tanh", W0, b0, np.zeros((1, d1)), [-700.0]),
    ]
    for name, loss, act, w0, bb0, w1, bb1 in plans:
        d_out = 1 if loss == "bce" else d2
        module = Module()
        build_chain_loss(module, "chain", (d0, d1, d_out), (act, "identity"), n, loss)
        if loss == "bce":
            Y = np.array([0.0, 1.0] * (n // 2))
        else:
            Y = np.zeros((n, d_out))
            Y[np.arange(n), np.arange(n) % d_out] = 1.0
        params = [(f32(w0), f32(bb0)), (f32(w1), f32(np.array(bb1)))]
        args = []
        for W, b in params:
            args += [DenseTensor(W), DenseTensor(b)]
        args += [DenseTensor(X), DenseTensor(Y)]
        out = {"name": name, "loss_kind": loss, "acts": [act, "identity"], "X": X.tolist(),
               "Y": Y.reshape(n, -1).tolist(),
               "params": [[W.tolist(), b.tolist()] for W, b in params]}
        try:
            lv = Machine(module).call("chain", tuple(args))[0]
            g = grad(module, "chain", tuple(args))
            fn = module.get("chain")
            out["raises"] = None
            out["loss"] = lv
            # where the reference's float64 pullback itself overflows (s*s in the
            # div adjoint, 1/p of a subnormal p) its gradients are not the
            # derivative; and log of a subnormal p carries fewer than 53 bits
            try:
                with np.errstate(over="raise", invalid="raise", divide="raise"):
                    grad(module, "chain", tuple(args))
                out["pullback_overflow"] = False
            except FloatingPointError:
                out["pullback_overflow"] = True
            h = X @ params[0][0].T + params[0][1]
            h = np.tanh(h) if act == "tanh" else 1.0 / (1.0 + np.exp(-h))
            z = h @ params[1][0].T + params[1][1]
            with np.errstate(over="ignore"):
                e = np.exp(z)
            p = e / e.sum(axis=1, keepdims=True)
            out["p_subnormal"] = bool(loss == "softmax_xent" and ((p > 0) & (p < np.finfo(np.float64).tiny)).any())
            out["grads"] = [[g[fn.params[2 * k][0]].data.tolist(), g[fn.params[2 * k + 1][0]].data.tolist()]
                            for k in range(2)]
        except EvalError as e:
            out["raises"] = "EvalError"
            out["message"] = e.message
            out["cause"] = type(e.__cause__).__name__
        except OverflowError as e:
            out["raises"] = "OverflowError"
            out["message"] = str(e)
        cases.append(out)
    return cases


def main():
    with open(os.path.join(HERE, "fused.json"), "w") as f:
        json.dump(fused_cases(), f, indent=0)
    with open(os.path.join(HERE, "machine.json"), "w") as f:
        json.dump(machine_cases(), f, indent=0)
    with open(os.path.join(HERE, "fuzz.json"), "w") as f:
        json.dump(fuzz_cases(), f, indent=0)
    save_spmd()
    with open(os.path.join(HERE, "dan_train.json"), "w") as f:
        json.dump(dan_train_case(), f)
    np.savez_compressed(os.path.join(HERE, "tensor.npz"), **tensor_cases())
    np.savez_compressed(os.path.join(HERE, "mlp_c1_b32.npz"),
                        **chain_case((784, 32, 10), ("sigmoid", "identity"), 32, "softmax_xent", 1))
    np.savez_compressed(os.path.join(HERE, "mlp_mse.npz"),
                        **chain_case((24, 24, 24, 24), ("tanh", "tanh", "identity"), 16, "mse", 2,
                                     y_kind="uniform"))
    save_bce()
    with open(os.path.join(HERE, "domain.json"), "w") as f:
        json.dump(domain_cases(), f, indent=0)
    np.savez_compressed(os.path.join(HERE, "dense_sigmoid.npz"),
                        **chain_case((40, 24), ("sigmoid",), 16, "dot", 3, y_kind="uniform"))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
