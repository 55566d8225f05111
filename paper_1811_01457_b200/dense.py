"""Dense layers, Chain, and the device engine of one training step.

Mirrors the reference's Dense recipe (``nn_train._batch_trunk`` /
``_batch_head``, nn_train.py:189-210)::

    wt = transpose(W); z = matmul(h, wt); zb = add(z, b); h' = act(zb)

with ``DenseLayerParams(W: out x in, b: out)`` (nn_train.py:40-45) and the
parameter order ``[W0, b0, W1, b1, ...]`` of ``_weight_args``
(nn_train.py:99-103), which is also the order of the flat gradient buffer
that data parallelism all-reduces.

HBM layout of :class:`ChainEngine` (one per GPU):

* ``P`` flat master parameters (fp32; fp64 in STRICT_FP64), ``G`` the flat
  gradients in the same layout, ``S`` a bf16 shadow of ``P`` that the SGD
  kernel rewrites for the next step's tensor-core GEMMs.  Each ``W`` is
  stored row-major ``[out][ld(in)]`` with ``ld`` rounded up to 8 elements
  and every segment 256-byte aligned (TMA row-stride/alignment rules);
* activations ``H[l]`` ``[B][ld(d_l)]`` in bf16 (saved for ``act'`` and as
  the next layer's input and the dW operand), top-layer outputs ``Zt`` in
  fp32 for the loss, two ping-pong ``dZ`` buffers, per-32-row column-sum
  partials for the bias gradients.

Precision modes: ``bf16`` (tcgen05 tensor cores, fp32 accumulate),
``strict_fp32`` / ``strict_fp64`` (ordered CUDA-core GEMMs, reference
fold order, everything in fp32/fp64).
"""

from __future__ import annotations

import ctypes
import os
import math
from dataclasses import dataclass

import numpy as np

from . import runtime as rt
from .gemm import ACT
from .tape import Tape, TapeEntry

LOSSES = {"softmax_xent": 0, "mse": 1, "bce": 2}


def _ld(d: int) -> int:
    return (d + 7) // 8 * 8


@dataclass
class Dense:
    """One dense layer ``act.(W * x .+ b)`` with W of shape (out, in)."""

    fan_in: int
    fan_out: int
    act: str = "identity"
    W: np.ndarray | None = None
    b: np.ndarray | None = None

    def __post_init__(self):
        if self.act not in ACT:
            raise ValueError(f"unknown activation {self.act!r}")


class Chain:
    """Sequential composition of Dense layers (Flux ``Chain``)."""

    def __init__(self, *layers: Dense):
        if not layers:
            raise ValueError("Chain needs at least one layer")
        for a, b in zip(layers, layers[1:]):
            if a.fan_out != b.fan_in:
                raise ValueError(f"layer sizes do not chain: {a.fan_out} -> {b.fan_in}")
        self.layers = list(layers)

    @property
    def sizes(self) -> tuple:
        return (self.layers[0].fan_in,) + tuple(l.fan_out for l in self.layers)

    @property
    def acts(self) -> tuple:
        return tuple(l.act for l in self.layers)

    def init_params(self, rng: np.random.Generator, bias: float = 0.0):
        """Uniform fan-in/fan-out init of init_params (nn_train.py:130-140)."""
        for l in self.layers:
            r = math.sqrt(6.0 / (l.fan_in + l.fan_out))
            l.W = rng.uniform(-r, r, (l.fan_out, l.fan_in)).astype(np.float32)
            l.b = np.full(l.fan_out, bias, dtype=np.float32)
        return self


# ---------------------------------------------------------------- C binding
class DenseDesc(ctypes.Structure):  # sg_dense_desc
    _fields_ = [
        ("batch", ctypes.c_int64), ("fan_in", ctypes.c_int64), ("fan_out", ctypes.c_int64),
        ("precision", ctypes.c_int32), ("act", ctypes.c_int32),
        ("X", ctypes.c_void_p), ("ldx", ctypes.c_int64),
        ("W", ctypes.c_void_p), ("ldw", ctypes.c_int64),
        ("b", ctypes.c_void_p),
    ]


class DenseGrad(ctypes.Structure):  # sg_dense_grad
    _fields_ = [
        ("dZ", ctypes.c_void_p), ("ld_dz", ctypes.c_int64),
        ("colsum_in", ctypes.c_void_p), ("ld_colsum_in", ctypes.c_int64),
        ("act_prev", ctypes.c_int32),
        ("dX", ctypes.c_void_p), ("ld_dx", ctypes.c_int64), ("dx_dtype", ctypes.c_int32),
        ("colsum_out", ctypes.c_void_p), ("ld_colsum_out", ctypes.c_int64),
        ("dW", ctypes.c_void_p), ("ld_dw", ctypes.c_int64),
        ("db", ctypes.c_void_p),
    ]


class MlpSmallDesc(ctypes.Structure):  # sg_mlp_small_desc
    MAXL = 4
    _fields_ = [
        ("L", ctypes.c_int32), ("sizes", ctypes.c_int32 * 5), ("act", ctypes.c_int32 * 4),
        ("w_off", ctypes.c_int64 * 4), ("b_off", ctypes.c_int64 * 4), ("ldw", ctypes.c_int64 * 4),
        ("loss", ctypes.c_int32), ("B", ctypes.c_int32), ("scale", ctypes.c_double), ("lr", ctypes.c_double),
    ]


_bound = False


def _lib():
    global _bound
    lib = rt.load_library()
    if not _bound:
        P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        lib.sg_act_grad.argtypes = [P, P, I32, I64, P, I32, I64, I64, I64, I32, P, I32, I64, P, I32, I64,
                                    P, I64, P]
        lib.sg_colsum_finalize.argtypes = [P, P, I64, I64, I64, P, P]
        lib.sg_colsum_finalize_multi.argtypes = [P, I32, P, P, P, P, P, P]
        lib.sg_colsum_strict.argtypes = [P, P, I32, I64, I64, I64, P, P]
        lib.sg_loss.argtypes = [P, I32, P, I32, I64, P, I64, I64, I64, D, P, P, I64, P, I32, I64, P, I32,
                                I64, P, I64, P]
        lib.sg_sgd.argtypes = [P, P, P, I32, I64, D, P, P]
        lib.sg_mlp_small_scratch_bytes.argtypes = [P, ctypes.POINTER(I64)]
        lib.sg_mlp_small_step.argtypes = [P, P, P, P, P, P, I64, P, I64, P, I64, P, P, I64, P]
        lib.sg_cast.argtypes = [P, P, I32, P, I32, I64, P]
        lib.sg_cast_2d.argtypes = [P, P, I32, I64, P, I32, I64, I64, I64, P]
        lib.sg_sum_f64.argtypes = [P, P, I64, P, P]
        lib.sg_dense_forward.argtypes = [P, ctypes.POINTER(DenseDesc), P, I64, P, I64, P, I64, P]
        lib.sg_dense_backward.argtypes = [P, ctypes.POINTER(DenseDesc), ctypes.POINTER(DenseGrad), P]
        for n in ("sg_act_grad", "sg_colsum_finalize", "sg_colsum_finalize_multi", "sg_colsum_strict", "sg_loss", "sg_sgd", "sg_cast", "sg_cast_2d",
                  "sg_sum_f64", "sg_dense_forward", "sg_dense_backward"):
            getattr(lib, n).restype = ctypes.c_int
        _bound = True
    return lib


def _p(t):
    return None if t is None else t.data_ptr()


def _dt(t):
    return rt.dtype_code(t.dtype)


def _ldt(t):
    return 0 if t is None else t.stride(0)


def cast_rows(src, dst, stream=None) -> None:
    """dst[:, :] = src (cast to dst's dtype) with the library's 2-D cast kernel
    (``sg_cast_2d``): rows may be padded (row strides), columns unit-stride."""
    if src.dim() != 2 or dst.dim() != 2 or tuple(src.shape) != tuple(dst.shape):
        raise ValueError(f"cast_rows: shapes {tuple(src.shape)} -> {tuple(dst.shape)}")
    if src.stride(1) != 1 or dst.stride(1) != 1:
        raise ValueError("cast_rows: rows must be unit-stride")
    if not src.is_cuda:
        raise ValueError("cast_rows: the source must be a device tensor (copy host batches in first)")
    rt.check(_lib().sg_cast_2d(rt.context(), _p(src), _dt(src), src.stride(0), _p(dst), _dt(dst), dst.stride(0),
                               src.shape[0], src.shape[1], rt.stream_ptr(stream)), "sg_cast_2d")


def dense_desc(X, W, b, act: str, precision: str) -> DenseDesc:
    """sg_dense_desc of one layer: X [batch][fan_in], W [fan_out][fan_in] (the
    precision's operand dtype), b [fan_out]."""
    from .gemm import PREC

    from .gemm import check_dtypes

    check_dtypes(precision, operands=(("X", X), ("W", W)), fp32=(("b", b),))
    d = DenseDesc()
    d.batch, d.fan_in = X.shape
    d.fan_out = W.shape[0]
    if W.shape[1] != d.fan_in:
        raise ValueError(f"dense: W of shape {tuple(W.shape)} does not take {d.fan_in} inputs")
    d.precision, d.act = PREC[precision], ACT[act]
    d.X, d.ldx = _p(X), _ldt(X)
    d.W, d.ldw = _p(W), _ldt(W)
    d.b = _p(b)
    return d


def _need(name, t, rows, cols):
    if t is not None and (t.dim() != 2 or t.shape[0] < rows or t.shape[1] < cols):
        raise ValueError(f"dense: {name} of shape {tuple(t.shape)} cannot hold {rows} x {cols}")


def _prec(desc: DenseDesc) -> str:
    from .gemm import PREC

    return {v: k for k, v in PREC.items()}[desc.precision]


def dense_forward(desc: DenseDesc, H=None, H_f32=None, Z=None, stream=None) -> None:
    """sg_dense_forward: H = act(X W^T + b) (nn_train.py:189-196) in one GEMM."""
    from .gemm import check_dtypes

    for name, t in (("H", H), ("H_f32", H_f32), ("Z", Z)):
        _need(name, t, desc.batch, desc.fan_out)
    prec = _prec(desc)
    if prec == "bf16":
        check_dtypes(prec, fp32=(("H_f32", H_f32), ("Z", Z)), lp=(("H", H),))
    else:
        check_dtypes(prec, fp32=(("H", H), ("Z", Z)), lp=(("H_f32", H_f32),))
    rt.check(_lib().sg_dense_forward(rt.context(), ctypes.byref(desc), _p(H), _ldt(H), _p(H_f32), _ldt(H_f32),
                                     _p(Z), _ldt(Z), rt.stream_ptr(stream)), "sg_dense_forward")


def dense_backward(desc: DenseDesc, dZ, dW, db, dX=None, act_prev: str = "identity", colsum_in=None,
                   colsum_out=None, stream=None) -> None:
    """sg_dense_backward: dW = dZ^T X, db = colsum(dZ), dX = dZ W [.* act_prev'(X)]
    (rules.py:45-46, 82-94, 113-124)."""
    _need("dZ", dZ, desc.batch, desc.fan_out)
    _need("dW", dW, desc.fan_out, desc.fan_in)
    _need("dX", dX, desc.batch, desc.fan_in)
    for name, t in (("colsum_in", colsum_in), ("colsum_out", colsum_out)):
        _need(name, t, (desc.batch + 31) // 32, desc.fan_out if name == "colsum_in" else desc.fan_in)
    if db is None or db.numel() < desc.fan_out:
        raise ValueError(f"dense: db needs {desc.fan_out} elements")
    from .gemm import check_dtypes

    prec = _prec(desc)
    check_dtypes(prec, operands=(("dZ", dZ),), fp32=(("dW", dW), ("db", db)))
    check_dtypes(prec, colsum=colsum_in)
    check_dtypes(prec, colsum=colsum_out)
    if dX is not None:
        import torch

        ok = (torch.bfloat16, torch.float32) if prec == "bf16" else (dZ.dtype,)
        if dX.dtype not in ok:
            raise ValueError(f"dense: dX must be one of {ok} for precision {prec!r}, not {dX.dtype}")
    g = DenseGrad()
    g.dZ, g.ld_dz = _p(dZ), _ldt(dZ)
    g.colsum_in, g.ld_colsum_in = _p(colsum_in), _ldt(colsum_in)
    g.act_prev = ACT[act_prev]
    g.dX, g.ld_dx = _p(dX), _ldt(dX)
    g.dx_dtype = _dt(dX) if dX is not None else 0
    g.colsum_out, g.ld_colsum_out = _p(colsum_out), _ldt(colsum_out)
    g.dW, g.ld_dw = _p(dW), _ldt(dW)
    g.db = _p(db)
    rt.check(_lib().sg_dense_backward(rt.context(), ctypes.byref(desc), ctypes.byref(g), rt.stream_ptr(stream)),
             "sg_dense_backward")


class DenseLayer:
    """One Dense layer's forward and pullback with preallocated device buffers.

    The single-layer form of the chain engine, used for the c3 workload
    (one Dense 4096->4096 fwd + pullback with an external seed ybar):

    * forward:  H = act(X . W^T + b)   -- one tcgen05 GEMM, bias+act epilogue
    * pullback: dZ = ybar .* act'(H)   (+ per-32-row column sums)
                dX = dZ . W            -- GEMM, W read MN-major
                dW = dZ^T . X          -- GEMM, both operands MN-major
                db = colsum(dZ)        -- finalize of the partial sums

    precision "bf16": bf16 operands/activations (W has a bf16 shadow);
    "tf32": fp32 operands/activations read as TF32 by the tensor cores.
    """

    def __init__(self, M: int, fan_in: int, fan_out: int, act: str = "sigmoid", precision: str = "bf16"):
        import torch

        if precision not in ("bf16", "tf32"):
            raise ValueError(f"DenseLayer precision must be bf16 or tf32, not {precision!r}")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.M, self.K, self.N, self.act = M, fan_in, fan_out, act
        self.precision = precision
        bf = torch.bfloat16 if precision == "bf16" else torch.float32
        self.X = torch.zeros((M, _ld(fan_in)), dtype=bf, device=dev)[:, :fan_in]
        self.W = torch.zeros((fan_out, _ld(fan_in)), dtype=torch.float32, device=dev)[:, :fan_in]
        self.Wb = (torch.zeros((fan_out, _ld(fan_in)), dtype=bf, device=dev)[:, :fan_in]
                   if precision == "bf16" else self.W)
        self.b = torch.zeros(fan_out, dtype=torch.float32, device=dev)
        self.H = torch.zeros((M, _ld(fan_out)), dtype=bf, device=dev)[:, :fan_out]
        self.dZ = torch.zeros((M, _ld(fan_out)), dtype=bf, device=dev)[:, :fan_out]
        self.dX = torch.zeros((M, _ld(fan_in)), dtype=torch.float32, device=dev)[:, :fan_in]
        self.dW = torch.zeros((fan_out, _ld(fan_in)), dtype=torch.float32, device=dev)[:, :fan_in]
        self.db = torch.zeros(fan_out, dtype=torch.float32, device=dev)
        self.colsum = torch.zeros(((M + 31) // 32, _ld(fan_out)), dtype=torch.float32, device=dev)

    def set_params(self, W, b):
        import torch

        self.W.copy_(torch.as_tensor(np.asarray(W), dtype=torch.float32))
        if self.Wb is not self.W:
            self.Wb.copy_(self.W.to(torch.bfloat16))
        self.b.copy_(torch.as_tensor(np.asarray(b), dtype=torch.float32))

    def forward(self, X=None):
        if X is not None:
            cast_rows(X, self.X)
        dense_forward(self.desc(), H=self.H)
        return self.H

    def desc(self) -> DenseDesc:
        return dense_desc(self.X, self.Wb, self.b, self.act, self.precision)

    def pullback(self, ybar, need_dx: bool = True):
        lib = _lib()
        ctx, st = rt.context(), rt.stream_ptr()
        rt.check(lib.sg_act_grad(ctx, _p(ybar), _dt(ybar), ybar.stride(0), _p(self.H), _dt(self.H),
                                 self.H.stride(0), self.M, self.N, ACT[self.act], _p(self.dZ), _dt(self.dZ),
                                 self.dZ.stride(0), None, 0, 0, _p(self.colsum), self.colsum.stride(0), st),
                 "sg_act_grad")
        dense_backward(self.desc(), self.dZ, self.dW, self.db, dX=self.dX if need_dx else None,
                       colsum_in=self.colsum)
        return self.dX, self.dW, self.db

    def value_and_pullback(self, ybar, X=None, need_dx: bool = True):
        """Forward and pullback with the output cotangent known up front (the
        reference's ``grad`` with seeds, reverse_ad.py:633-663): ONE forward
        GEMM whose epilogue also forms dZ = ybar .* act'(H) and its column sums
        (``bias_act_seed``), then dX and dW -- no separate act' pass.  bf16 or TF32."""
        from .gemm import gemm

        if X is not None:
            cast_rows(X, self.X)
        if self.precision == "bf16":
            gemm(self.X, self.Wb, epilogue="bias_act_seed", act=self.act, bias=self.b, seed=ybar, out_lp=self.H,
                 out2_lp=self.dZ, colsum=self.colsum)
        else:  # TF32: h and dz in fp32
            gemm(self.X, self.Wb, precision="tf32", epilogue="bias_act_seed", act=self.act, bias=self.b, seed=ybar,
                 out=self.H, out2_lp=self.dZ, colsum=self.colsum)
        dense_backward(self.desc(), self.dZ, self.dW, self.db, dX=self.dX if need_dx else None,
                       colsum_in=self.colsum)
        return self.H, self.dX, self.dW, self.db

    def flops(self, need_dx: bool = True) -> float:
        return 2.0 * self.M * self.K * self.N * (3 if need_dx else 2)


def slice_first_layer_buckets(buckets, w_off0: int, fan_in: int, fan_out: int, slices: int):
    """Bucket list with layer 0's bucket split into `slices` row blocks of W0
    (the last one running on through b0 to the end of the layer's bucket), or
    None when fan_out does not split into 64-row multiples.  Host-only (the
    data-parallel bucket layout; ChainEngine.enable_first_layer_slices)."""
    rows = fan_out // max(1, slices)
    if slices < 2 or fan_out % slices or rows % 64:
        return None
    ldi = _ld(fan_in)
    end0 = buckets[0][1]
    sub = [(w_off0 + k * rows * ldi, w_off0 + (k + 1) * rows * ldi) for k in range(slices - 1)]
    sub.append((w_off0 + (slices - 1) * rows * ldi, end0))
    return sub + list(buckets[1:])


def _pair_splits(M: int, N: int, K: int, pairs: int) -> int:
    """The split-K factor the CTA-pair GEMM picks for a plain-store product
    (gemm_tc.cu run_pair): used for the chained dW so the K-split sums --
    and hence the gradients -- are bit-identical to the per-layer path."""
    tiles = -(-M // 256) * -(-N // 256)
    num_kb = -(-K // 64)
    if tiles * 2 > pairs or num_kb < 8:
        return 1
    s = min(pairs // tiles, num_kb // 4, 16)
    if s < 2:
        return 1
    kb_per = -(-num_kb // s)
    return -(-num_kb // kb_per)


def bucket_of_layer(layer: int, l0_slices: int = 1, slice_k: int = 0) -> int:
    """Index of the gradient bucket that holds `layer` (and, for layer 0 in
    `l0_slices` > 1 row slices, its slice `slice_k`) in the bucket list of
    slice_first_layer_buckets: [W0 slice 0..S-1 (+ b0), layer 1, layer 2, ...]."""
    if l0_slices <= 1:
        return layer
    return slice_k if layer == 0 else layer + l0_slices - 1


def pullback_ready_order(n_layers: int, l0_slices: int = 1) -> list:
    """Bucket indices in the order the pullback readies them: the top layer
    first, down to layer 1, then layer 0's slices in ascending row order
    (ChainEngine._make_backward / _ready).  Host-only; the gloo tests replay it."""
    order = [bucket_of_layer(l, l0_slices) for l in range(n_layers - 1, 0, -1)]
    return order + [bucket_of_layer(0, l0_slices, k) for k in range(max(1, l0_slices))]


class ChainEngine:
    """Device state + kernels of a Dense chain's training step on one GPU."""

    def __init__(self, chain: Chain, batch: int, loss: str = "mse", precision: str = "bf16",
                 global_batch: int | None = None, small: bool = True, gemm_chain: bool | None = None):
        import os

        import torch

        if loss not in LOSSES:
            raise ValueError(f"unknown loss {loss!r}")
        if precision not in ("bf16", "tf32", "strict_fp32", "strict_fp64"):
            raise ValueError(f"unknown precision {precision!r}")
        # tensor-core modes: bf16 (bf16 operands, bf16 shadow of W) and tf32 (fp32
        # operands read as TF32); both use the fused colsum bias-gradient stage
        self.tc = precision in ("bf16", "tf32")
        self.chain = chain
        self.B = int(batch)
        self.loss_kind = loss
        self.precision = precision
        self.scale = 1.0 / float(global_batch or batch)
        self.sizes = chain.sizes
        self.acts = chain.acts
        self.L = len(chain.layers)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.mdt = torch.float64 if precision == "strict_fp64" else torch.float32  # master dtype
        self.adt = torch.bfloat16 if precision == "bf16" else self.mdt          # activation dtype
        self.gprec = precision

        # flat parameter layout [W0, b0, W1, b1, ...], 64-element (256 B) aligned segments
        off = 0
        self.seg = []
        for l in chain.layers:
            wo = off
            off += l.fan_out * _ld(l.fan_in)
            off = (off + 63) // 64 * 64
            bo = off
            off += l.fan_out
            off = (off + 63) // 64 * 64
            self.seg.append((wo, bo))
        self.numel = off
        self.P = torch.zeros(off, dtype=self.mdt, device=dev)
        self.G = torch.zeros(off, dtype=self.mdt, device=dev)
        self.S = torch.zeros(off, dtype=torch.bfloat16, device=dev) if precision == "bf16" else None
        self.W, self.b, self.gW, self.gb, self.Ws = [], [], [], [], []
        for l, (wo, bo) in zip(chain.layers, self.seg):
            ldi = _ld(l.fan_in)
            n = l.fan_out * ldi
            self.W.append(self.P[wo:wo + n].view(l.fan_out, ldi)[:, :l.fan_in])
            self.gW.append(self.G[wo:wo + n].view(l.fan_out, ldi)[:, :l.fan_in])
            self.b.append(self.P[bo:bo + l.fan_out])
            self.gb.append(self.G[bo:bo + l.fan_out])
            if self.S is not None:
                self.Ws.append(self.S[wo:wo + n].view(l.fan_out, ldi)[:, :l.fan_in])
        self.bucket_bounds = [(wo, (bo + l.fan_out + 63) // 64 * 64)
                              for l, (wo, bo) in zip(chain.layers, self.seg)]

        B = self.B
        self.H = [torch.zeros((B, _ld(d)), dtype=self.adt, device=dev)[:, :d] for d in self.sizes[:-1]]
        dL = self.sizes[-1]
        self.Zt = torch.zeros((B, _ld(dL)), dtype=self.mdt, device=dev)[:, :dL]
        self.Y = torch.zeros((B, _ld(dL)), dtype=self.mdt, device=dev)[:, :dL]
        dmax = max(self.sizes[1:])
        # persistent GEMM chains (sg_chain_*): the forward GEMMs of all layers in
        # one launch and the dX / dW GEMMs of all layers in another.  They need
        # every layer's dZ and bias-gradient partials in their own buffers (no
        # ping-pong: a chained dX may run while an earlier layer's dW still
        # reads the dZ it would overwrite).  bf16 only; off under data
        # parallelism (buckets are all-reduced per layer as the pullback goes).
        # Opt-in (SGB200_CHAIN=1 or gemm_chain=True): bit-identical to the
        # per-layer path but, measured on B200, not yet faster:
        # a chained unit's epilogue also waits for its TMA stores to land and
        # publishes them, and that is on the critical path at K = 1024.
        # Modes: "full" (SGB200_CHAIN=1): forward and pullback as one chain each;
        # "pairwise" (SGB200_CHAIN=2): per layer, the pullback's dW and dX -- two
        # independent GEMMs -- in ONE persistent launch (the dW's K-splits and
        # the dX tiles share the CTA pairs: no idle pairs beside the split-K
        # dW, one fill / drain instead of two), every db finalised at the end.
        # "forward" (SGB200_CHAIN=3): only the forward GEMMs below the top layer
        # as one chain; the top layer (with its fused loss) and the pullback
        # layer by layer.
        if gemm_chain is None:
            gemm_chain = {"1": "full", "2": "pairwise", "3": "forward"}.get(os.environ.get("SGB200_CHAIN", "0"))
        elif gemm_chain is True:
            gemm_chain = "full"
        if gemm_chain not in (None, False, "full", "pairwise", "forward"):
            raise ValueError(f"unknown gemm_chain mode {gemm_chain!r}")
        # (a chain's backward holds 2 L - 1 GEMMs: deeper chains run layer by layer)
        from .gemm import CHAIN_MAX_PROBLEMS

        self.chainable = (bool(gemm_chain) and precision == "bf16" and self.L >= 2
                          and 2 * self.L - 1 <= CHAIN_MAX_PROBLEMS)
        self.chain_mode = gemm_chain if self.chainable else None
        self.chains = None
        if self.chainable:
            self.dZl = [torch.zeros((B, _ld(d)), dtype=self.adt, device=dev)[:, :d] for d in self.sizes[1:]]
            self.csl = [torch.zeros(((B + 31) // 32, _ld(d)), dtype=torch.float32, device=dev)
                        for d in self.sizes[1:]]
        else:
            self.dZ = [torch.zeros((B, _ld(dmax)), dtype=self.adt, device=dev) for _ in range(2)]
            self.colsum = torch.zeros(((B + 31) // 32, _ld(dmax)), dtype=torch.float32, device=dev)
            if precision == "bf16" and self.L >= 2:
                # per-layer bias-gradient partials: every db finalised in one
                # launch after the pullback (deferred_db) instead of one per layer
                self.csl = [torch.zeros(((B + 31) // 32, _ld(d)), dtype=torch.float32, device=dev)
                            for d in self.sizes[1:]]
        self.dH = torch.zeros((B, _ld(dL)), dtype=self.mdt, device=dev)[:, :dL]
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        n_part = max(1, ((dmax + 31) // 32) * ((B + 31) // 32))
        self.loss_part = torch.zeros(n_part, dtype=torch.float64, device=dev)
        self.descs = [dense_desc(self.H[l], self.Ws[l] if precision == "bf16" else self.W[l], self.b[l],
                                 self.acts[l], precision) for l in range(self.L)]
        # bf16 + MSE + linear top layer: the training step computes the loss and
        # its seed dz in the top GEMM's epilogue (SG_EPI_BIAS_MSE) -- the fp32
        # top outputs are neither written nor read back (forward(fuse_loss=True));
        # SGB200_FUSED_LOSS=0 keeps the separate loss kernel
        self.fused_mse = (precision == "bf16" and loss == "mse" and self.acts[-1] == "identity"
                          and os.environ.get("SGB200_FUSED_LOSS", "1") != "0")
        self._loss_fused = False
        self.tape = Tape()
        self.grad_ready = None  # optional callback(bucket_index) when a bucket's gradients are written
        self.l0_slices = 1      # data parallel: layer 0's dW in row slices (enable_first_layer_slices)
        self.small = self._plan_small() if small else None
        # deferred split-K (bf16 pullback without per-layer hooks): a dW GEMM
        # that splits K leaves its partials in its own buffer and every layer's
        # are reduced in ONE launch after the pullback (sg_splitk_reduce_multi,
        # the same ordered sum) -- the per-layer reduce launch sat between the
        # layer's dW and the next dX.  SGB200_DEFER_SPLITK=0 reduces per GEMM.
        # (planned on the first deferred pullback -- an eager step, before any
        # graph capture -- so a data-parallel engine never allocates them)
        self.dw_split = None
        if chain.layers[0].W is not None:
            self.set_params([(l.W, l.b) for l in chain.layers])

    # ---------------------------------------------------------- parameters
    def set_params(self, params) -> None:
        import torch

        for l, (W, b) in enumerate(params):
            self.W[l].copy_(torch.as_tensor(np.asarray(W), dtype=self.mdt))
            self.b[l].copy_(torch.as_tensor(np.asarray(b), dtype=self.mdt))
        if self.S is not None:
            self.S.copy_(self.P.to(torch.bfloat16))

    def get_params(self):
        return [(self.W[l].double().cpu().numpy(), self.b[l].double().cpu().numpy()) for l in range(self.L)]

    def get_grads(self):
        return [(self.gW[l].double().cpu().numpy(), self.gb[l].double().cpu().numpy()) for l in range(self.L)]

    def dz_of(self, l):
        """dL/d(z_l + b_l) of layer l, [B][fan_out_l] (the layer's pullback seed)."""
        if self.chainable:
            return self.dZl[l]
        return self.dZ[l % 2][:, :self.sizes[l + 1]]

    def cs_of(self, l):
        """Per-32-row column-sum partials of dz_of(l) (tensor-core precisions)."""
        if not self.tc:
            return None
        return self.csl[l] if hasattr(self, "csl") else self.colsum

    @property
    def compute_precision(self) -> str:
        """The arithmetic the training step actually runs: the requested
        precision, except that a chain small enough for the one-launch step
        (``small``: c1-sized) computes in fp32 on the CUDA cores -- more
        accurate than a bf16 / tf32 request, and the tensor cores are not used."""
        return "fp32" if self.small is not None else self.precision

    def _deferred_db(self) -> bool:
        """bf16 pullback without per-layer hooks: dW and dX per layer, every db
        finalised at the end in one launch (sg_colsum_finalize_multi) -- the
        same kernels and arithmetic as sg_dense_backward, 15 launches fewer on
        c5.  Off under data parallelism: a bucket's db must be final when the
        pullback readies it."""
        import os

        return (hasattr(self, "csl") and self.grad_ready is None and self.l0_slices <= 1
                and os.environ.get("SGB200_DEFER_DB", "1") != "0")

    # ------------------------------------------------------------- inputs
    def load_batch(self, X, Y) -> None:
        """Load one minibatch (device tensors) with the library's kernels: X is
        cast into the first layer's activation rows (the operand dtype of the
        first GEMM) by ``sg_cast_2d``; Y is read IN PLACE by the loss kernel
        when it already has the master dtype and unit-stride rows (else it is
        cast into the engine's own target buffer).  No torch kernels: this
        runs inside the captured training step."""
        d0 = self.sizes[0]
        if tuple(X.shape) != (self.B, d0) or tuple(Y.shape) != (self.B, self.sizes[-1]):
            raise ValueError(f"batch shapes {tuple(X.shape)}, {tuple(Y.shape)} do not match the engine")
        cast_rows(X, self.H[0])
        if Y.dtype == self.mdt and Y.is_cuda and Y.stride(1) == 1:
            self.Yin = Y
        else:
            cast_rows(Y, self.Y)
            self.Yin = self.Y

    # ------------------------------------------------------------ forward
    def _top_forward_mse(self):
        """The top layer's forward GEMM with the MSE loss in its epilogue:
        dz_top = 2 (z - y) scale and its bias-gradient partials, the loss as
        per-block partials (summed by loss_and_seed).  z is not stored."""
        from .gemm import gemm

        top = self.L - 1
        Y = getattr(self, "Yin", None)
        Y = self.Y if Y is None else Y
        gemm(self.H[top], self.Ws[top], epilogue="bias_mse", bias=self.b[top], seed=Y,
             out2_lp=self.dz_of(top), colsum=self.cs_of(top), loss_part=self.loss_part, loss_scale=self.scale)
        self._loss_fused = True

    def forward(self, fuse_loss: bool = False):
        """Record the forward pass on the tape; returns the top-layer outputs.
        ``fuse_loss`` (training steps): when the engine fuses its loss
        (``fused_mse``), the top layer computes the loss and its seed instead
        of its outputs -- the return value is then None and loss_and_seed only
        sums the loss partials."""
        self.tape.clear()
        self._loss_fused = False
        fuse = fuse_loss and self.fused_mse
        use_chain = self._use_chain()
        if use_chain and self.chain_mode == "full":
            self.chains[0].run()
            # one tape entry for the whole chain: its pullback is the chained
            # dX / dW pass (the save set is every H[l] and W[l], as per layer)
            self.tape.push(TapeEntry("dense_chain", tuple(self.H) + tuple(self.W), self._chain_backward, None))
            return self.Zt
        L = self.L
        if use_chain and self.chain_mode == "forward":
            self.chains[0].run()  # layers 0 .. L-2 in one launch
            top = L - 1
            if fuse:
                self._top_forward_mse()
            else:
                dense_forward(self.descs[top], H=None, H_f32=self.Zt)
            for l in range(L):  # the pullback layer by layer, as without chains
                self.tape.push(TapeEntry(f"dense{l}", (self.H[l], self.W[l]), self._make_backward(l), self._ready(l)))
            return None if fuse else self.Zt
        if use_chain:  # pairwise: per-layer forward GEMMs, the pullback in L launches
            for l in range(L):
                last = l == L - 1
                if last and fuse:
                    self._top_forward_mse()
                else:
                    dense_forward(self.descs[l], H=None if last else self.H[l + 1], H_f32=self.Zt if last else None)
            self.tape.push(TapeEntry("dense_pairwise", tuple(self.H) + tuple(self.W), self._chain_backward, None))
            return None if fuse else self.Zt
        for l in range(L):
            last = l == L - 1
            if last and fuse:
                self._top_forward_mse()
            elif self.precision == "bf16":
                dense_forward(self.descs[l], H=None if last else self.H[l + 1], H_f32=self.Zt if last else None)
            else:
                dense_forward(self.descs[l], H=self.Zt if last else self.H[l + 1])
            self.tape.push(TapeEntry(f"dense{l}", (self.H[l], self.W[l]),
                                     self._make_backward(l), self._ready(l)))
        return None if fuse else self.Zt

    def _use_chain(self) -> bool:
        """Chains run when this engine can use them and no per-layer hooks are
        installed (data-parallel buckets, layer-0 slices); planned on first use."""
        if not self.chainable or self.grad_ready is not None or self.l0_slices > 1:
            return False
        if self.chains is None:
            self.chains = self._plan_chains()
        return True

    def _plan_chains(self):
        """The forward and backward GemmChains of this engine's buffers: the
        same GEMMs (operands, epilogues, split-K factors) sg_dense_forward /
        sg_dense_backward issue layer by layer, with row-block dependencies."""
        import torch

        from .gemm import GemmChain, gemm_desc

        L, B = self.L, self.B
        pairs = max(1, torch.cuda.get_device_properties(self.P.device).multi_processor_count // 2)
        if self.chain_mode == "forward":
            fwd = [(gemm_desc(self.H[l], self.Ws[l], epilogue="bias_act", act=self.acts[l], bias=self.b[l],
                              out_lp=self.H[l + 1]), 1, [("rows", l - 1)] if l > 0 else [])
                   for l in range(L - 1)]
            return GemmChain(fwd), None
        if self.chain_mode == "pairwise":
            per_layer = []
            for l in range(L):
                probs = [(gemm_desc(self.dz_of(l), self.H[l], a_mn=True, b_mn=True, out=self.gW[l]),
                          _pair_splits(self.sizes[l + 1], self.sizes[l], B, pairs), [])]
                if l > 0:  # the long dW K-splits are planned first, the dX tiles fill around them
                    act_prev = self.acts[l - 1]
                    probs.append((gemm_desc(self.dz_of(l), self.Ws[l], b_mn=True,
                                            epilogue="store" if act_prev == "identity" else "act_grad",
                                            act=act_prev, aux=self.H[l], out_lp=self.dz_of(l - 1),
                                            colsum=self.cs_of(l - 1)), 1, []))
                per_layer.append(GemmChain(probs))
            return None, per_layer
        fwd = []
        for l in range(L):
            top = l == L - 1
            d = gemm_desc(self.H[l], self.Ws[l], epilogue="bias_act", act=self.acts[l], bias=self.b[l],
                          out_lp=None if top else self.H[l + 1], out=self.Zt if top else None)
            fwd.append((d, 1, [("rows", l - 1)] if l > 0 else []))
        # backward order: the dX chain is the critical path (each layer's dZ
        # feeds the next dX row block by row block); layer l's dW (which only
        # needs dZ_l) is placed one layer later so it fills the gaps
        bwd, dx_idx = [], {}

        def add_dw(l):
            d = gemm_desc(self.dz_of(l), self.H[l], a_mn=True, b_mn=True, out=self.gW[l])
            bwd.append((d, _pair_splits(self.sizes[l + 1], self.sizes[l], B, pairs),
                        [("krows", dx_idx[l + 1])] if l + 1 in dx_idx else []))

        for l in range(L - 1, -1, -1):
            if l > 0:
                act_prev = self.acts[l - 1]
                d = gemm_desc(self.dz_of(l), self.Ws[l], b_mn=True,
                              epilogue="store" if act_prev == "identity" else "act_grad", act=act_prev,
                              aux=self.H[l], out_lp=self.dz_of(l - 1), colsum=self.cs_of(l - 1))
                bwd.append((d, 1, [("rows", dx_idx[l + 1])] if l + 1 in dx_idx else []))
                dx_idx[l] = len(bwd) - 1
            if l + 1 < L:
                add_dw(l + 1)
        add_dw(0)
        return GemmChain(fwd), GemmChain(bwd)

    def _finalize_all_db(self):
        """db_l = sum of dz_l's per-32-row partials, every layer in one launch."""
        lib = _lib()
        n = self.L
        parts = (ctypes.c_void_p * n)(*[_p(self.cs_of(l)) for l in range(n)])
        outs = (ctypes.c_void_p * n)(*[_p(self.gb[l]) for l in range(n)])
        G = (ctypes.c_int64 * n)(*[(self.B + 31) // 32] * n)
        ld = (ctypes.c_int64 * n)(*[self.cs_of(l).stride(0) for l in range(n)])
        N = (ctypes.c_int64 * n)(*[self.sizes[l + 1] for l in range(n)])
        rt.check(lib.sg_colsum_finalize_multi(rt.context(), n, parts, G, ld, N, outs, rt.stream_ptr()),
                 "sg_colsum_finalize_multi")

    def _dw_split_plan(self):
        """Per layer (partials, splits, ld) of a dW GEMM that splits K, else None."""
        if self.dw_split is None:
            import torch

            from .gemm import gemm_desc, gemm_splits

            self.dw_split = [None] * self.L
            if os.environ.get("SGB200_DEFER_SPLITK", "1") != "0":
                for l in range(self.L):
                    splits, ld = gemm_splits(gemm_desc(self.dz_of(l), self.H[l], a_mn=True, b_mn=True,
                                                       out=self.gW[l]))
                    if splits > 1:
                        part = torch.empty(splits * self.sizes[l + 1] * ld, dtype=torch.float32,
                                           device=self.P.device)
                        self.dw_split[l] = (part, splits, ld)
        return self.dw_split

    def _reduce_all_dw(self):
        """dW_l = sum of its deferred split-K partials, every split layer in one launch."""
        from .gemm import splitk_reduce

        splitk_reduce([(sp[0], sp[1], self.sizes[l + 1], self.sizes[l], sp[2], self.gW[l])
                       for l, sp in enumerate(self._dw_split_plan()) if sp is not None])

    def _chain_backward(self, _ctx):
        """Chained pullback: every layer's dX (with the lower layer's act' and
        bias-gradient partials fused) and dW in one launch -- or, pairwise, one
        launch per layer -- then every db."""
        if self.chain_mode == "pairwise":
            for l in range(self.L - 1, -1, -1):
                self.chains[1][l].run()
        else:
            self.chains[1].run()
        self._finalize_all_db()

    def _ready(self, l):
        def cb(_entry):
            if self.grad_ready is None:
                return
            if l > 0 or self.l0_slices <= 1:  # layer 0's slices ready their own buckets
                self.grad_ready(bucket_of_layer(l, self.l0_slices))
        return cb

    def enable_first_layer_slices(self, slices: int = 4, min_params: int = 8 << 20) -> bool:
        """Data parallel: split layer 0's dW into `slices` row blocks, each
        all-reduced as soon as it is written.  Layer 0's bucket is the last
        one the pullback produces and nothing is left to overlap it, so its
        exposed collective shrinks to one slice.  The buckets become
        [W0 rows 0, ..., W0 rows S-1 (+ b0), layer 1, layer 2, ...].  Each
        slice is the same GEMM restricted to its rows, so gradients are
        bit-identical to the unsliced step.  Returns whether slicing is on."""
        # worth it only for a large last bucket (c4: 16.8 M parameters, 67 MB; the
        # 1 M of c5 would pay ~50 us of smaller GEMMs to hide ~10 us of collective)
        if self.sizes[0] * self.sizes[1] < min_params:
            return False
        b = slice_first_layer_buckets(self.bucket_bounds, self.seg[0][0], self.sizes[0], self.sizes[1], slices)
        if b is None:
            return False
        self.l0_slices = slices
        self.bucket_bounds = b
        return True

    # --------------------------------------------------------------- loss
    def loss_and_seed(self):
        """Fused loss fwd+grad: loss scalar and dZ of the top layer (+ its bias sums)."""
        lib = _lib()
        ctx, st = rt.context(), rt.stream_ptr()
        top = self.L - 1
        dL = self.sizes[-1]
        if self._loss_fused:  # forward(fuse_loss=True) wrote dz and the loss partials
            n = ((self.B + 31) // 32) * ((dL + 31) // 32)
            rt.check(lib.sg_sum_f64(ctx, _p(self.loss_part), n, _p(self.loss), st), "sg_sum_f64")
            return self.loss
        dz = self.dz_of(top)
        cs = self.cs_of(top)
        ident = self.acts[top] == "identity"
        strict = not self.tc
        target = dz if ident else self.dH
        Y = getattr(self, "Yin", None)
        Y = self.Y if Y is None else Y
        rt.check(lib.sg_loss(ctx, LOSSES[self.loss_kind], _p(self.Zt), _dt(self.Zt), self.Zt.stride(0),
                             _p(Y), Y.stride(0), self.B, dL, self.scale, _p(self.loss),
                             _p(self.loss_part), self.loss_part.numel(), _p(target), _dt(target),
                             target.stride(0), None, 0, 0,
                             None if (strict or not ident) else _p(cs), 0 if cs is None else cs.stride(0), st),
                 "sg_loss")
        if not ident:  # top activation: dz = dL/dh * act'(h)  (rules.py:82-94)
            rt.check(lib.sg_act_grad(ctx, _p(self.dH), _dt(self.dH), self.dH.stride(0), _p(self.Zt),
                                     _dt(self.Zt), self.Zt.stride(0), self.B, dL, ACT[self.acts[top]],
                                     _p(dz), _dt(dz), dz.stride(0), None, 0, 0,
                                     None if strict else _p(cs), 0 if cs is None else cs.stride(0), st),
                     "sg_act_grad")
        return self.loss

    # ----------------------------------------------------------- pullback
    def _make_backward(self, l):
        def backward(_ctx):
            d_out, d_in = self.sizes[l + 1], self.sizes[l]
            dz = self.dz_of(l)
            cs = self.cs_of(l)
            if l == 0 and self.l0_slices > 1:
                S = self.l0_slices
                rows = d_out // S
                Wop = self.Ws[0] if self.precision == "bf16" else self.W[0]
                for k in range(S):
                    r = slice(k * rows, (k + 1) * rows)
                    desc = dense_desc(self.H[0], Wop[r], self.b[0][r], self.acts[0], self.precision)
                    dense_backward(desc, dz[:, r], self.gW[0][r], self.gb[0][r],
                                   colsum_in=None if cs is None else cs[:, r])
                    if self.grad_ready is not None:
                        self.grad_ready(bucket_of_layer(0, S, k))
                return
            if self._deferred_db():
                # the two GEMMs of sg_dense_backward (rules.py:113-115, 82-94);
                # db of every layer after layer 0's (rules.py:45-46)
                from .gemm import gemm

                sp = self._dw_split_plan()[l]
                gemm(dz, self.H[l], a_mn=True, b_mn=True, out=self.gW[l], split_part=None if sp is None else sp[0])
                if l > 0:
                    act_prev = self.acts[l - 1]
                    gemm(dz, self.Ws[l], b_mn=True, epilogue="store" if act_prev == "identity" else "act_grad",
                         act=act_prev, aux=self.H[l], out_lp=self.dz_of(l - 1), colsum=self.cs_of(l - 1))
                else:
                    self._finalize_all_db()
                    self._reduce_all_dw()
                return
            # dW = dZ^T H[l]; db = colsum(dZ) (partials fused upstream on the
            # tensor-core paths); dZ[l-1] = (dZ W) .* act'(H[l]) of the layer below
            dense_backward(self.descs[l], dz, self.gW[l], self.gb[l],
                           dX=self.dz_of(l - 1) if l > 0 else None,
                           act_prev=self.acts[l - 1] if l > 0 else "identity",
                           colsum_in=cs, colsum_out=self.cs_of(l - 1) if l > 0 else None)
        return backward

    def pullback(self):
        self.tape.pullback()

    # ------------------------------------------------- one-launch small step
    def _plan_small(self):
        """Descriptor + scratch of the one-launch step (``sg_mlp_small_step``)
        when this chain qualifies: tensor-core precision (the step then runs
        in fp32, more accurate than requested), softmax-CE or MSE loss, <= 4
        layers, widths <= 1024, batch <= 512 and a per-launch working set
        that fits in shared memory; ``None`` otherwise (the layer-by-layer
        path).  ``SGB200_MLP_SMALL=0`` disables it."""
        import os

        import torch

        if os.environ.get("SGB200_MLP_SMALL", "1") == "0":
            return None
        if not self.tc or self.loss_kind not in ("softmax_xent", "mse") or self.L > MlpSmallDesc.MAXL:
            return None
        if self.B > 512 or max(self.sizes) > 1024 or self.scale != 1.0 / self.B:
            return None
        if self.flops_per_step() > 64e6:  # beyond latency-bound sizes the tensor-core chain wins
            return None
        d = MlpSmallDesc()
        d.L, d.loss, d.B, d.scale = self.L, LOSSES[self.loss_kind], self.B, self.scale
        for i, v in enumerate(self.sizes):
            d.sizes[i] = v
        for l, (wo, bo) in enumerate(self.seg):
            d.act[l] = ACT[self.acts[l]]
            d.w_off[l], d.b_off[l], d.ldw[l] = wo, bo, _ld(self.sizes[l])
        lib = _lib()
        n = ctypes.c_int64()
        if lib.sg_mlp_small_scratch_bytes(ctypes.byref(d), ctypes.byref(n)) != 0:
            return None  # outside the kernel's limits
        dev = self.P.device
        self.small_scratch = torch.zeros(n.value, dtype=torch.uint8, device=dev)
        self.X32 = torch.zeros((self.B, self.sizes[0]), dtype=torch.float32, device=dev)
        self.Y32 = torch.zeros((self.B, self.sizes[-1]), dtype=torch.float32, device=dev)
        return d

    def small_step(self, X, Y, lr: float):
        """forward + loss + pullback + SGD of the loaded batch in ONE launch
        (``sg_mlp_small_step``); X, Y fp32 rows are read in place when they
        are row-contiguous, else copied first.  Returns the loss (device).

        The step is a ~20 us kernel, so the host path matters: the ctypes
        argument tuple is cached per (X, Y, stream) and reused."""
        import torch

        stream = torch.cuda.current_stream()
        key = (X.data_ptr(), Y.data_ptr(), tuple(X.shape), tuple(Y.shape), X.stride(0), Y.stride(0),
               X.dtype, Y.dtype, stream.cuda_stream)
        cache = getattr(self, "_small_args", None)
        if cache is None or cache[0] != key:
            if tuple(X.shape) != (self.B, self.sizes[0]) or tuple(Y.shape) != (self.B, self.sizes[-1]):
                raise ValueError(f"batch shapes {tuple(X.shape)}, {tuple(Y.shape)} do not match the engine")

            def direct(t):
                return t.dtype == torch.float32 and t.is_cuda and t.stride(1) == 1 and t.data_ptr() % 16 == 0

            Xd, Yd = (X if direct(X) else self.X32), (Y if direct(Y) else self.Y32)
            args = (rt.context(), ctypes.byref(self.small), _p(self.P), _p(self.G), _p(self.S), _p(Xd),
                    Xd.stride(0), _p(Yd), Yd.stride(0), _p(self.Zt), self.Zt.stride(0), _p(self.loss),
                    _p(self.small_scratch), self.small_scratch.numel(), int(stream.cuda_stream))
            cache = (key, args, None if Xd is X else self.X32, None if Yd is Y else self.Y32)
            self._small_args = cache
        _, args, xcopy, ycopy = cache
        if xcopy is not None:  # the cache key pins the source tensors; their contents are re-copied
            xcopy.copy_(X, non_blocking=True)
        if ycopy is not None:
            ycopy.copy_(Y, non_blocking=True)
        self.small.lr = float(lr)
        rc = _lib().sg_mlp_small_step(*args)
        if rc:
            rt.check(rc, "sg_mlp_small_step")
        return self.loss

    # ---------------------------------------------------------------- SGD
    def sgd(self, lr: float):
        lib = _lib()
        rt.check(lib.sg_sgd(rt.context(), _p(self.P), _p(self.G), _dt(self.P), self.numel, float(lr),
                            _p(self.S), rt.stream_ptr()), "sg_sgd")

    def step(self, lr: float):
        """forward + loss + pullback + SGD on the loaded batch (all device-side)."""
        self.forward(fuse_loss=True)
        self.loss_and_seed()
        self.pullback()
        self.sgd(lr)
        return self.loss

    def flops_per_step(self, skip_first_dx: bool = True) -> float:
        f = 0.0
        for l in range(self.L):
            mnk = self.B * self.sizes[l] * self.sizes[l + 1]
            f += 2 * mnk * (3 if (l > 0 or not skip_first_dx) else 2)
        return f
