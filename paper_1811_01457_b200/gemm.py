"""Python binding of ``sg_gemm`` (include/sgb200.h): Dense-layer GEMMs.

``gemm(A, B)`` computes ``D[m, n] = sum_k A[m, k] B[n, k]`` with a fused
epilogue, where each operand is passed in its storage layout:

* ``a_mn=False``: ``A`` is ``[M, K]``; ``a_mn=True``: ``A`` is ``[K, M]``;
* ``b_mn=False``: ``B`` is ``[N, K]``; ``b_mn=True``: ``B`` is ``[K, N]``.

This is the reference's ``matmul`` (tensor.py:351-361) specialised to the
three products of a Dense layer (nn_train.py:192-193, rules.py:113-115).
"""

from __future__ import annotations

import ctypes

from . import runtime as rt

PREC = {"bf16": 0, "strict_fp32": 1, "strict_fp64": 2, "tf32": 3}
EPI = {"store": 0, "bias_act": 1, "act_grad": 2, "bias_act_seed": 3, "bias_mse": 4}
ACT = {"identity": 0, "sigmoid": 1, "tanh": 2, "relu": 3}


class GemmDesc(ctypes.Structure):
    _fields_ = [
        ("M", ctypes.c_int64), ("N", ctypes.c_int64), ("K", ctypes.c_int64),
        ("A", ctypes.c_void_p), ("lda", ctypes.c_int64), ("a_mn_major", ctypes.c_int32),
        ("B", ctypes.c_void_p), ("ldb", ctypes.c_int64), ("b_mn_major", ctypes.c_int32),
        ("precision", ctypes.c_int32), ("epilogue", ctypes.c_int32), ("act", ctypes.c_int32),
        ("bias", ctypes.c_void_p),
        ("aux", ctypes.c_void_p), ("ld_aux", ctypes.c_int64),
        ("out_pre", ctypes.c_void_p), ("ld_pre", ctypes.c_int64),
        ("out", ctypes.c_void_p), ("ld_out", ctypes.c_int64),
        ("out_lp", ctypes.c_void_p), ("ld_lp", ctypes.c_int64),
        ("colsum", ctypes.c_void_p), ("ld_colsum", ctypes.c_int64),
        ("batch", ctypes.c_int64),
        ("stride_a", ctypes.c_int64), ("stride_b", ctypes.c_int64),
        ("stride_out", ctypes.c_int64), ("stride_lp", ctypes.c_int64),
        ("out2_lp", ctypes.c_void_p), ("ld_out2", ctypes.c_int64),
        ("loss_part", ctypes.c_void_p), ("loss_scale", ctypes.c_double),
        ("split_part", ctypes.c_void_p), ("split_part_elems", ctypes.c_int64),
    ]


_bound = False


def _lib():
    global _bound
    lib = rt.load_library()
    if not _bound:
        lib.sg_gemm.argtypes = [ctypes.c_void_p, ctypes.POINTER(GemmDesc), ctypes.c_void_p]
        lib.sg_gemm.restype = ctypes.c_int
        lib.sg_gemm_splits.argtypes = [ctypes.c_void_p, ctypes.POINTER(GemmDesc), ctypes.POINTER(ctypes.c_int32),
                                       ctypes.POINTER(ctypes.c_int64)]
        lib.sg_gemm_splits.restype = ctypes.c_int
        P, I64 = ctypes.c_void_p, ctypes.c_int64
        lib.sg_splitk_reduce_multi.argtypes = [P, ctypes.c_int32, P, P, P, P, P, P, P, P]
        lib.sg_splitk_reduce_multi.restype = ctypes.c_int
        _bound = True
    return lib


def _ptr(t):
    return None if t is None else t.data_ptr()


def _ld(t):
    """Row stride (elements) of a 2-D operand with unit column stride.  A
    size-1 dimension's stride is arbitrary in torch: one column needs no
    column stride, and one row takes at least its own width."""
    if t is None:
        return 0
    if t.dim() != 2:
        raise ValueError("gemm operands must be 2-D with unit column stride")
    rows, cols = t.shape
    if cols != 1 and t.stride(1) != 1:
        raise ValueError("gemm operands must be 2-D with unit column stride")
    if rows == 1:
        return max(cols, t.stride(0))
    return t.stride(0)


def _want_dtypes(precision: str):
    """(operand, fp32-side, bf16-side) torch dtypes of a precision: operands
    A/B/aux, the fp32 outputs out/out_pre/bias/colsum, and out_lp."""
    import torch

    if precision not in PREC:
        raise ValueError(f"gemm: unknown precision {precision!r}")
    if precision == "bf16":
        return torch.bfloat16, torch.float32, torch.bfloat16
    if precision == "strict_fp64":
        return torch.float64, torch.float64, None
    return torch.float32, torch.float32, None


def check_dtypes(precision: str, operands=(), fp32=(), lp=(), colsum=None) -> None:
    """Reject tensors whose dtype the kernel would misread: the C descriptors
    carry no dtype, so a wrong one would be read as garbage or written past
    its allocation (an fp32 epilogue into a bf16 buffer writes twice its
    size).  ``operands``/``fp32``/``lp`` are (name, tensor-or-None) pairs."""
    op, wide, narrow = _want_dtypes(precision)
    import torch

    def need(name, t, dt):
        if t is not None and t.dtype != dt:
            raise ValueError(f"{name} must be {dt} for precision {precision!r}, not {t.dtype}")

    for name, t in operands:
        need(name, t, op)
    for name, t in fp32:
        need(name, t, wide)
    for name, t in lp:
        if t is not None and narrow is None:
            raise ValueError(f"{name} is a bf16-precision output (precision {precision!r})")
        need(name, t, narrow)
    need("colsum", colsum, torch.float32)


def gemm(A, B, *, M=None, N=None, K=None, a_mn=False, b_mn=False, precision="bf16",
         epilogue="store", act="identity", bias=None, aux=None, out=None, out_lp=None,
         out_pre=None, colsum=None, seed=None, out2_lp=None, loss_part=None, loss_scale=1.0, split_part=None,
         stream=None):
    """Launch one GEMM; outputs are written in place into the given tensors.

    ``split_part`` (fp32, contiguous): deferred split-K -- when the GEMM splits
    K (see :func:`gemm_splits`) its partials land there unreduced and ``out``
    is left untouched until :func:`splitk_reduce` runs.

    ``colsum`` (fp32 ``[ceil(M/32)][>=N]``) receives per-32-row column sums of
    the result (the first stage of a bias gradient).  ``epilogue="bias_act_seed"``
    (a forward with a known cotangent ``seed`` of its activation, fp32): ``out_lp``
    = act(z + b) and ``out2_lp`` = seed .* act'(out_lp), with ``colsum`` of the latter.
    ``epilogue="bias_mse"`` (a linear top layer with its MSE loss, targets
    ``seed`` fp32): ``out2_lp`` = 2 (z - y) loss_scale (+ ``colsum``), ``loss_part``
    (f64, ``ceil(M/32) * ceil(N/32)``) the per-block partial losses; ``out`` optional.
    """
    d = gemm_desc(A, B, M=M, N=N, K=K, a_mn=a_mn, b_mn=b_mn, precision=precision, epilogue=epilogue, act=act,
                  bias=bias, aux=aux, out=out, out_lp=out_lp, out_pre=out_pre, colsum=colsum, seed=seed,
                  out2_lp=out2_lp, loss_part=loss_part, loss_scale=loss_scale, split_part=split_part)
    rt.check(_lib().sg_gemm(rt.context(), ctypes.byref(d), rt.stream_ptr(stream)), "sg_gemm")


def gemm_splits(desc: "GemmDesc") -> tuple:
    """(splits, ld) sg_gemm picks for a descriptor: a deferred split-K needs
    ``splits * M * ld`` fp32 partials (splits == 1: no split)."""
    s, ld = ctypes.c_int32(1), ctypes.c_int64(0)
    rt.check(_lib().sg_gemm_splits(rt.context(), ctypes.byref(desc), ctypes.byref(s), ctypes.byref(ld)),
             "sg_gemm_splits")
    return int(s.value), int(ld.value)


def splitk_reduce(jobs, stream=None) -> None:
    """Reduce deferred split-K partials, several GEMMs in one launch:
    ``jobs`` = [(part, splits, M, N, ld_part, out)], out fp32 2-D (unit column
    stride); out = sum over splits in ascending order (sg_gemm's own reduce)."""
    n = len(jobs)
    if n == 0:
        return
    import torch

    for part, splits, M, N, ld, out in jobs:
        if (part.dtype != torch.float32 or out.dtype != torch.float32 or not part.is_contiguous()
                or out.dim() != 2 or out.shape[0] < M or out.shape[1] < N or ld < N):
            raise ValueError("splitk_reduce: contiguous fp32 partials (ld >= N) and an M x N fp32 output")
        if part.numel() < splits * M * ld:
            raise ValueError(f"splitk_reduce: {part.numel()} partials, {splits * M * ld} needed")
    A = ctypes.c_void_p * n
    I32, I64 = ctypes.c_int32 * n, ctypes.c_int64 * n
    rt.check(_lib().sg_splitk_reduce_multi(
        rt.context(), n, A(*[j[0].data_ptr() for j in jobs]), I32(*[j[1] for j in jobs]), I64(*[j[2] for j in jobs]),
        I64(*[j[3] for j in jobs]), I64(*[j[4] for j in jobs]), A(*[j[5].data_ptr() for j in jobs]),
        I64(*[_ld(j[5]) for j in jobs]), rt.stream_ptr(stream)), "sg_splitk_reduce_multi")


def gemm_desc(A, B, *, M=None, N=None, K=None, a_mn=False, b_mn=False, precision="bf16",
              epilogue="store", act="identity", bias=None, aux=None, out=None, out_lp=None,
              out_pre=None, colsum=None, seed=None, out2_lp=None, loss_part=None, loss_scale=1.0,
              split_part=None) -> GemmDesc:
    """The validated ``sg_gemm_desc`` of a GEMM (see :func:`gemm`), without launching it."""
    if a_mn:
        Ka, Ma = A.shape
    else:
        Ma, Ka = A.shape
    if b_mn:
        Kb, Nb = B.shape
    else:
        Nb, Kb = B.shape
    if K is None and Ka != Kb:
        raise ValueError(f"gemm: inner dimensions differ ({Ka} vs {Kb}); pass K to use a prefix")
    M = Ma if M is None else M
    N = Nb if N is None else N
    K = Ka if K is None else K
    if M > Ma or N > Nb or K > min(Ka, Kb):
        raise ValueError(f"gemm: M, N, K = {M}, {N}, {K} exceed the operands {tuple(A.shape)} x {tuple(B.shape)}")
    for name, t in (("out", out), ("out_lp", out_lp), ("out_pre", out_pre), ("aux", aux)):
        if t is not None and (t.dim() != 2 or t.shape[0] < M or t.shape[1] < N):
            raise ValueError(f"gemm: {name} of shape {tuple(t.shape)} cannot hold the {M} x {N} result")
    if bias is not None and bias.numel() < N:
        raise ValueError(f"gemm: bias has {bias.numel()} elements, {N} needed")
    if epilogue == "act_grad" and aux is None:
        raise ValueError("gemm: the act_grad epilogue needs aux (the saved activation)")
    if epilogue == "bias_act_seed":
        import torch

        # bf16: h in out_lp, dz in out2_lp (bf16); tf32: h in out, dz in out2_lp (fp32)
        bf = precision == "bf16"
        if (precision not in ("bf16", "tf32") or seed is None or out2_lp is None
                or (bf and (out_lp is None or out is not None)) or (not bf and (out is None or out_lp is not None))):
            raise ValueError("gemm: bias_act_seed needs seed and out2_lp, with out_lp (bf16) or out (tf32)")
        for name, t in (("seed", seed), ("out2_lp", out2_lp)):
            if t.dim() != 2 or t.shape[0] < M or t.shape[1] < N:
                raise ValueError(f"gemm: {name} of shape {tuple(t.shape)} cannot hold the {M} x {N} result")
        if seed.dtype != torch.float32 or out2_lp.dtype != (torch.bfloat16 if bf else torch.float32):
            raise ValueError("gemm: seed must be float32 and out2_lp bfloat16 (bf16) / float32 (tf32)")
        aux = seed  # the descriptor carries the seed in aux
    elif epilogue == "bias_mse":
        import torch

        if (precision != "bf16" or seed is None or out2_lp is None or loss_part is None or out_lp is not None
                or act != "identity"):
            raise ValueError("gemm: bias_mse needs bf16, identity, seed (targets), out2_lp and loss_part, no out_lp")
        for name, t in (("seed", seed), ("out2_lp", out2_lp)):
            if t.dim() != 2 or t.shape[0] < M or t.shape[1] < N:
                raise ValueError(f"gemm: {name} of shape {tuple(t.shape)} cannot hold the {M} x {N} result")
        if seed.dtype != torch.float32 or out2_lp.dtype != torch.bfloat16 or loss_part.dtype != torch.float64:
            raise ValueError("gemm: seed must be float32, out2_lp bfloat16 and loss_part float64")
        if loss_part.numel() < ((M + 31) // 32) * ((N + 31) // 32):
            raise ValueError(f"gemm: loss_part needs {((M + 31) // 32) * ((N + 31) // 32)} elements")
        aux = seed
    elif seed is not None or out2_lp is not None:
        raise ValueError("gemm: seed / out2_lp belong to the bias_act_seed / bias_mse epilogues")
    if loss_part is not None and epilogue != "bias_mse":
        raise ValueError("gemm: loss_part belongs to the bias_mse epilogue")
    check_dtypes(precision, operands=(("A", A), ("B", B)) + ((("aux", aux),) if seed is None else ()),
                 fp32=(("out", out), ("out_pre", out_pre), ("bias", bias)), lp=(("out_lp", out_lp),),
                 colsum=colsum)
    if colsum is not None and (colsum.dim() != 2 or colsum.shape[0] < (M + 31) // 32 or colsum.shape[1] < N):
        raise ValueError(f"gemm: colsum of shape {tuple(colsum.shape)} cannot hold ({(M + 31) // 32}, {N}) partials")
    d = GemmDesc()
    d.M, d.N, d.K = int(M), int(N), int(K)
    d.A, d.lda, d.a_mn_major = _ptr(A), _ld(A), int(a_mn)
    d.B, d.ldb, d.b_mn_major = _ptr(B), _ld(B), int(b_mn)
    d.precision = PREC[precision]
    d.epilogue = EPI[epilogue]
    d.act = ACT[act]
    d.bias = _ptr(bias)
    d.aux, d.ld_aux = _ptr(aux), _ld(aux)
    d.out_pre, d.ld_pre = _ptr(out_pre), _ld(out_pre)
    d.out, d.ld_out = _ptr(out), _ld(out)
    d.out_lp, d.ld_lp = _ptr(out_lp), _ld(out_lp)
    d.colsum, d.ld_colsum = _ptr(colsum), _ld(colsum)
    d.out2_lp, d.ld_out2 = _ptr(out2_lp), _ld(out2_lp)
    d.loss_part, d.loss_scale = _ptr(loss_part), float(loss_scale)
    if split_part is not None:
        import torch

        if split_part.dtype != torch.float32 or not split_part.is_contiguous():
            raise ValueError("gemm: split_part must be a contiguous float32 buffer")
    d.split_part, d.split_part_elems = _ptr(split_part), 0 if split_part is None else split_part.numel()
    d.keep = (A, B, bias, aux, out, out_lp, out_pre, colsum, out2_lp, loss_part, split_part)  # the buffers stay alive with the descriptor
    return d


DEP = {"rows": 1, "krows": 2, "all": 3}


class ChainProblem(ctypes.Structure):  # sg_chain_problem
    _fields_ = [("gemm", GemmDesc), ("splits", ctypes.c_int32), ("n_deps", ctypes.c_int32),
                ("dep_kind", ctypes.c_int32 * 2), ("dep_on", ctypes.c_int32 * 2)]


# problems per chain: their descriptions fill the 32 KB kernel parameter space
# (gemm_chain.cu MAX_PROBS; sg_chain_create refuses more)
CHAIN_MAX_PROBLEMS = 84


class GemmChain:
    """A persistent GEMM chain (``sg_chain_*``, include/sgb200.h): a list of
    GEMMs -- each a :class:`GemmDesc` with optional dependencies on earlier
    ones, ``[(kind, index), ...]`` with kind "rows" / "krows" / "all" -- planned
    once and run as ONE launch per :meth:`run`.  Bit-identical to running the
    same GEMMs one by one with :func:`gemm` (same tiles, k order and split-K
    summation order)."""

    def __init__(self, problems):
        lib = _lib()
        if not getattr(lib, "_chain_bound", False):
            P = ctypes.c_void_p
            lib.sg_chain_create.argtypes = [P, ctypes.POINTER(ChainProblem), ctypes.c_int32, ctypes.POINTER(P)]
            lib.sg_chain_run.argtypes = [P, P]
            lib.sg_chain_info.argtypes = [P, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                          ctypes.POINTER(ctypes.c_double)]
            lib.sg_chain_destroy.argtypes = [P]
            for n in ("sg_chain_create", "sg_chain_run", "sg_chain_info", "sg_chain_destroy"):
                getattr(lib, n).restype = ctypes.c_int
            lib._chain_bound = True
        self.lib = lib
        arr = (ChainProblem * len(problems))()
        self.keep = []
        for i, (desc, splits, deps) in enumerate(problems):
            if desc.precision != PREC["bf16"]:
                raise ValueError("chained GEMMs are bf16 tensor-core GEMMs")
            arr[i].gemm = desc
            self.keep.append(getattr(desc, "keep", None))
            arr[i].splits = int(splits)
            arr[i].n_deps = len(deps)
            for k, (kind, q) in enumerate(deps):
                if not 0 <= q < i:
                    raise ValueError(f"chain problem {i}: dependency on {q} is not an earlier problem")
                arr[i].dep_kind[k] = DEP[kind]
                arr[i].dep_on[k] = q
        h = ctypes.c_void_p()
        rt.check(lib.sg_chain_create(rt.context(), arr, len(problems), ctypes.byref(h)), "sg_chain_create")
        self.handle = h
        u, c, est = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
        rt.check(lib.sg_chain_info(h, ctypes.byref(u), ctypes.byref(c), ctypes.byref(est)), "sg_chain_info")
        self.units, self.ctas, self.est_us = u.value, c.value, est.value

    def run(self, stream=None) -> None:
        rt.check(self.lib.sg_chain_run(self.handle, rt.stream_ptr(stream)), "sg_chain_run")

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.sg_chain_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ld3(t):
    if t is None:
        return 0, 0
    if t.dim() != 3 or t.stride(2) != 1:
        raise ValueError("bmm operands must be 3-D [lanes, rows, cols] with unit column stride")
    return t.stride(1), t.stride(0)


def bmm(A, B, out=None, *, a_mn=False, b_mn=False, precision="bf16", epilogue="store", act="identity",
        bias=None, out_lp=None, stream=None):
    """Batched GEMM, one launch: ``out[l] = A[l] . B[l]^T`` per lane l (the
    reference's ``bmm``, tensor.py:364-369, with ``B`` given ``[lanes, N, K]``
    or, with ``b_mn``, ``[lanes, K, N]``).  Operands/outputs are 3-D with
    the lane axis first."""
    L = A.shape[0]
    if B.shape[0] != L:
        raise ValueError(f"bmm lane counts differ: {A.shape} x {B.shape}")
    Ka, Ma = (A.shape[1], A.shape[2]) if a_mn else (A.shape[2], A.shape[1])
    Kb, Nb = (B.shape[1], B.shape[2]) if b_mn else (B.shape[2], B.shape[1])
    if Ka != Kb:
        raise ValueError(f"bmm shapes {tuple(A.shape)} x {tuple(B.shape)}")
    for name, t in (("out", out), ("out_lp", out_lp)):
        if t is not None and (t.dim() != 3 or t.shape[0] != L or t.shape[1] < Ma or t.shape[2] < Nb):
            raise ValueError(f"bmm: {name} of shape {tuple(t.shape)} cannot hold {L} x {Ma} x {Nb}")
    if bias is not None and bias.numel() < Nb:
        raise ValueError(f"bmm: bias has {bias.numel()} elements, {Nb} needed")
    check_dtypes(precision, operands=(("A", A), ("B", B)), fp32=(("out", out), ("bias", bias)),
                 lp=(("out_lp", out_lp),))
    d = GemmDesc()
    d.M, d.N, d.K = int(Ma), int(Nb), int(Ka)
    (d.lda, d.stride_a), (d.ldb, d.stride_b) = _ld3(A), _ld3(B)
    d.A, d.a_mn_major, d.B, d.b_mn_major = _ptr(A), int(a_mn), _ptr(B), int(b_mn)
    d.precision, d.epilogue, d.act = PREC[precision], EPI[epilogue], ACT[act]
    d.bias = _ptr(bias)
    d.out, (d.ld_out, d.stride_out) = _ptr(out), _ld3(out)
    d.out_lp, (d.ld_lp, d.stride_lp) = _ptr(out_lp), _ld3(out_lp)
    d.batch = int(L)
    if L == 0 or d.M == 0 or d.N == 0:
        return
    rt.check(_lib().sg_gemm(rt.context(), ctypes.byref(d), rt.stream_ptr(stream)), "sg_gemm")
