"""ctypes binding of the in-tree C-ABI library ``_lib/libsgb200.so``.

The product path has no CPU fallback: if the library is missing or no
CUDA device is present, calls raise :class:`RuntimeUnavailable`.
Status codes map to the reference's exception types (include/sgb200.h):
SG_EDOMAIN -> DomainError/EvalError, SG_EINVAL -> ValueError.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libsgb200.so")
# tools only (tools/gemm_trace.py): an instrumented build of the same library
if os.environ.get("SGB200_LIB"):
    LIB_PATH = os.path.join(_HERE, "_lib", os.path.basename(os.environ["SGB200_LIB"]))

SG_OK, SG_EDOMAIN, SG_EINVAL, SG_ECUDA, SG_ENCCL = 0, 1, 2, 3, 4
SG_F32, SG_F64, SG_BF16 = 0, 1, 2
MAX_DIMS = 8

# every symbol include/sgb200.h declares (checked by the CPU test-suite)
EXPORTS = (
    "sg_version", "sg_create", "sg_destroy", "sg_last_error",
    "sg_ew_compile", "sg_ew_forward", "sg_ew_grad", "sg_ew_pack", "sg_ew_check",
    "sg_ew_set_step_limit", "sg_ew_compile_only", "sg_ew_variant_count", "sg_reduce_to",
    "sg_gemm", "sg_gemm_splits", "sg_splitk_reduce_multi", "sg_act_grad", "sg_colsum_finalize", "sg_colsum_finalize_multi", "sg_colsum_strict", "sg_loss", "sg_sgd", "sg_cast", "sg_cast_2d", "sg_sum_f64",
    "sg_dense_forward", "sg_dense_backward", "sg_mlp_small_scratch_bytes", "sg_mlp_small_step",
    "sg_dp_available", "sg_dp_unique_id", "sg_dp_init", "sg_dp_allreduce", "sg_dp_wait", "sg_dp_finalize",
    "sg_domain_check", "sg_chain_create", "sg_chain_run", "sg_chain_info", "sg_chain_destroy",
)


class RuntimeUnavailable(RuntimeError):
    """The CUDA library or device is missing; there is deliberately no fallback."""


class DomainError(ValueError):
    """Numerically undefined element op (mirror of reference tensor.py:25-26)."""


class CudaError(RuntimeError):
    pass


class SgTensor(ctypes.Structure):
    _fields_ = [
        ("ptr", ctypes.c_void_p),
        ("dtype", ctypes.c_int32),
        ("ndim", ctypes.c_int32),
        ("shape", ctypes.c_int64 * MAX_DIMS),
        ("scalar", ctypes.c_double),
    ]


_lib = None
_lib_lock = threading.Lock()


def load_library():
    """Load (once) and return the C-ABI library."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeUnavailable(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        P, I, I64, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
        T = ctypes.POINTER(SgTensor)
        sig = {
            "sg_version": ([], I),
            "sg_create": ([I, ctypes.POINTER(P)], I),
            "sg_destroy": ([P], I),
            "sg_last_error": ([ctypes.c_char_p, SZ], I),
            "sg_ew_compile": ([P, ctypes.c_char_p, ctypes.c_char_p, I, I, ctypes.POINTER(P)], I),
            "sg_ew_forward": ([P, P, I, T, T, P], I),
            "sg_ew_grad": ([P, P, I, T, T, T, T, P], I),
            "sg_ew_pack": ([P, P, I, T, T, P], I),
            "sg_ew_check": ([P, P, ctypes.POINTER(I64), ctypes.POINTER(ctypes.c_int32)], I),
            "sg_ew_set_step_limit": ([P, I64], I),
            "sg_ew_compile_only": ([ctypes.c_char_p, I, I, ctypes.POINTER(I), I, I, I,
                                    ctypes.POINTER(SZ)], I),
            "sg_ew_variant_count": ([P], I),
            "sg_reduce_to": ([P, T, T, T, P], I),
        }
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(8192)
    load_library().sg_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(status: int, what: str = "") -> None:
    if status == SG_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if status == SG_EDOMAIN:
        raise DomainError(msg)
    if status == SG_EINVAL:
        raise ValueError(msg)
    raise CudaError(msg)


# ------------------------------------------------------------- contexts

_ctxs: dict[int, int] = {}


def context(device: int | None = None) -> int:
    """The per-device ``sg_ctx*`` (created on first use)."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeUnavailable("no CUDA device: the sgb200 path has no CPU fallback")
    dev = torch.cuda.current_device() if device is None else int(device)
    if dev not in _ctxs:
        lib = load_library()
        torch.cuda.init()
        with torch.cuda.device(dev):
            h = ctypes.c_void_p()
            check(lib.sg_create(dev, ctypes.byref(h)), "sg_create")
        _ctxs[dev] = h.value
    return _ctxs[dev]


def stream_ptr(stream=None) -> int:
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


# ------------------------------------------------------- domain errors
SG_DOM_EXP_OVERFLOW, SG_DOM_DIV_ZERO, SG_DOM_LOG_NONPOS = 1, 2, 4


def domain_check(stream=None, function: str = "loss") -> None:
    """Surface the Dense-path domain flags (``sg_domain_check``) the way the
    reference raises them: ``math.exp`` overflow as ``OverflowError("math
    range error")`` (uncaught by run_blocks, tensor.py:245-250), division by
    zero and log of p <= 0 as ``EvalError`` wrapping a ``DomainError``
    (tensor.py:197-205, 230-233, interp.py:117-119).  When several are set,
    the one the reference's op order reaches first wins: the forward's
    exp/sigmoid, then the loss's div, then its log.  Synchronises ``stream``
    and clears the flags."""
    lib = load_library()
    if not getattr(lib.sg_domain_check, "_bound", False):
        lib.sg_domain_check.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32)]
        lib.sg_domain_check.restype = ctypes.c_int
        lib.sg_domain_check._bound = True
    flags = ctypes.c_int32(0)
    st = lib.sg_domain_check(context(), stream_ptr(stream), ctypes.byref(flags))
    if st not in (SG_OK, SG_EDOMAIN):
        check(st, "sg_domain_check")
    f = flags.value
    if not f:
        return
    if f & SG_DOM_EXP_OVERFLOW:
        raise OverflowError("math range error")
    from .fused import EvalError

    msg = "division by zero" if f & SG_DOM_DIV_ZERO else "log of non-positive value 0.0"
    raise EvalError(function, "", -1, msg) from DomainError(msg)


# ---------------------------------------------------------- descriptors

def dtype_code(dtype) -> int:
    import torch

    if dtype == torch.float32:
        return SG_F32
    if dtype == torch.float64:
        return SG_F64
    if dtype == torch.bfloat16:
        return SG_BF16
    raise ValueError(f"unsupported dtype {dtype}")


def tensor_desc(t) -> SgTensor:
    """Descriptor of a contiguous CUDA tensor (rank >= 1)."""
    d = SgTensor()
    if not t.is_contiguous():
        raise ValueError("sgb200 descriptors need contiguous tensors")
    if t.dim() > MAX_DIMS:
        raise ValueError(f"rank {t.dim()} exceeds {MAX_DIMS}")
    d.ptr = t.data_ptr()
    d.dtype = dtype_code(t.dtype)
    d.ndim = t.dim()
    for i, s in enumerate(t.shape):
        d.shape[i] = int(s)
    d.scalar = 0.0
    return d


def scalar_desc(x: float, dtype_c: int) -> SgTensor:
    d = SgTensor()
    d.ptr = None
    d.dtype = dtype_c
    d.ndim = 0
    d.scalar = float(x)
    return d


def desc_array(descs) -> "ctypes.Array":
    arr = (SgTensor * max(1, len(descs)))()
    for i, d in enumerate(descs):
        arr[i] = d
    return arr
