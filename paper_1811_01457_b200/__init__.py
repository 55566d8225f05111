"""B200-native hot path of the ssagrad reference (arXiv 1811.01457, "Flux").

Public surface (mirrors the reference names for this path):

* fused broadcast: :func:`fused_map`, :func:`fused_map_with_partials`,
  :func:`fused_map_pullback`, :func:`fused_map_grad`
  (reference forward_ad.py:194-235, interp.py:322-352);
* IR: :class:`Module` and :func:`parse_ir` for building scalar functions
  (reference Module objects are accepted directly).

Kernels are hand-written CUDA for sm_100a behind the C ABI in
``include/sgb200.h`` (``_lib/libsgb200.so``); there is no CPU fallback.
"""

from .dense import Chain, ChainEngine, Dense, DenseLayer
from .fused import (DEFAULT_STEP_LIMIT, EvalError, check_errors, fused_map, fused_map_grad,
                    fused_map_pullback, fused_map_with_partials, set_step_limit)
from .gpu_machine import GpuMachine, eval_function, grad
from .tape import Tape
from .train import DataParallel, Trainer
from .ir import BOOL, F64, I64, Module, Type, tensor_type
from .irtext import parse_ir
from .runtime import DomainError, RuntimeUnavailable

__all__ = [
    "BOOL", "Chain", "ChainEngine", "DEFAULT_STEP_LIMIT", "DataParallel", "Dense", "DenseLayer",
    "DomainError", "EvalError", "F64", "GpuMachine", "I64", "Module", "RuntimeUnavailable", "Tape",
    "Trainer", "Type", "check_errors", "eval_function", "fused_map", "fused_map_grad",
    "fused_map_pullback", "fused_map_with_partials", "grad", "parse_ir", "set_step_limit", "tensor_type",
]
