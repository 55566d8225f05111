"""B200-native hot path of the ssagrad reference (arXiv 1811.01457, "Flux").

Public surface (mirrors the reference names for this path):

* fused broadcast: :func:`fused_map`, :func:`fused_map_with_partials`,
  :func:`fused_map_pullback`, :func:`fused_map_grad`
  (reference forward_ad.py:194-235, interp.py:322-352);
* IR: :class:`Module` and :func:`parse_ir` for building scalar functions
  (reference Module objects are accepted directly);
* Dense layers and training: :class:`Dense`, :class:`Chain`, :class:`Trainer`
  (nn_train.py:189-210, 337-375), data parallelism (:class:`NcclDataParallel`);
* whole reference programs on the device: :class:`GpuMachine`, :func:`grad`,
  :func:`batched_grad`, :func:`trace_grad` with :class:`CudaBuilder`
  (interp.py, reverse_ad.py:633-663, spmd_batch.py:718-745, oracle.py:140-197).

Kernels are hand-written CUDA for sm_100a behind the C ABI in
``include/sgb200.h`` (``_lib/libsgb200.so``); there is no CPU fallback.
"""

from .dense import Chain, ChainEngine, Dense, DenseLayer
from .fused import (DEFAULT_STEP_LIMIT, EvalError, check_errors, fused_map, fused_map_grad,
                    fused_map_pullback, fused_map_with_partials, set_step_limit)
from .gpu_machine import GpuMachine, batched_grad, eval_function, grad
from .tape import Tape
from .taping import CudaBuilder, trace_eval, trace_grad
from .train import DataParallel, NcclDataParallel, Trainer
from .ir import BOOL, F64, I64, Module, Type, tensor_type
from .irtext import parse_ir
from .runtime import DomainError, RuntimeUnavailable

__all__ = [
    "BOOL", "Chain", "ChainEngine", "CudaBuilder", "DEFAULT_STEP_LIMIT", "DataParallel", "Dense",
    "DenseLayer", "DomainError", "EvalError", "F64", "GpuMachine", "I64", "Module", "NcclDataParallel",
    "RuntimeUnavailable", "Tape", "Trainer", "Type", "batched_grad", "check_errors", "eval_function",
    "fused_map", "fused_map_grad", "fused_map_pullback", "fused_map_with_partials", "grad", "parse_ir",
    "set_step_limit", "tensor_type", "trace_eval", "trace_grad",
]
