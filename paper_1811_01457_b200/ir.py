"""Minimal SSA IR data model for the hot path.

The GPU path consumes the reference's IR *objects*; it never needs the
reference's transforms.  This module is a small, independent model with
the same attribute surface (duck-typed), so that

* a ``Module`` built by the reference (``ssagrad.ir.Module``, its parser,
  ``SEmitter`` …) can be handed straight to :func:`fused_map` and friends,
* and tests on the GPU box, where the reference is absent, can build
  modules with :mod:`.irtext` instead.

Attribute surface mirrored (reference ``pkg/src/ssagrad/ir.py``):

* ``Type(kind, shape, lanes)`` with ``is_tensor``/``is_differentiable``
  (ir.py:29-57);
* ``Instruction(result, op, operands, attrs)`` (ir.py:93-98);
* terminators ``Ret(values)``, ``Jmp(target, args)``,
  ``Br(cond, then_target, then_args, else_target, else_args)``
  (ir.py:101-118);
* ``Block(name, params, body, term)`` and ``Function(name, results,
  blocks, vnames)`` with ``params`` = entry-block parameters
  (ir.py:124-166);
* ``Module.functions`` / ``get`` / ``add`` (ir.py:169-192).

Nothing here executes; evaluation lives in the CUDA codegen
(:mod:`.codegen`) and, for tests only, in ``oracle/``.
"""

from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class Type:
    kind: str  # "f64" | "i64" | "bool" | "tensor" | "tape" | "tapes"
    shape: tuple = ()
    lanes: int = 0

    @property
    def is_tensor(self) -> bool:
        return self.kind == "tensor"

    @property
    def is_differentiable(self) -> bool:
        return self.kind in ("f64", "tensor")

    def __str__(self) -> str:
        if self.kind == "tensor":
            return "tensor<" + "x".join(map(str, self.shape)) + "xf64>"
        if self.kind == "tapes":
            return f"tapes<{self.lanes}>"
        return self.kind


F64 = Type("f64")
I64 = Type("i64")
BOOL = Type("bool")
TAPE = Type("tape")


def tensor_type(*shape: int) -> Type:
    if not shape or any(int(d) < 1 for d in shape):
        raise ValueError(f"bad tensor shape {shape}")
    return Type("tensor", tuple(int(d) for d in shape))


@dataclass(frozen=True)
class FnRef:
    name: str

    def __str__(self) -> str:
        return "@" + self.name


@dataclass
class Instruction:
    result: int
    op: str
    operands: tuple = ()
    attrs: dict = field(default_factory=dict)


@dataclass
class Ret:
    values: tuple = ()


@dataclass
class Jmp:
    target: str
    args: tuple = ()


@dataclass
class Br:
    cond: int
    then_target: str
    then_args: tuple
    else_target: str
    else_args: tuple = ()


@dataclass
class Block:
    name: str
    params: list = field(default_factory=list)  # [(vid, Type)]
    body: list = field(default_factory=list)  # [Instruction]
    term: object = None


@dataclass
class Function:
    name: str
    results: tuple = ()
    blocks: list = field(default_factory=list)
    vnames: dict = field(default_factory=dict)
    next_id: int = 0

    @property
    def params(self) -> list:
        return self.blocks[0].params if self.blocks else []

    def value_name(self, vid: int) -> str:
        return self.vnames.get(vid, f"v{vid}")


@dataclass
class Module:
    functions: dict = field(default_factory=dict)

    def add(self, fn: Function) -> None:
        self.functions[fn.name] = fn

    def get(self, name: str) -> Function:
        try:
            return self.functions[name]
        except KeyError:
            raise KeyError(f"no function @{name} in module") from None


def kind_of(ty) -> str:
    """Kind string of any duck-typed IR type (ours or the reference's)."""
    return getattr(ty, "kind", str(ty))
