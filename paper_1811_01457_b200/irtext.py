"""Reader for the ``.ssair`` textual IR.

Independent implementation of the text format the reference prints and
parses (format described at reference ``pkg/src/ssagrad/parser.py:1-20``,
printer ``ir.py:213-313``).  It exists so that the GPU tests and the
bench can build user scalar functions on a box where the reference is not
installed; modules the reference itself builds are consumed directly.

Only what a module needs to *describe* functions is implemented: types,
block parameters, instructions with attributes, ``ret``/``jmp``/``br``.
No verification is done beyond name resolution; the GPU codegen rejects
what it cannot lower.
"""

from __future__ import annotations

import re

from .ir import (BOOL, F64, I64, TAPE, Block, Br, FnRef, Function, Instruction,
                 Jmp, Module, Ret, Type, tensor_type)


class IRSyntaxError(ValueError):
    pass


_TOKENS = re.compile(r"""
    (?P<skip>\s+|//[^\n]*)
  | (?P<tensor>tensor<\d+(?:x\d+)*xf64>)
  | (?P<tapes>tapes<\d+>)
  | (?P<num>-?(?:\d+\.?\d*(?:[eE][-+]?\d+)?|inf\b|nan\b))
  | (?P<word>[A-Za-z_]\w*)
  | (?P<arrow>->)
  | (?P<sym>[@%^(){}\[\],:=])
""", re.VERBOSE)


def _tokenize(text: str) -> list[tuple[str, str, int]]:
    out = []
    i, line = 0, 1
    while i < len(text):
        m = _TOKENS.match(text, i)
        if not m:
            raise IRSyntaxError(f"line {line}: cannot read {text[i:i + 12]!r}")
        kind = m.lastgroup
        if kind != "skip":
            out.append((kind, m.group(), line))
        line += m.group().count("\n")
        i = m.end()
    out.append(("end", "", line))
    return out


def _type_of(tok: str) -> Type:
    if tok.startswith("tensor<"):
        dims = tok[len("tensor<"):-len("xf64>")]
        return tensor_type(*(int(d) for d in dims.split("x")))
    if tok.startswith("tapes<"):
        return Type("tapes", lanes=int(tok[6:-1]))
    simple = {"f64": F64, "i64": I64, "bool": BOOL, "tape": TAPE}
    if tok not in simple:
        raise IRSyntaxError(f"unknown type {tok!r}")
    return simple[tok]


class _Reader:
    def __init__(self, text: str):
        self.toks = _tokenize(text)
        self.i = 0

    # token helpers
    def peek(self, k: int = 0):
        return self.toks[min(self.i + k, len(self.toks) - 1)]

    def take(self, text: str | None = None, kind: str | None = None) -> str:
        k, t, line = self.toks[self.i]
        if (text is not None and t != text) or (kind is not None and k != kind):
            want = text if text is not None else kind
            raise IRSyntaxError(f"line {line}: expected {want!r}, found {t!r}")
        self.i += 1
        return t

    def maybe(self, text: str) -> bool:
        if self.toks[self.i][1] == text:
            self.i += 1
            return True
        return False

    def name(self, sigil: str) -> str:
        self.take(sigil)
        k, t, line = self.toks[self.i]
        if k not in ("word", "num"):
            raise IRSyntaxError(f"line {line}: bad name after {sigil}")
        self.i += 1
        return t

    def type_(self) -> Type:
        k, t, _ = self.peek()
        self.i += 1
        return _type_of(t)

    # grammar
    def module(self) -> Module:
        mod = Module()
        while self.peek()[0] != "end":
            mod.add(self.function())
        return mod

    def function(self) -> Function:
        self.take("func")
        fname = self.name("@")
        self.take("(")
        params = []
        while not self.maybe(")"):
            pname = self.name("%")
            self.take(":")
            params.append((pname, self.type_()))
            self.maybe(",")
        self.take("->")
        results = []
        if self.maybe("("):
            while not self.maybe(")"):
                results.append(self.type_())
                self.maybe(",")
        else:
            results.append(self.type_())
            while self.peek()[1] == ",":
                self.take(",")
                results.append(self.type_())
        self.take("{")
        raw_blocks = []
        first = True
        while not self.maybe("}"):
            raw_blocks.append(self.block(params if first else None))
            first = False
        return _resolve(fname, tuple(results), raw_blocks)

    def block(self, entry_params):
        bname = self.name("^")
        bparams = list(entry_params or [])
        if self.maybe("("):
            while not self.maybe(")"):
                pname = self.name("%")
                self.take(":")
                bparams.append((pname, self.type_()))
                self.maybe(",")
        self.take(":")
        body = []
        while self.peek()[1] == "%":
            body.append(self.instr())
        return bname, bparams, body, self.term()

    def operands(self) -> list[str]:
        ops = []
        # `%x` followed by `=` starts the next instruction (zero-operand ops
        # like tape_new are followed directly by the next result name)
        while self.peek()[1] == "%" and self.peek(2)[1] != "=":
            ops.append(self.name("%"))
            if not self.maybe(","):
                break
        return ops

    def instr(self):
        res = self.name("%")
        self.take("=")
        op = self.take(kind="word")
        if op == "const":
            ty = self.type_()
            if ty.is_tensor:
                self.take("[")
                vals = []
                while not self.maybe("]"):
                    vals.append(float(self.take(kind="num")))
                    self.maybe(",")
                value = tuple(vals)
            else:
                t = self.take()
                if ty.kind == "bool":
                    value = t == "true"
                elif ty.kind == "i64":
                    value = int(t)
                else:
                    value = float(t)
            return res, op, [], {"ty": ty, "value": value}
        ops = self.operands()
        attrs = {}
        if self.maybe("{"):
            while not self.maybe("}"):
                key = self.take(kind="word")
                self.take("=")
                attrs[key] = self.attr_value()
                self.maybe(",")
        return res, op, ops, attrs

    def attr_value(self):
        k, t, line = self.peek()
        if t == "@":
            return FnRef(self.name("@"))
        if t == "[":
            self.take("[")
            vals = []
            while not self.maybe("]"):
                vals.append(int(self.take(kind="num")))
                self.maybe(",")
            return tuple(vals)
        self.i += 1
        if k in ("tensor", "tapes") or t in ("f64", "i64", "bool", "tape"):
            return _type_of(t)
        if t in ("true", "false"):
            return t == "true"
        if k == "num":
            return float(t) if any(c in t for c in ".eEin") else int(t)
        return t  # bare identifier such as axis = all

    def args(self) -> list[str]:
        out = []
        if self.maybe("("):
            while not self.maybe(")"):
                out.append(self.name("%"))
                self.maybe(",")
        return out

    def term(self):
        kw = self.take(kind="word")
        if kw == "ret":
            return ("ret", self.operands())
        if kw == "jmp":
            tgt = self.name("^")
            return ("jmp", tgt, self.args())
        if kw == "br":
            cond = self.name("%")
            self.take(",")
            t1 = self.name("^")
            a1 = self.args()
            self.take(",")
            t2 = self.name("^")
            a2 = self.args()
            return ("br", cond, t1, a1, t2, a2)
        raise IRSyntaxError(f"unknown terminator {kw!r}")


def _resolve(fname, results, raw_blocks) -> Function:
    fn = Function(fname, results)
    ids: dict[str, int] = {}

    def define(n: str) -> int:
        vid = len(fn.vnames)
        fn.vnames[vid] = n
        ids[n] = vid
        return vid

    # definitions first, so forward references resolve
    for _, bparams, body, _ in raw_blocks:
        for pname, _ in bparams:
            define(pname)
        for res, *_ in body:
            define(res)

    def use(n: str) -> int:
        if n not in ids:
            raise IRSyntaxError(f"@{fname}: undefined value %{n}")
        return ids[n]

    for bname, bparams, body, term in raw_blocks:
        blk = Block(bname, [(ids[p], t) for p, t in bparams])
        for res, op, ops, attrs in body:
            blk.body.append(Instruction(ids[res], op, tuple(use(o) for o in ops), attrs))
        if term[0] == "ret":
            blk.term = Ret(tuple(use(o) for o in term[1]))
        elif term[0] == "jmp":
            blk.term = Jmp(term[1], tuple(use(o) for o in term[2]))
        else:
            _, c, t1, a1, t2, a2 = term
            blk.term = Br(use(c), t1, tuple(use(o) for o in a1), t2,
                          tuple(use(o) for o in a2))
        fn.blocks.append(blk)
    fn.next_id = len(fn.vnames)
    return fn


def parse_ir(text: str) -> Module:
    """Parse ``.ssair`` text into a :class:`Module`."""
    return _Reader(text).module()
