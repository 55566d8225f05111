"""Lower a scalar IR sub-function to CUDA C++ device code.

The reference evaluates ``fused_map``/``fused_pack`` by interpreting the
scalar sub-function once per element (``interp.py:322-352``,
``forward_ad.py:56-149``).  Here the sub-function is compiled instead:
every block becomes a label, block parameters become locals assigned at
each jump, and ``br``/``jmp``/``ret`` become ``if``/``goto``/``return``.
Loops and branches therefore need no structurization pass, and a user
function with data-dependent control flow runs per element exactly as in
the interpreter.

Two forms are emitted per function:

* **primal** -- scalar semantics of ``Machine.dispatch`` for scalar
  operands (``interp.py:194-269``) with the scalar kernels of
  ``tensor.py:197-233`` (sigmoid = 1/(1+e^-x), relu, pow_int as
  left-to-right repeated multiply, DomainError for div by zero and
  log(x <= 0));
* **dual** -- the forward-mode rules of ``_DualRunner.dispatch``
  (``forward_ad.py:72-143``): a dual carries the primal plus K tangents,
  seeded one-hot per argument as ``pack_rows`` does (``forward_ad.py:178-191``).

Floating point: ``T`` is ``float`` or ``double``.  The kernels are built
with ``--fmad=false`` so ``+ - * /`` round exactly like the reference's
Python floats (no contraction); in f64 mode straight-line arithmetic is
bit-identical to the reference, transcendentals differ by libm ulps.

Errors: a domain error or an exhausted step budget stores a *site* id
(index into :attr:`Lowered.sites`, 1-based) into the thread's error
variable and unwinds; the kernel then publishes ``(element, site)`` with
an ``atomicMin`` so the lowest failing element wins, which is the element
the reference's sequential loop would have raised on.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

from .ir import kind_of

_SCALAR_OPS = {
    "const", "add", "sub", "mul", "div", "neg", "exp", "log", "tanh", "sigmoid",
    "relu", "pow_int", "itof", "lt", "gt", "eq", "select", "call",
}


class CodegenError(ValueError):
    """The function cannot be lowered (non-scalar op, recursion, bad types)."""


@dataclass
class Site:
    function: str
    block: str
    index: int
    message: str


@dataclass
class Lowered:
    source: str                 # device functions + entry wrappers
    k: int                      # number of sub-function arguments
    key: str                    # content hash (cache key)
    sites: list = field(default_factory=list)
    entry: str = ""


def _lit(x: float) -> str:
    if math.isnan(x):
        return "((T)__longlong_as_double(0x7ff8000000000000LL))"
    if math.isinf(x):
        s = "0x7ff0000000000000LL" if x > 0 else "0xfff0000000000000LL"
        return f"((T)__longlong_as_double({s}))"
    return f"((T){float(x).hex()})"


def check_scalar_fn(fn) -> None:
    """Mirror of ``forward_ad._check_scalar_fn`` (forward_ad.py:152-157)."""
    if len(fn.results) != 1 or kind_of(fn.results[0]) != "f64":
        raise ValueError(f"@{fn.name} must return a single f64")
    for _, ty in fn.params:
        if kind_of(ty) != "f64":
            raise ValueError(f"@{fn.name} takes a non-f64 parameter")


def _cyclic(fn) -> bool:
    """Whether the CFG has a back edge (then the step budget is enforced)."""
    succ = {}
    for b in fn.blocks:
        t = b.term
        names = []
        if hasattr(t, "target"):
            names = [t.target]
        elif hasattr(t, "then_target"):
            names = [t.then_target, t.else_target]
        succ[b.name] = names
    state = {}

    def dfs(n):
        state[n] = 1
        for m in succ.get(n, ()):
            s = state.get(m, 0)
            if s == 1 or (s == 0 and dfs(m)):
                return True
        state[n] = 2
        return False

    return bool(fn.blocks) and dfs(fn.blocks[0].name)


class _FnLowering:
    def __init__(self, owner: "_Lowerer", fn, index: int):
        self.o = owner
        self.fn = fn
        self.idx = index
        self.dual = owner.dual
        self.types = {}
        for b in fn.blocks:
            for vid, ty in b.params:
                self.types[vid] = kind_of(ty)
        self.lines: list[str] = []

    # names
    def v(self, vid: int) -> str:
        return f"v{vid}"

    def ctype(self, kind: str) -> str:
        if kind == "f64":
            return "D" if self.dual else "T"
        if kind == "i64":
            return "long long"
        if kind == "bool":
            return "bool"
        raise CodegenError(f"@{self.fn.name}: values of type {kind} are not scalar")

    @property
    def fname(self) -> str:
        return f"sgfn{self.idx}_{'d' if self.dual else 'p'}"

    def site(self, block: str, index: int, message: str) -> int:
        self.o.sites.append(Site(self.fn.name, block, index, message))
        return len(self.o.sites)

    def zero_ret(self) -> str:
        return "sg_zero<D>()" if self.dual else "(T)0"

    def fail(self, sid: int) -> str:
        return f"{{ sg_err = {sid}; return {self.zero_ret()}; }}"

    # ---------------------------------------------------------- types
    def infer(self):
        """Result kinds of every instruction (scalar subset of ops.py typing)."""
        changed = True
        while changed:
            changed = False
            for b in self.fn.blocks:
                for ins in b.body:
                    if ins.result in self.types:
                        continue
                    k = self.kind_of_result(ins)
                    if k is not None:
                        self.types[ins.result] = k
                        changed = True
        for b in self.fn.blocks:
            for ins in b.body:
                if ins.result not in self.types:
                    raise CodegenError(
                        f"@{self.fn.name}: cannot type %{self.fn.value_name(ins.result)}")

    def kind_of_result(self, ins):
        op, a = ins.op, ins.operands
        if op not in _SCALAR_OPS:
            raise CodegenError(
                f"op '{op}' is not scalar; forward mode runs scalar code only")
        if op == "const":
            k = kind_of(ins.attrs["ty"])
            if k not in ("f64", "i64", "bool"):
                raise CodegenError(f"{ins.attrs['ty']} constant in scalar code")
            return k
        if op == "call":
            callee = self.o.module.get(ins.attrs["fn"].name)
            if len(callee.results) != 1:
                raise CodegenError(f"call: @{callee.name} must have exactly one result")
            return kind_of(callee.results[0])
        if any(x not in self.types for x in a):
            return None
        ks = [self.types[x] for x in a]
        if op in ("add", "sub", "mul"):
            return "i64" if ks == ["i64", "i64"] else "f64"
        if op in ("div", "exp", "log", "tanh", "sigmoid", "relu", "pow_int", "itof"):
            if op == "div" and ks == ["i64", "i64"]:
                raise CodegenError("div is not defined on i64")
            return "f64"
        if op == "neg":
            return ks[0]
        if op in ("lt", "gt", "eq"):
            return "bool"
        if op == "select":
            if ks[0] != "bool":
                raise CodegenError("select over a mask in scalar code")
            return ks[1]
        return None

    # ------------------------------------------------------ emission
    def emit(self) -> str:
        fn = self.fn
        self.infer()
        cyc = _cyclic(fn)
        rkind = kind_of(fn.results[0])
        rty = self.ctype(rkind)
        params = [f"{self.ctype(kind_of(t))} a{vid}" for vid, t in fn.params]
        params += ["int& sg_err", "long long& sg_steps"]
        L = self.lines
        L.append(f"__device__ __forceinline__ {rty} {self.fname}({', '.join(params)}) {{")
        # declare every value up front: gotos may not jump over initialisations
        for vid, kind in sorted(self.types.items()):
            L.append(f"  {self.ctype(kind)} {self.v(vid)};")
        for vid, _ in fn.params:
            L.append(f"  {self.v(vid)} = a{vid};")
        for b in fn.blocks:
            L.append(f" B_{b.name}:")
            if cyc:
                sid = self.site(b.name, len(b.body), "step limit exhausted")
                L.append(f"  sg_steps -= {len(b.body) + 1};")
                L.append(f"  if (sg_steps < 0) {self.fail(sid)}")
            for i, ins in enumerate(b.body):
                self.instr(b, i, ins)
            self.term(b)
        L.append("}")
        return "\n".join(L)

    def instr(self, b, i, ins):
        op = ins.op
        r = self.v(ins.result)
        a = [self.v(x) for x in ins.operands]
        ks = [self.types[x] for x in ins.operands]
        L = self.lines
        D = self.dual
        rk = self.types[ins.result]

        if op == "const":
            val = ins.attrs["value"]
            if rk == "f64":
                L.append(f"  {r} = sg_lift<{'D' if D else 'T'}>({_lit(float(val))});")
            elif rk == "i64":
                L.append(f"  {r} = {int(val)}LL;")
            else:
                L.append(f"  {r} = {'true' if val else 'false'};")
            return
        if op == "call":
            callee = self.o.module.get(ins.attrs["fn"].name)
            ci = self.o.index_of(callee)
            nm = f"sgfn{ci}_{'d' if D else 'p'}"
            args = ", ".join(a + ["sg_err", "sg_steps"])
            L.append(f"  {r} = {nm}({args});")
            L.append(f"  if (sg_err) return {self.zero_ret()};")
            return
        if op in ("lt", "gt", "eq"):
            sym = {"lt": "<", "gt": ">", "eq": "=="}[op]
            x = [self.prim(v, k) for v, k in zip(a, ks)]
            L.append(f"  {r} = ({x[0]} {sym} {x[1]});")
            return
        if op == "select":
            L.append(f"  {r} = {a[0]} ? {a[1]} : {a[2]};")
            return
        if rk == "i64":
            if op == "neg":
                L.append(f"  {r} = -{a[0]};")
            else:
                sym = {"add": "+", "sub": "-", "mul": "*"}[op]
                L.append(f"  {r} = {a[0]} {sym} {a[1]};")
            return
        if op == "itof":
            L.append(f"  {r} = sg_lift<{'D' if D else 'T'}>((T){a[0]});")
            return

        # f64 arithmetic from here on
        if op == "div":
            sid = self.site(b.name, i, "division by zero")
            L.append(f"  if ({self.prim(a[1], 'f64')} == (T)0) {self.fail(sid)}")
        if op == "log":
            sid = self.site(b.name, i, "log of non-positive value")
            L.append(f"  if ({self.prim(a[0], 'f64')} <= (T)0) {self.fail(sid)}")
        if not D:
            L.append(f"  {r} = {self.primal_expr(op, a, ins)};")
        else:
            L.append(f"  {{ {self.dual_block(op, r, a, ins)} }}")

    def prim(self, v: str, kind: str) -> str:
        return f"{v}.p" if (self.dual and kind == "f64") else v

    @staticmethod
    def primal_expr(op, a, ins) -> str:
        if op == "add":
            return f"{a[0]} + {a[1]}"
        if op == "sub":
            return f"{a[0]} - {a[1]}"
        if op == "mul":
            return f"{a[0]} * {a[1]}"
        if op == "div":
            return f"{a[0]} / {a[1]}"
        if op == "neg":
            return f"-{a[0]}"
        if op == "exp":
            return f"sg_exp({a[0]})"
        if op == "log":
            return f"sg_log({a[0]})"
        if op == "tanh":
            return f"sg_tanh({a[0]})"
        if op == "sigmoid":
            return f"sg_sigmoid({a[0]})"
        if op == "relu":
            return f"({a[0]} > (T)0 ? {a[0]} : (T)0)"
        if op == "pow_int":
            return f"sg_pow_int({a[0]}, {int(ins.attrs['n'])})"
        raise CodegenError(f"op '{op}' has no scalar lowering")

    @staticmethod
    def dual_block(op, r, a, ins) -> str:
        # formulas of forward_ad._DualRunner.dispatch, same operation order
        loop = "_Pragma(\"unroll\") for (int j = 0; j < SG_KT; ++j)"
        x = a[0]
        if op in ("add", "sub"):
            s = "+" if op == "add" else "-"
            y = a[1]
            return (f"{r}.p = {x}.p {s} {y}.p; {loop} {r}.t[j] = {x}.t[j] {s} {y}.t[j];")
        if op == "mul":
            y = a[1]
            return (f"{r}.p = {x}.p * {y}.p; "
                    f"{loop} {r}.t[j] = {x}.t[j] * {y}.p + {x}.p * {y}.t[j];")
        if op == "div":
            y = a[1]
            return (f"T p_ = {x}.p / {y}.p; {r}.p = p_; "
                    f"{loop} {r}.t[j] = ({x}.t[j] - p_ * {y}.t[j]) / {y}.p;")
        if op == "neg":
            return f"{r}.p = -{x}.p; {loop} {r}.t[j] = -{x}.t[j];"
        if op == "exp":
            return f"T y_ = sg_exp({x}.p); {r}.p = y_; {loop} {r}.t[j] = y_ * {x}.t[j];"
        if op == "log":
            return (f"{r}.p = sg_log({x}.p); {loop} {r}.t[j] = {x}.t[j] / {x}.p;")
        if op == "tanh":
            return (f"T y_ = sg_tanh({x}.p); T d_ = (T)1 - y_ * y_; {r}.p = y_; "
                    f"{loop} {r}.t[j] = d_ * {x}.t[j];")
        if op == "sigmoid":
            return (f"T y_ = sg_sigmoid({x}.p); T d_ = y_ * ((T)1 - y_); {r}.p = y_; "
                    f"{loop} {r}.t[j] = d_ * {x}.t[j];")
        if op == "relu":
            return (f"T d_ = {x}.p > (T)0 ? (T)1 : (T)0; "
                    f"{r}.p = {x}.p > (T)0 ? {x}.p : (T)0; {loop} {r}.t[j] = d_ * {x}.t[j];")
        if op == "pow_int":
            n = int(ins.attrs["n"])
            if n == 0:
                return f"{r}.p = sg_pow_int({x}.p, 0); {loop} {r}.t[j] = (T)0;"
            return (f"{r}.p = sg_pow_int({x}.p, {n}); "
                    f"T d_ = (T){n} * sg_pow_int({x}.p, {n - 1}); "
                    f"{loop} {r}.t[j] = d_ * {x}.t[j];")
        raise CodegenError(f"op '{op}' has no dual lowering")

    def assign(self, target_name: str, args) -> str:
        tgt = next(b for b in self.fn.blocks if b.name == target_name)
        if not tgt.params:
            return ""
        tmps = []
        outs = []
        for j, ((pv, _), av) in enumerate(zip(tgt.params, args)):
            ty = self.ctype(self.types[pv])
            tmps.append(f"{ty} t{j}_ = {self.v(av)};")
            outs.append(f"{self.v(pv)} = t{j}_;")
        return "{ " + " ".join(tmps + outs) + " } "

    def term(self, b):
        t = b.term
        L = self.lines
        if t is None:
            raise CodegenError(f"@{self.fn.name} ^{b.name}: missing terminator")
        if hasattr(t, "values"):
            L.append(f"  return {self.v(t.values[0])};")
        elif hasattr(t, "then_target"):
            c = self.v(t.cond)
            L.append(f"  if ({c}) {{ {self.assign(t.then_target, t.then_args)}goto B_{t.then_target}; }}")
            L.append(f"  else {{ {self.assign(t.else_target, t.else_args)}goto B_{t.else_target}; }}")
        else:
            L.append(f"  {self.assign(t.target, t.args)}goto B_{t.target};")


class _Lowerer:
    def __init__(self, module, dual: bool):
        self.module = module
        self.dual = dual
        self.order: list = []   # callees first
        self.sites: list[Site] = []

    def index_of(self, fn) -> int:
        for i, f in enumerate(self.order):
            if f.name == fn.name:
                return i
        raise CodegenError(f"@{fn.name} not scheduled")

    def schedule(self, fn, active=()):
        if fn.name in active:
            raise CodegenError(f"@{fn.name} is recursive; the GPU path needs a call DAG")
        if any(f.name == fn.name for f in self.order):
            return
        for b in fn.blocks:
            for ins in b.body:
                if ins.op == "call":
                    self.schedule(self.module.get(ins.attrs["fn"].name), active + (fn.name,))
        self.order.append(fn)


_PRELUDE = r"""
template <class X> __device__ __forceinline__ X sg_zero();
template <> __device__ __forceinline__ T sg_zero<T>() { return (T)0; }
template <> __device__ __forceinline__ D sg_zero<D>() { D d; d.p = (T)0;
  _Pragma("unroll") for (int j = 0; j < SG_KT; ++j) d.t[j] = (T)0; return d; }
template <class X> __device__ __forceinline__ X sg_lift(T v);
template <> __device__ __forceinline__ T sg_lift<T>(T v) { return v; }
template <> __device__ __forceinline__ D sg_lift<D>(T v) { D d; d.p = v;
  _Pragma("unroll") for (int j = 0; j < SG_KT; ++j) d.t[j] = (T)0; return d; }
__device__ __forceinline__ T sg_sigmoid(T x) { return (T)1 / ((T)1 + sg_exp(-x)); }
__device__ __forceinline__ T sg_pow_int(T x, int n) {
  T acc = (T)1; for (int i = 0; i < n; ++i) acc = acc * x; return acc; }
"""


def lower(module, name: str) -> Lowered:
    """Lower ``@name`` (and its callees) to primal + dual device code.

    The returned source expects the kernel skeleton's prelude (``T``,
    ``SG_K``, ``SG_KT``, ``D``, ``sg_exp``/``sg_log``/``sg_tanh``) and
    defines ``sg_entry_p`` / ``sg_entry_d`` over ``T x[SG_K]``.
    """
    fn = module.get(name)
    check_scalar_fn(fn)
    k = len(fn.params)
    chunks = [_PRELUDE]
    sites: list[Site] = []
    entries = {}
    for dual in (False, True):
        lo = _Lowerer(module, dual)
        lo.sites = sites
        lo.schedule(fn)
        for i, f in enumerate(lo.order):
            chunks.append(_FnLowering(lo, f, i).emit())
        entries[dual] = f"sgfn{lo.index_of(fn)}_{'d' if dual else 'p'}"
    xs = ", ".join(f"x[{i}]" for i in range(k))
    sep = ", " if k else ""
    chunks.append(
        "__device__ __forceinline__ void sg_entry_p(const T (&x)[SG_KT], T& y, int& sg_err,"
        " long long& sg_steps) {\n"
        f"  y = {entries[False]}({xs}{sep}sg_err, sg_steps);\n}}")
    seeds = []
    for i in range(k):
        seeds.append(f"  D a{i}; a{i}.p = x[{i}]; _Pragma(\"unroll\") for (int j = 0; j < SG_KT; ++j)"
                     f" a{i}.t[j] = (j == {i}) ? (T)1 : (T)0;")
    ds = ", ".join(f"a{i}" for i in range(k))
    chunks.append(
        "__device__ __forceinline__ void sg_entry_d(const T (&x)[SG_KT], T& y, T (&dy)[SG_KT],"
        " int& sg_err, long long& sg_steps) {\n" + "\n".join(seeds) + "\n"
        f"  D r = {entries[True]}({ds}{sep}sg_err, sg_steps);\n"
        "  y = r.p; _Pragma(\"unroll\") for (int j = 0; j < SG_KT; ++j) dy[j] = r.t[j];\n}")
    src = "\n\n".join(chunks) + "\n"
    key = hashlib.sha256(src.encode()).hexdigest()[:24]
    return Lowered(src, k, key, sites, name)
