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
    def __init__(self, owner: "_Lowerer", fn, index: int, is_entry: bool = False):
        self.o = owner
        self.is_entry = is_entry
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

    # ---------------------------------------------------- tangent lanes
    # Dual values carry K tangent lanes.  Seeds are one-hot (pack_rows,
    # forward_ad.py:178-191), so most lanes are structurally 0 or 1; a
    # forward dataflow pass over the CFG finds them and the emitter never
    # computes them (a 0 lane contributes 0*p, which equals 0 for every
    # finite primal p).  States: "Z" zero, "O" one, "V" computed.
    def lane_ref(self, vid: int, j: int):
        s = self.lanes[vid][j]
        if s == "V":
            return ("V", f"{self.v(vid)}.t[{j}]")
        return (s, "(T)1" if s == "O" else "(T)0")

    def dual_rule(self, op, ins, r, xs):
        """(primal statements, lane list) for an f64 op; xs = [(pexpr, [lane refs])]."""
        K = self.o.k
        P = f"{r}.p"
        pre = []
        out = []

        def lit(ln):
            return ln[1]

        if op in ("const", "itof"):
            return pre, [("Z", "(T)0")] * K
        if op == "pow_int" and int(ins.attrs["n"]) == 0:  # forward_ad.py:123-124
            return [f"{P} = sg_pow_int({xs[0][0]}, 0);"], [("Z", "(T)0")] * K
        (xp, xl) = xs[0]
        yp, yl = xs[1] if len(xs) > 1 else (None, None)
        for j in range(K):
            sx, ex = xl[j]
            if op == "add":
                sy, ey = yl[j]
                out.append((sy, ey) if sx == "Z" else (sx, ex) if sy == "Z"
                           else ("V", f"{ex} + {ey}"))
            elif op == "sub":
                sy, ey = yl[j]
                out.append((sx, ex) if sy == "Z" else ("V", f"-({ey})") if sx == "Z"
                           else ("V", f"{ex} - {ey}"))
            elif op == "mul":  # s*y.p + x.p*t  (forward_ad.py:81)
                sy, ey = yl[j]
                t1 = None if sx == "Z" else (yp if sx == "O" else f"{ex} * {yp}")
                t2 = None if sy == "Z" else (xp if sy == "O" else f"{xp} * {ey}")
                terms = [t for t in (t1, t2) if t is not None]
                out.append(("Z", "(T)0") if not terms else ("V", " + ".join(terms)))
            elif op == "div":  # (s - p*t)/y.p  (forward_ad.py:87-88)
                sy, ey = yl[j]
                if sy == "Z":
                    num = None if sx == "Z" else ex
                else:
                    pt = P if sy == "O" else f"{P} * {ey}"
                    num = f"-({pt})" if sx == "Z" else f"{ex} - {pt}"
                out.append(("Z", "(T)0") if num is None else ("V", f"({num}) / {yp}"))
            elif op == "neg":
                out.append(("Z", "(T)0") if sx == "Z" else ("V", f"-({ex})"))
            elif op == "log":
                out.append(("Z", "(T)0") if sx == "Z" else ("V", f"{ex} / {xp}"))
            elif op in ("exp",):
                out.append(("Z", "(T)0") if sx == "Z" else ("V", P if sx == "O" else f"{P} * {ex}"))
            elif op in ("tanh", "sigmoid", "relu", "pow_int"):
                out.append(("Z", "(T)0") if sx == "Z" else ("V", "d_" if sx == "O" else f"d_ * {ex}"))
            else:
                raise CodegenError(f"op '{op}' has no dual lowering")
        if op == "div":
            pre.append(f"{P} = {xp} / {yp};")
        elif op == "tanh":
            pre.append(f"{P} = sg_tanh({xp}); T d_ = (T)1 - {P} * {P};")
        elif op == "sigmoid":
            pre.append(f"{P} = sg_sigmoid({xp}); T d_ = {P} * ((T)1 - {P});")
        elif op == "relu":
            pre.append(f"T d_ = {xp} > (T)0 ? (T)1 : (T)0; {P} = {xp} > (T)0 ? {xp} : (T)0;")
        elif op == "pow_int":
            n = int(ins.attrs["n"])
            pre.append(f"{P} = sg_pow_int({xp}, {n}); T d_ = (T){n} * sg_pow_int({xp}, {n - 1});")
        else:
            pre.append(f"{P} = {self.primal_expr(op, [xp, yp], ins)};")
        return pre, out

    def lane_states_of(self, ins):
        op = ins.op
        K = self.o.k
        rk = self.types[ins.result]
        if rk != "f64":
            return None
        if op == "call":
            return ("V",) * K
        if op == "select":
            a, b = self.lanes[ins.operands[1]], self.lanes[ins.operands[2]]
            return tuple(x if x == y and x != "V" else "V" for x, y in zip(a, b))
        xs = []
        for o in ins.operands:
            if self.types[o] == "f64":
                xs.append(("p", [(s, "e") for s in self.lanes[o]]))
            else:
                xs.append(("p", [("Z", "0")] * K))
        _, lanes = self.dual_rule(op, ins, "r", xs or [("p", [("Z", "0")] * K)])
        return tuple(s for s, _ in lanes)

    def analyze_lanes(self):
        K = self.o.k
        fn = self.fn
        self.lanes = {}
        for i, (vid, ty) in enumerate(fn.params):
            if kind_of(ty) == "f64":
                if self.is_entry:
                    self.lanes[vid] = tuple("O" if j == i else "Z" for j in range(K))
                else:
                    self.lanes[vid] = ("V",) * K
        blocks = {b.name: b for b in fn.blocks}

        def edges(b):
            t = b.term
            if hasattr(t, "then_target"):
                return [(t.then_target, t.then_args), (t.else_target, t.else_args)]
            if hasattr(t, "target"):
                return [(t.target, t.args)]
            return []

        def ready(b):
            return all(self.types[v] != "f64" or v in self.lanes for v, _ in b.params)

        changed = True
        while changed:
            changed = False
            for b in fn.blocks:
                if not ready(b):
                    continue
                for ins in b.body:
                    st = self.lane_states_of(ins)
                    if st is not None:
                        self.lanes[ins.result] = st
                for tgt, args in edges(b):
                    for (pv, _), av in zip(blocks[tgt].params, args):
                        if self.types[pv] != "f64":
                            continue
                        new = self.lanes[av]
                        old = self.lanes.get(pv)
                        if old is not None:
                            new = tuple(x if x == y else "V" for x, y in zip(old, new))
                        if new != old:
                            self.lanes[pv] = new
                            changed = True
        # unreachable blocks: anything goes
        for b in fn.blocks:
            for v, _ in b.params:
                if self.types[v] == "f64" and v not in self.lanes:
                    self.lanes[v] = ("V",) * K
            for ins in b.body:
                if self.types[ins.result] == "f64" and ins.result not in self.lanes:
                    self.lanes[ins.result] = ("V",) * K
        for b in fn.blocks:  # final states for every instruction
            for ins in b.body:
                st = self.lane_states_of(ins)
                if st is not None:
                    self.lanes[ins.result] = st

    def materialize(self, vid: int) -> str:
        """Write the literal value of virtual (Z/O) lanes into the struct."""
        if not self.dual or self.types[vid] != "f64":
            return ""
        return " ".join(f"{self.v(vid)}.t[{j}] = {'(T)1' if s == 'O' else '(T)0'};"
                        for j, s in enumerate(self.lanes[vid]) if s != "V")

    # ------------------------------------------------------ emission
    def emit(self) -> str:
        fn = self.fn
        self.infer()
        if self.dual:
            self.analyze_lanes()
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
                L.append(f"  {r}{'.p' if D else ''} = {_lit(float(val))};")
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
            mats = " ".join(self.materialize(o) for o in ins.operands)
            if mats.strip():
                L.append(f"  {mats}")
            L.append(f"  {r} = {nm}({args});")
            L.append(f"  if (sg_err) return {self.zero_ret()};")
            return
        if op in ("lt", "gt", "eq"):
            sym = {"lt": "<", "gt": ">", "eq": "=="}[op]
            x = [self.prim(v, k) for v, k in zip(a, ks)]
            L.append(f"  {r} = ({x[0]} {sym} {x[1]});")
            return
        if op == "select":
            if D and rk == "f64":
                o1, o2 = ins.operands[1], ins.operands[2]
                parts = [f"{r}.p = {a[0]} ? {a[1]}.p : {a[2]}.p;"]
                for j, st in enumerate(self.lanes[ins.result]):
                    if st == "V":
                        parts.append(f"{r}.t[{j}] = {a[0]} ? {self.lane_ref(o1, j)[1]} : "
                                     f"{self.lane_ref(o2, j)[1]};")
                L.append("  " + " ".join(parts))
            else:
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
            L.append(f"  {r}{'.p' if D else ''} = (T){a[0]};")
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
            xs = [(f"{self.v(o)}.p", [self.lane_ref(o, j) for j in range(self.o.k)])
                  for o in ins.operands]
            pre, lanes = self.dual_rule(op, ins, r, xs)
            body = pre + [f"{r}.t[{j}] = {e};" for j, (st, e) in enumerate(lanes) if st == "V"]
            L.append("  { " + " ".join(body) + " }")

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

    def assign(self, target_name: str, args) -> str:
        tgt = next(b for b in self.fn.blocks if b.name == target_name)
        if not tgt.params:
            return ""
        tmps = []
        outs = []
        for j, ((pv, _), av) in enumerate(zip(tgt.params, args)):
            if self.dual and self.types[pv] == "f64":
                tmps.append(f"T t{j}_p = {self.v(av)}.p;")
                outs.append(f"{self.v(pv)}.p = t{j}_p;")
                for l, st in enumerate(self.lanes[pv]):
                    if st == "V":
                        tmps.append(f"T t{j}_{l} = {self.lane_ref(av, l)[1]};")
                        outs.append(f"{self.v(pv)}.t[{l}] = t{j}_{l};")
                continue
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
            m = self.materialize(t.values[0])
            L.append(f"  {m + ' ' if m else ''}return {self.v(t.values[0])};")
        elif hasattr(t, "then_target"):
            c = self.v(t.cond)
            L.append(f"  if ({c}) {{ {self.assign(t.then_target, t.then_args)}goto B_{t.then_target}; }}")
            L.append(f"  else {{ {self.assign(t.else_target, t.else_args)}goto B_{t.else_target}; }}")
        else:
            L.append(f"  {self.assign(t.target, t.args)}goto B_{t.target};")


class _Lowerer:
    def __init__(self, module, dual: bool, k: int = 0):
        self.module = module
        self.dual = dual
        self.k = max(1, k)
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
        lo = _Lowerer(module, dual, k)
        lo.sites = sites
        lo.schedule(fn)
        for i, f in enumerate(lo.order):
            chunks.append(_FnLowering(lo, f, i, is_entry=(f.name == fn.name)).emit())
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
