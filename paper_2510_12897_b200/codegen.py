"""Per-pattern kernel generator: tape -> straight-line fp64 CUDA.

For every distinct tape pattern (:meth:`.tape.TermTape.pattern_key`) this
module *symbolically executes* the reference's four per-term passes --
``values`` (``autodiff.py:127-168``), ``adjoints`` (173-218), ``slot_sums``
(220-226), ``tangents`` (231-297), ``adjoint_tangents`` (302-382) with the
``_acc``/``_accd`` accumulators (385-396) -- and records every floating-point
operation the reference would perform on an array as one CUDA statement.

Values the reference holds as Python scalars are folded here, at generation
time, with the same arithmetic (numpy / IEEE double).  In particular
``_is_zero`` (``autodiff.py:69-70``) -- which is true only for a *scalar*
structural zero -- is decided exactly as the reference decides it, so
structural zeros stay literal and the emitted statement sequence performs
the reference's IEEE operations in the reference's order.  Built with
``--fmad=false``, a generated kernel therefore reproduces the reference
bit-for-bit except where the reference calls a transcendental: sin/cos use
the correctly-rounded ``exa_sincos`` (glibc, the reference's libm, is CR on
~99.8% of arguments); exp/log/general pow use CUDA's libdevice.

Symbolic value kinds:

* ``float``  -- a reference *scalar* (Python float / np.float64);
* ``Arr``    -- a reference *array* whose every element is a known constant
  (``np.ones``/``np.zeros`` and arithmetic on them);
* ``Sym``    -- a reference array with data-dependent values: a CUDA local.

Only exact rewrites are applied (x*1 -> x, x*-1 -> -x, x/1 -> x, x-(+0) -> x);
``0.0 + x`` is kept because it maps -0.0 to +0.0 exactly like numpy does.
"""

from __future__ import annotations

import math
import re
import os

import numpy as np

_SIN_COS = ("sin", "cos")


def _zero_const(v) -> bool:
    """A generation-time constant 0 (structural zero of a derivative)."""
    if isinstance(v, Sym):
        return False
    return float(v.value if isinstance(v, Arr) else v) == 0.0


def _elem(T: str, r: str) -> str:
    """Element (per-element table row) of record r: r / per, or the key index
    column's block position / per - g0 (device._periodic)."""
    return f"({T}.kcol < 0 ? {r} / {T}.per : __ldg({T}.ix[{T}.kcol] + {r}) / {T}.per - {T}.g0)"


def _inst(T: str, r: str) -> str:
    """Instance / period of record r within its element."""
    return f"({T}.kcol < 0 ? {r} % {T}.per : __ldg({T}.ix[{T}.kcol] + {r}) % {T}.per)"


def _field_load(T: str, fi: int, r: str) -> str:
    """Field fi of term T at record r.  Per-element columns (``T.fmask`` bit
    fi, batched element-major models) are read at the record's element; the
    selection folds at compile time in model-specialised modules (T is built
    from literals).  The per-record form stays an evict-first candidate
    (jit._cache_hints rewrites ``__ldg(T.f[..] + r)``)."""
    return f"((({T}.fmask >> {fi}) & 1u) ? __ldg({T}.f[{fi}] + {_elem(T, r)}) : __ldg({T}.f[{fi}] + {r}))"


def _index_load(T: str, c: int, r: str) -> str:
    """Index column c of term T at record r (per-element columns: the
    element's g(e) * per + the record's instance)."""
    return (f"((({T}.imask >> {c}) & 1u) ? __ldg({T}.ix[{c}] + {_elem(T, r)}) + {_inst(T, r)}"
            f" : __ldg({T}.ix[{c}] + {r}))")


# Zero-sign mode of the generated code.  Exact: every 0 + x of the reference
# and the structural zeros w * 0 with their weight's sign (bit-identical J/H,
# NaN / inf multipliers propagate like the reference's).  Relaxed: the former
# dropped in derivative space (see Gen.bin), the latter written as +0.0
# without loading the weight -- IEEE-equal for finite weights.  The default is
# EXA_EXACT_ZERO_SIGN (1 = exact); a layout may choose per plan (relax=...).
_DERIV_ZERO_ELISION = os.environ.get("EXA_EXACT_ZERO_SIGN", "0") != "1"
# term-group members' multipliers (their own rows: each read once per set) are
# loaded evict-first like the parameters (case13659 6.08 -> 5.99 us, MP96 39.4
# -> 38.9); balance-row multipliers (augments, row buckets) are shared and
# keep __ldg
_WGT_CS = os.environ.get("EXA_WGT_CS", "1") == "1"


class Arr:
    __slots__ = ("value",)

    def __init__(self, value):
        self.value = float(value)


class Sym:
    """A data-dependent value held in a CUDA local.  ``nz`` records that the
    value can never be -0.0 (then ``0.0 + x == x`` bitwise and the add is
    dropped): true for ``0 + x``, for any sum/difference whose first operand
    (or, for sums, either operand) can never be -0.0 -- IEEE round-to-nearest
    gives -0.0 from a + b only for (-0) + (-0) and from a - b only for
    (-0) - (+0) -- and for cos(), which is never zero for a double argument."""

    __slots__ = ("name", "nz")

    def __init__(self, name: str, nz: bool = False):
        self.name = name
        self.nz = nz


def _nz(v) -> bool:
    """Value can never be -0.0."""
    if isinstance(v, Sym):
        return v.nz
    c = v.value if isinstance(v, Arr) else float(v)
    return not (c == 0.0 and math.copysign(1.0, c) < 0)


def _is_zero(v) -> bool:
    """Reference ``_is_zero``: a *scalar* equal to zero."""
    return isinstance(v, float) and not isinstance(v, Arr) and v == 0.0


def lit(v: float) -> str:
    v = float(v)
    if math.isnan(v):
        return "__longlong_as_double(0x7ff8000000000000LL)"
    if math.isinf(v):
        return "__longlong_as_double(0x7ff0000000000000LL)" if v > 0 else "__longlong_as_double(0xfff0000000000000LL)"
    h = v.hex()
    return f"({h})" if h.startswith("-") else h


def _fold(op, a, b):
    """IEEE double fold of a binary op on two known constants (numpy semantics)."""
    with np.errstate(all="ignore"):
        x, y = np.float64(a), np.float64(b)
        if op == "add":
            return float(x + y)
        if op == "sub":
            return float(x - y)
        if op == "mul":
            return float(x * y)
        if op == "div":
            return float(x / y)
    raise ValueError(op)


class Gen:
    """Emits statements; every array-valued operation becomes one local."""

    def __init__(self):
        self.lines: list[str] = []
        self.n = 0
        self.memo: dict = {}
        self.sincos: dict = {}
        self.diffs: dict = {}  # name of a Sym defined as x - y -> (x, y)
        # derivative-space emission (see bin add); off while emitting values
        self.deriv = False
        self.checks: list = []

    def new(self, expr: str, nz: bool = False) -> Sym:
        got = self.memo.get(expr)
        if got is not None:
            return got
        name = f"t{self.n}"
        self.n += 1
        self.lines.append(f"  const double {name} = {expr};")
        s = Sym(name, nz)
        self.memo[expr] = s
        return s

    @staticmethod
    def r(v) -> str:
        if isinstance(v, Sym):
            return v.name
        if isinstance(v, Arr):
            return lit(v.value)
        return lit(v)

    # -- arithmetic on symbolic values -----------------------------------
    def bin(self, op, a, b):
        sa, sb = isinstance(a, Sym), isinstance(b, Sym)
        if not sa and not sb:
            val = _fold(op, a.value if isinstance(a, Arr) else a, b.value if isinstance(b, Arr) else b)
            return Arr(val) if (isinstance(a, Arr) or isinstance(b, Arr)) else val
        # exact rewrites only
        ca = None if sa else (a.value if isinstance(a, Arr) else float(a))
        cb = None if sb else (b.value if isinstance(b, Arr) else float(b))
        if op == "mul":
            if cb == 1.0:
                return a
            if ca == 1.0:
                return b
            if cb == -1.0:
                return self.neg(a)
            if ca == -1.0:
                return self.neg(b)
        elif op == "div":
            if cb == 1.0:
                return a
        elif op == "sub":
            if cb == 0.0 and not math.copysign(1.0, cb) < 0:
                return a
        elif op == "add":
            # x + (-0) == x;  (+0) + x == x unless x is -0.0.  In derivative
            # space (adjoints, tangents, their slot sums) the sign of a zero can
            # only ever reach the sign of an exactly-zero output -- derivative
            # quantities are only added and multiplied, never divided by or fed
            # to a function -- so there the normalising 0 + x is dropped.
            if cb == 0.0 and (math.copysign(1.0, cb) < 0 or _nz(a) or self.deriv):
                return a
            if ca == 0.0 and (math.copysign(1.0, ca) < 0 or _nz(b) or self.deriv):
                return b
        sym = {"add": "+", "sub": "-", "mul": "*", "div": "/"}[op]
        nz = (op == "add" and (_nz(a) or _nz(b))) or (op == "sub" and _nz(a))
        out = self.new(f"{self.r(a)} {sym} {self.r(b)}", nz)
        if op == "sub":
            self.diffs[out.name] = (self.r(a), self.r(b))
        return out

    def add(self, a, b):
        return self.bin("add", a, b)

    def sub(self, a, b):
        return self.bin("sub", a, b)

    def mul(self, a, b):
        return self.bin("mul", a, b)

    def div(self, a, b):
        return self.bin("div", a, b)

    def neg(self, a):
        if isinstance(a, Sym):
            return self.new(f"-{a.name}")
        if isinstance(a, Arr):
            return Arr(-a.value)
        return float(-np.float64(a))

    def fn(self, name, a):
        """np.<name>(a) for sin, cos, exp, log, sqrt."""
        if not isinstance(a, Sym):
            c = a.value if isinstance(a, Arr) else a
            with np.errstate(all="ignore"):
                val = float(getattr(np, name)(np.array([c], dtype=np.float64))[0])
            return Arr(val) if isinstance(a, Arr) else val
        if name in _SIN_COS:
            pair = self.sincos.get(a.name)
            if pair is None and a.name in self.diffs:
                # sin(y - x) = -sin(x - y), cos(y - x) = cos(x - y): IEEE subtraction is
                # exactly antisymmetric and exa_sincos is odd/even symmetric
                lhs, rhs = self.diffs[a.name]
                other = self.memo.get(f"{rhs} - {lhs}")
                if other is not None and other.name in self.sincos:
                    s_o, c_o = self.sincos[other.name]
                    pair = (self.new(f"-{s_o.name}"), c_o)
                    self.sincos[a.name] = pair
            if pair is None:
                s, c = f"s_{a.name}", f"c_{a.name}"
                self.lines.append(f"  double {s}, {c}; exa_sincos({a.name}, &{s}, &{c});")
                pair = (Sym(s), Sym(c, nz=True))  # cos(x) != 0 for every double x
                self.sincos[a.name] = pair
            return pair[0] if name == "sin" else pair[1]
        return self.new(f"{name}({a.name})")

    def powi(self, a, n: int):
        """np.power(a, n) for a Python int n (numpy: n=2 -> square, 1 -> copy,
        0 -> ones, -1 -> reciprocal; measured bit-identical)."""
        if not isinstance(a, Sym):
            c = a.value if isinstance(a, Arr) else a
            with np.errstate(all="ignore"):
                val = float(np.power(np.array([c], dtype=np.float64), n)[0])
            return Arr(val) if isinstance(a, Arr) else val
        if n == 1:
            return a
        if n == 0:
            return Arr(1.0)
        if n == 2:
            return self.new(f"{a.name} * {a.name}")
        if n == -1:
            return self.new(f"1.0 / {a.name}")
        return self.new(f"exa_powi({a.name}, {int(n)})")

    def pow(self, a, b):
        if not isinstance(a, Sym) and not isinstance(b, Sym):
            ca = a.value if isinstance(a, Arr) else a
            cb = b.value if isinstance(b, Arr) else b
            with np.errstate(all="ignore"):
                val = float(np.power(np.array([ca]), np.array([cb]))[0])
            return Arr(val) if (isinstance(a, Arr) or isinstance(b, Arr)) else val
        return self.new(f"pow({self.r(a)}, {self.r(b)})")

    # -- domain checks (values pass only) ----------------------------------
    def check(self, kind, v, instr_idx):
        """kind 'pos' (log/sqrt/pow) or 'nz' (div/ipow<0)."""
        if isinstance(v, Sym):
            cond = f"!({v.name} > 0.0)" if kind == "pos" else f"{v.name} == 0.0"
            self.lines.append(f"  if ({cond}) EXA_DOMAIN({instr_idx});")
            self.checks.append(instr_idx)
        else:
            c = v.value if isinstance(v, Arr) else v
            bad = (not (c > 0.0)) if kind == "pos" else (c == 0.0)
            if bad:
                rec = "EXA_REC_ALL" if not isinstance(v, Arr) else "EXA_REC_FIRST"
                self.lines.append(f"  EXA_DOMAIN_AT({instr_idx}, {rec});")
                self.checks.append(instr_idx)


class PatternCode:
    """Generated source for one tape pattern plus what it needs at run time."""

    def __init__(self, pid: int, tape, field_count: int, index_count: int, slot_struct, relax: bool | None = None):
        self.pid = pid
        self.relax = _DERIV_ZERO_ELISION if relax is None else bool(relax)
        self.tape = tape
        self.nf = field_count
        self.ni = index_count
        self.slot_struct = slot_struct  # per slot: (block class, index column)
        self.k = tape.k
        self.has_checks = False
        self.source = self._generate()

    # ---------------------------------------------------------------- passes
    def _values(self, g: Gen, loads):
        v = [None] * len(self.instr)
        for p, ins in enumerate(self.instr):
            op = ins[0]
            if op == "const":
                v[p] = float(ins[1])
            elif op == "field":
                v[p] = loads["field"][ins[1]]
            elif op == "var":
                v[p] = loads["var"][ins[1]]
            elif op == "neg":
                v[p] = g.neg(v[ins[1]])
            elif op in ("sin", "cos", "exp"):
                v[p] = g.fn(op, v[ins[1]])
            elif op in ("log", "sqrt"):
                g.check("pos", v[ins[1]], p)
                v[p] = g.fn(op, v[ins[1]])
            elif op in ("add", "sub", "mul"):
                v[p] = g.bin(op, v[ins[1]], v[ins[2]])
            elif op == "div":
                g.check("nz", v[ins[2]], p)
                v[p] = g.div(v[ins[1]], v[ins[2]])
            elif op == "ipow":
                n = ins[2]
                if n < 0:
                    g.check("nz", v[ins[1]], p)
                v[p] = g.mul(v[ins[1]], v[ins[1]]) if n == 2 else g.powi(v[ins[1]], n)
            elif op == "pow":
                g.check("pos", v[ins[1]], p)
                v[p] = g.pow(v[ins[1]], v[ins[2]])
            else:
                raise ValueError(op)
        return v

    def _adjoints(self, g: Gen, v):
        adj = [None] * len(self.instr)
        adj[-1] = Arr(1.0)

        def acc(at, val):
            adj[at] = val if adj[at] is None else g.add(adj[at], val)

        for p in range(len(self.instr) - 1, -1, -1):
            a_p = adj[p]
            ins = self.instr[p]
            op = ins[0]
            if a_p is None or op in ("const", "field", "var"):
                continue
            a = ins[1]
            if op == "neg":
                acc(a, g.neg(a_p))
            elif op == "sin":
                acc(a, g.mul(a_p, g.fn("cos", v[a])))
            elif op == "cos":
                acc(a, g.mul(g.neg(a_p), g.fn("sin", v[a])))
            elif op == "exp":
                acc(a, g.mul(a_p, v[p]))
            elif op == "log":
                acc(a, g.div(a_p, v[a]))
            elif op == "sqrt":
                acc(a, g.div(a_p, g.mul(2.0, v[p])))
            elif op == "add":
                acc(a, a_p)
                acc(ins[2], a_p)
            elif op == "sub":
                acc(a, a_p)
                acc(ins[2], g.neg(a_p))
            elif op == "mul":
                acc(a, g.mul(a_p, v[ins[2]]))
                acc(ins[2], g.mul(a_p, v[a]))
            elif op == "div":
                b = ins[2]
                acc(a, g.div(a_p, v[b]))
                acc(b, g.div(g.mul(g.neg(a_p), v[p]), v[b]))
            elif op == "ipow":
                n = ins[2]
                if n != 0:
                    acc(a, g.mul(g.mul(a_p, float(n)), g.powi(v[a], n - 1)))
            else:  # pow
                b = ins[2]
                acc(a, g.div(g.mul(g.mul(a_p, v[b]), v[p]), v[a]))
                acc(b, g.mul(g.mul(a_p, v[p]), g.fn("log", v[a])))
        return adj

    def _slot_sums(self, g: Gen, per_node):
        out = [Arr(0.0) for _ in range(self.k)]
        for p, ins in enumerate(self.instr):
            if ins[0] == "var" and per_node[p] is not None:
                out[ins[1]] = g.add(out[ins[1]], per_node[p])
        return out

    def _tangents(self, g: Gen, v, seed):
        Z = _is_zero
        t = [0.0] * len(self.instr)
        for p, ins in enumerate(self.instr):
            op = ins[0]
            if op == "var":
                t[p] = 1.0 if ins[1] == seed else 0.0
                continue
            if op in ("const", "field"):
                t[p] = 0.0
                continue
            ta = t[ins[1]]
            if op == "neg":
                t[p] = 0.0 if Z(ta) else g.neg(ta)
            elif op == "sin":
                t[p] = 0.0 if Z(ta) else g.mul(g.fn("cos", v[ins[1]]), ta)
            elif op == "cos":
                t[p] = 0.0 if Z(ta) else g.mul(g.neg(g.fn("sin", v[ins[1]])), ta)
            elif op == "exp":
                t[p] = 0.0 if Z(ta) else g.mul(v[p], ta)
            elif op == "log":
                t[p] = 0.0 if Z(ta) else g.div(ta, v[ins[1]])
            elif op == "sqrt":
                t[p] = 0.0 if Z(ta) else g.div(ta, g.mul(2.0, v[p]))
            elif op == "add":
                tb = t[ins[2]]
                t[p] = tb if Z(ta) else (ta if Z(tb) else g.add(ta, tb))
            elif op == "sub":
                tb = t[ins[2]]
                t[p] = ta if Z(tb) else (g.neg(tb) if Z(ta) else g.sub(ta, tb))
            elif op == "mul":
                tb = t[ins[2]]
                lhs = 0.0 if Z(ta) else g.mul(ta, v[ins[2]])
                rhs = 0.0 if Z(tb) else g.mul(v[ins[1]], tb)
                t[p] = 0.0 if (Z(lhs) and Z(rhs)) else g.add(lhs, rhs)
            elif op == "div":
                tb = t[ins[2]]
                if Z(ta) and Z(tb):
                    t[p] = 0.0
                else:
                    lhs = 0.0 if Z(ta) else g.div(ta, v[ins[2]])
                    rhs = 0.0 if Z(tb) else g.div(g.mul(v[p], tb), v[ins[2]])
                    t[p] = g.sub(lhs, rhs)
            elif op == "ipow":
                n = ins[2]
                if Z(ta) or n == 0:
                    t[p] = 0.0
                else:
                    t[p] = g.mul(g.mul(float(n), g.powi(v[ins[1]], n - 1)), ta)
            else:  # pow
                tb = t[ins[2]]
                if Z(ta) and Z(tb):
                    t[p] = 0.0
                else:
                    base, ex = v[ins[1]], v[ins[2]]
                    d = 0.0 if Z(ta) else g.div(g.mul(ex, ta), base)
                    if not Z(tb):
                        d = g.add(d, g.mul(g.fn("log", base), tb))
                    t[p] = g.mul(v[p], d)
        return t

    def _adjoint_tangents(self, g: Gen, v, adj, t):
        Z = _is_zero
        dot = [None] * len(self.instr)
        dot[-1] = 0.0

        def accd(at, d_parent, partial, a_parent, partial_dot):
            contrib = 0.0 if Z(d_parent) else g.mul(d_parent, partial)
            if not Z(partial_dot):
                contrib = g.add(contrib, g.mul(a_parent, partial_dot))
            dot[at] = contrib if dot[at] is None else g.add(dot[at], contrib)

        for p in range(len(self.instr) - 1, -1, -1):
            a_p, d_p = adj[p], dot[p]
            ins = self.instr[p]
            op = ins[0]
            if a_p is None or op in ("const", "field", "var"):
                continue
            a = ins[1]
            if op == "neg":
                accd(a, d_p, -1.0, a_p, 0.0)
            elif op == "sin":
                ta = t[a]
                pd = 0.0 if Z(ta) else g.mul(g.neg(g.fn("sin", v[a])), ta)
                accd(a, d_p, g.fn("cos", v[a]), a_p, pd)
            elif op == "cos":
                ta = t[a]
                pd = 0.0 if Z(ta) else g.mul(g.neg(g.fn("cos", v[a])), ta)
                accd(a, d_p, g.neg(g.fn("sin", v[a])), a_p, pd)
            elif op == "exp":
                accd(a, d_p, v[p], a_p, t[p])
            elif op == "log":
                ta = t[a]
                pd = 0.0 if Z(ta) else g.div(g.neg(ta), g.mul(v[a], v[a]))
                accd(a, d_p, g.div(1.0, v[a]), a_p, pd)
            elif op == "sqrt":
                tp = t[p]
                pd = 0.0 if Z(tp) else g.div(g.neg(tp), g.mul(g.mul(2.0, v[p]), v[p]))
                accd(a, d_p, g.div(1.0, g.mul(2.0, v[p])), a_p, pd)
            elif op == "add":
                accd(a, d_p, 1.0, a_p, 0.0)
                accd(ins[2], d_p, 1.0, a_p, 0.0)
            elif op == "sub":
                accd(a, d_p, 1.0, a_p, 0.0)
                accd(ins[2], d_p, -1.0, a_p, 0.0)
            elif op == "mul":
                b = ins[2]
                accd(a, d_p, v[b], a_p, t[b])
                accd(b, d_p, v[a], a_p, t[a])
            elif op == "div":
                b = ins[2]
                den = v[b]
                ta, tb = t[a], t[b]
                pda = 0.0 if Z(tb) else g.div(g.neg(tb), g.mul(den, den))
                if Z(ta) and Z(tb):
                    pdb = 0.0
                else:
                    pdb = g.neg(0.0 if Z(ta) else g.div(ta, g.mul(den, den)))
                    if not Z(tb):
                        pdb = g.add(pdb, g.div(g.mul(g.mul(2.0, v[p]), tb), g.mul(den, den)))
                accd(a, d_p, g.div(1.0, den), a_p, pda)
                accd(b, d_p, g.div(g.neg(v[p]), den), a_p, pdb)
            elif op == "ipow":
                n = ins[2]
                if n == 0:
                    continue
                base, ta = v[a], t[a]
                part = g.mul(float(n), g.powi(base, n - 1))
                if n <= 1 or Z(ta):
                    pd = 0.0
                else:
                    pd = g.mul(g.mul(float(n * (n - 1)), g.powi(base, n - 2)), ta)
                accd(a, d_p, part, a_p, pd)
            else:  # pow
                b = ins[2]
                base, ex = v[a], v[b]
                ta, tb, tp = t[a], t[b], t[p]
                pa = g.div(g.mul(ex, v[p]), base)
                pb = g.mul(v[p], g.fn("log", base))
                pda = 0.0 if Z(tb) else g.div(g.mul(tb, v[p]), base)
                if not Z(tp):
                    pda = g.add(pda, g.div(g.mul(ex, tp), base))
                if not Z(ta):
                    pda = g.sub(pda, g.div(g.mul(g.mul(ex, v[p]), ta), g.mul(base, base)))
                pdb = 0.0 if Z(tp) else g.mul(tp, g.fn("log", base))
                if not Z(ta):
                    pdb = g.add(pdb, g.div(g.mul(v[p], ta), base))
                accd(a, d_p, pa, a_p, pda)
                accd(b, d_p, pb, a_p, pdb)
        return dot

    # -------------------------------------------------------------- emission
    def _generate(self) -> str:
        self.instr = self.tape_norm()
        k = self.k
        g = Gen()
        # loads: fields and gathered variables (each slot once)
        loads = {"field": {}, "var": []}
        pre = []
        for fi, fname in enumerate(self.tape.field_names):
            pre.append(f"  const double f{fi} = {_field_load('T', fi, 'r')};")
            loads["field"][fname] = Sym(f"f{fi}")
        for ii in range(self.ni):
            pre.append(f"  const int i{ii} = {_index_load('T', ii, 'r')};")
        pre_wait = len(pre)
        for s, (_, ic) in enumerate(self.slot_struct):
            pre.append(f"  const int c{s} = T.voff[{s}] + i{ic};")
            pre.append(f"  const double x{s} = __ldg(A.x + c{s});")
            loads["var"].append(Sym(f"x{s}"))
        v = self._values(g, loads)
        value_lines = list(g.lines)
        value_root = v[-1]
        self.root_const = None if isinstance(value_root, (Sym, Arr)) else float(value_root)
        self.has_checks = bool(g.checks)
        n_value_lines = len(g.lines)

        # first order
        g.deriv = self.relax
        adj = self._adjoints(g, v) if k else None
        grads = self._slot_sums(g, adj) if k else []
        n_grad_lines = len(g.lines)
        # second order: one forward-over-reverse sweep per seed slot
        by_seed = []
        for seed in range(k):
            t = self._tangents(g, v, seed)
            by_seed.append(self._slot_sums(g, self._adjoint_tangents(g, v, adj, t)))
        body_grad = g.lines[n_value_lines:n_grad_lines]
        body_hess = g.lines[n_grad_lines:]
        # x- and y-independent outputs (every record, every call): constant J
        # slots and, under the zero-sign relaxation, the structural-zero
        # Hessian pairs (written as +0.0).  The host path fills these into the
        # caller's arrays instead of copying them over PCIe (exa_eval_set_host).
        self.jconst = {s: float(grads[s].value if isinstance(grads[s], Arr) else grads[s])
                       for s in range(k) if not isinstance(grads[s], Sym)}
        # structural-zero Hessian pairs: (pair, the constant z) -- the slot's
        # value is weight * z, +0.0 under the relaxation (self.hzero); in the
        # exact mode the host path computes weight * z from the caller's
        # multipliers (self.hzero_w)
        self.hzero, self.hzero_w = [], []
        pair = 0
        for i in range(k):
            for j in range(i + 1):
                val = by_seed[j][i]
                if _zero_const(val):
                    (self.hzero if self.relax else self.hzero_w).append(
                        pair if self.relax else (pair, float(val.value if isinstance(val, Arr) else val)))
                pair += 1

        out = []
        pid = self.pid
        R = Gen.r
        # value-only function (row sums of augment-target rows, objective values)
        out.append(f"template <int LDH = 1>\n__device__ __forceinline__ double exa_val_{pid}(const ExaTerm& T, int r, const ExaArgs& A, int rank) {{")
        out.extend(pre)
        out.extend(value_lines)
        out.append(f"  return {R(value_root)};")
        out.append("}")

        # full term function, MODE-templated; unused temps are dead code.  All
        # loads (including the Hessian weight) are issued before the first
        # store, and outputs are __restrict__, so several records per thread
        # (light patterns) overlap their memory latency.
        # ``ro`` (default r): record index of the OUTPUT slots and the Hessian
        # weight, when the term's fields are read from a permuted copy (row buckets)
        out.append(f"template <int MODE, int LDH = 1>\n__device__ __forceinline__ void exa_term_{pid}(const ExaTerm& T, int r, const ExaArgs& A, int rank, int ro = -1) {{")
        out.append("  const int o = ro < 0 ? r : ro;")
        out.append("  double* __restrict__ Cout = A.c;")
        out.append("  double* __restrict__ Jout = A.J;")
        out.append("  double* __restrict__ Hout = A.H;")
        out.extend(pre[:pre_wait])
        out.append("  EXA_GRID_WAIT();")
        out.extend(pre[pre_wait:])
        if k:
            out.append("  const double wgt = !(MODE & EXA_M_HESS) ? 0.0 : (T.kind == EXA_OBJ) ? A.w"
                       " : __ldg(A.y + (T.rows ? __ldg(T.rows + o) : T.row_offset + o));")
        out.extend(value_lines)
        out.append("  if (MODE & (EXA_M_CONS | EXA_M_OBJV)) {")
        out.append(f"    const double root = {R(value_root)};")
        out.append("    if ((MODE & EXA_M_CONS) && T.cons_direct) Cout[T.row_offset + o] = 0.0 + root;")
        out.append("    if ((MODE & EXA_M_OBJV) && T.kind == EXA_OBJ) A.V[T.scr0 + o] = root;")
        out.append("  }")
        if k:
            out.append("  if (MODE & (EXA_M_JAC | EXA_M_GRAD | EXA_M_HESS)) {")
            out.extend("  " + l for l in body_grad)
            out.append("    if ((MODE & EXA_M_JAC) && T.kind != EXA_OBJ) {")
            for s in range(k):
                out.append(f"      Jout[T.jac0 + {s}LL * T.nrec + o] = {R(grads[s])};")
            out.append("    }")
            out.append("    if ((MODE & EXA_M_GRAD) && T.kind == EXA_OBJ) {")
            for s in range(k):
                out.append(f"      A.G[T.scr0 + {s}LL * T.nrec + o] = {R(grads[s])};")
            out.append("    }")
            out.append("    if (MODE & EXA_M_HESS) {")
            out.extend("    " + l for l in body_hess)
            pair = 0
            for i in range(k):
                for j in range(i + 1):
                    val = by_seed[j][i]
                    expr = R(val)
                    bi, bj = self.slot_struct[i][0], self.slot_struct[j][0]
                    if i != j and bi == bj:
                        expr = f"(c{i} == c{j} ? {expr} * 2.0 : {expr})"
                    if self.relax and _zero_const(val):
                        out.append(f"      Hout[T.hess0 + {pair}LL * T.nrec + o] = 0.0;  // structural zero")
                    else:
                        out.append(f"      Hout[T.hess0 + {pair}LL * T.nrec + o] = wgt * {expr};")
                    pair += 1
            out.append("    }")
            out.append("  }")
        out.append("}")
        # single-variable, field-free patterns also get a value function of the
        # gathered value itself (pre-resolved fold lanes, see device._row_layout)
        self.valx_ok = k == 1 and self.nf == 0 and not self.has_checks
        if self.valx_ok:
            gx = Gen()
            vx = self._values(gx, {"field": {}, "var": [Sym("x0")]})
            out.append(f"__device__ __forceinline__ double exa_valx_{pid}(const double x0) {{")
            out.extend(gx.lines)
            out.append(f"  return {R(vx[-1])};")
            out.append("}")
            # ... and its Jacobian / weighted Hessian entry (row buckets write the
            # augment's J/H slots from the row thread), same replay as above
            gx = Gen()
            vx = self._values(gx, {"field": {}, "var": [Sym("x0")]})
            gx.deriv = self.relax
            adjx = self._adjoints(gx, vx)
            gradx = self._slot_sums(gx, adjx)
            tx = self._tangents(gx, vx, 0)
            colx = self._slot_sums(gx, self._adjoint_tangents(gx, vx, adjx, tx))
            # x-independent J/H (pg, -p, ...: +-1 and w * 0): row buckets store
            # them before gathering the variable
            self.termx_const = not isinstance(gradx[0], Sym) and not isinstance(colx[0], Sym)
            # Hessian entry is the structural zero w * 0 (pg, -p, ...)
            self.termx_hzero = not isinstance(colx[0], Sym) and float(
                colx[0].value if isinstance(colx[0], Arr) else colx[0]) == 0.0
            out.append(f"__device__ __forceinline__ void exa_termx_{pid}(const double x0, const double wgt, double& jv, double& hv) {{")
            out.extend(gx.lines)
            out.append(f"  jv = {R(gradx[0])};")
            out.append("  hv = 0.0;" if (self.relax and _zero_const(colx[0])) else f"  hv = wgt * {R(colx[0])};")
            out.append("}")
        # records per thread: light patterns amortise per-thread overheads and
        # overlap several records' loads; heavy ones keep one record per thread
        n_ops = len(g.lines)
        heavy = bool(g.sincos) or any(ins[0] in ("exp", "log", "pow") for ins in self.instr) or k > 2
        self.rpt = int(os.environ.get("EXA_RPT_LIGHT", "1")) if (not heavy and n_ops <= 40) else 1
        self.heavy = heavy
        self.uses_sincos = bool(g.sincos)
        return "\n".join(out)

    def group_source(self, gid: int, members: list) -> str:
        """Group of terms of this one pattern (see :func:`group_source`)."""
        return group_source(gid, [(self, mem) for mem in members], relax=self.relax)

    def tape_norm(self):
        return list(self.tape.instr)


def _jst_flush(members, tail_sync: bool) -> str:
    """Coalesced stores of staged direct-Jacobian entries.  The warp's lanes
    hold consecutive records r0 .. r0 + nact - 1; in the block's last,
    partial warp the lanes past its last record have returned, so the mask
    comes from the record count (not __activemask(): every lane of it must
    reach the barrier, converged or not) and the store loops stride by the
    live lanes.  ``tail_sync``: the stage is reused after the flush."""
    T0 = members[0][3]
    fl = [f"  if ((MODE & EXA_M_JAC) && A.Jc) {{ const int lane_ = threadIdx.x & 31, r0_ = r - lane_; "
          f"const int nact_ = min(32, {T0}.nrec - r0_); "
          f"const unsigned act_ = nact_ >= 32 ? 0xffffffffu : ((1u << nact_) - 1u); __syncwarp(act_);"]
    for (_m, k_, jc0_, _T, off_) in members:
        fl.append(f" {{ double* __restrict__ jd_ = A.Jc + {jc0_}LL + {k_}LL * r0_; "
                  f"for (int i_ = lane_; i_ < {k_} * nact_; i_ += nact_) __stcs(jd_ + i_, EXA_JST[{off_} + i_]); }}")
    fl.append(" __syncwarp(act_); }" if tail_sync else " }")
    return "".join(fl)


def group_source(gid: int, entries: list, augs: list = (), relax: bool | None = None) -> str:
    """One thread evaluates record r of several terms (a *term group*).

    ``entries[m] = (PatternCode, {"cols": [group column id per index column],
    "blocks": [group block id per slot]})``; members may have different
    patterns (OPF: the two flow blocks of a branch side plus the thermal and
    angle-difference terms of the same branches).  Index columns with the same
    content are loaded once, variables with the same (block, column) are
    gathered once, and every identical sub-expression -- e.g. sin/cos(va_f -
    va_t) -- is computed once (the generator's CSE), while each member's
    outputs keep the reference's per-term operation order.

    ``augs[k] = (PatternCode, record offset, member, slot[, row source])``: in the set kernel
    the group also writes the J/H slots of augment ``U<k>``'s records
    ``off + r`` (single-variable, field-free pattern gathering the same
    variable as the member's slot), weighted by the multiplier of the row the
    augment record adds into."""
    relax = _DERIV_ZERO_ELISION if relax is None else bool(relax)
    M = len(entries)
    g = Gen()
    pre, post = [], []
    u_src: dict = {}
    for m, (pc, mem) in enumerate(entries):
        pc.instr = pc.tape_norm()
        for c, u in enumerate(mem["cols"]):
            u_src.setdefault(u, (m, c))
    for u, (m, c) in sorted(u_src.items()):
        pre.append(f"  const int i{u} = {_index_load(f'T{m}', c, 'r')};")
    fsyms = []
    for m, (pc, mem) in enumerate(entries):
        d = {}
        for fi, fname in enumerate(pc.tape.field_names):
            pre.append(f"  const double f{m}_{fi} = {_field_load(f'T{m}', fi, 'r')};")
            d[fname] = Sym(f"f{m}_{fi}")
        fsyms.append(d)
    xkey: dict = {}
    vsyms, cnames = [], []
    for m, (pc, mem) in enumerate(entries):
        vs, cn = [], []
        for s_, (_, ic) in enumerate(pc.slot_struct):
            key = (mem["blocks"][s_], mem["cols"][ic])
            if key not in xkey:
                n = len(xkey)
                xkey[key] = n
                post.append(f"  const int cg{n} = T{m}.voff[{s_}] + i{mem['cols'][ic]};")
                post.append(f"  const double xg{n} = __ldg(A.x + cg{n});")
            vs.append(Sym(f"xg{xkey[key]}"))
            cn.append(f"cg{xkey[key]}")
        vsyms.append(vs)
        cnames.append(cn)
    for m, (pc, mem) in enumerate(entries):
        if pc.k:
            ld = "EXA_LDP" if _WGT_CS else "__ldg"  # a member's own rows: each multiplier read once
            post.append(f"  const double wgt{m} = !(MODE & EXA_M_HESS) ? 0.0 : (T{m}.kind == EXA_OBJ) ? A.w"
                        f" : {ld}(A.y + (T{m}.rows ? __ldg(T{m}.rows + r) : T{m}.row_offset + r));")
    R = Gen.r
    # Stores are emitted as soon as their value is final (cons after the
    # value pass, J after the adjoint sweep, each Hessian column after its
    # seed's sweep) so that the LSU drains while the next sweep computes.
    # Stores whose value does not depend on x (constant J entries, structural
    # Hessian zeros w * 0) go right after the weight loads: their DRAM write
    # traffic then overlaps the gather phase instead of queueing behind it.
    early: list = []

    def const(v) -> bool:
        return not isinstance(v, Sym)

    # staged direct-Jacobian members still to flush: (m, k, jc0, T, stage offset)
    jst_members, jst_off, jst_size = [], 0, 0
    for m, (pc, mem) in enumerate(entries):
        k = pc.k
        T = f"T{m}"
        g.lines.append(f"  rank = rank{m};")
        g.deriv = False
        v = pc._values(g, {"field": fsyms[m], "var": vsyms[m]})
        root = v[-1]
        g.lines.append(f"  if ((MODE & EXA_M_CONS) && {T}.cons_direct) Cout[{T}.row_offset + r] = 0.0 + {R(root)};")
        g.lines.append(f"  if ((MODE & EXA_M_OBJV) && {T}.kind == EXA_OBJ) A.V[{T}.scr0 + r] = {R(root)};")
        if not k:
            continue
        g.deriv = relax
        adj = pc._adjoints(g, v)
        grads = pc._slot_sums(g, adj)
        # compressed-set module, direct member: the record's Jacobian row holds
        # exactly its k slots, in column order -> slot s is entry jc0 + k r +
        # rank (how many of the record's other columns are smaller), value
        # 0.0 + v (np.bincount's single-slot fold); without a compressed
        # Jacobian (A.Jc null) the raw slot as usual.  jst: the warp's 32
        # consecutive records own k * 32 consecutive entries -- staged in
        # shared memory (EXA_JST) and stored coalesced after the last slot.
        jc0 = mem.get("jc0")
        jst = mem.get("jst") if jc0 is not None else None  # "member" / "group" flush, or None
        if jst == "member":  # the member's own stage, flushed after its last slot
            jst_off = 0
        if jst:
            jst_members.append((m, k, int(jc0), T, jst_off))
        for s_ in range(k):
            # ("member" stages share one buffer: after the previous member's flush)
            dst = early if (const(grads[s_]) and jst != "member") else g.lines
            if jc0 is not None:
                rank = " + ".join(f"({cnames[m][t_]} < {cnames[m][s_]})" for t_ in range(k) if t_ != s_) or "0"
                tgt = (f"EXA_JST[{jst_off} + (threadIdx.x & 31) * {k} + ({rank})] =" if jst
                       else f"__stcs(A.Jc + ({int(jc0)}LL + {k}LL * r + ({rank})),")
                close = ";" if jst else ");"
                dst.append(f"  if (MODE & EXA_M_JAC) {{ if (A.Jc) {tgt} 0.0 + {R(grads[s_])}{close} "
                           f"else Jout[{T}.jac0 + {s_}LL * {T}.nrec + r] = {R(grads[s_])}; }}")
                continue
            dst.append(f"  if ((MODE & EXA_M_JAC) && {T}.kind != EXA_OBJ) Jout[{T}.jac0 + {s_}LL * {T}.nrec + r] = {R(grads[s_])};")
            dst.append(f"  if ((MODE & EXA_M_GRAD) && {T}.kind == EXA_OBJ) A.G[{T}.scr0 + {s_}LL * {T}.nrec + r] = {R(grads[s_])};")
        if jst:
            jst_off += 32 * k
            jst_size = max(jst_size, jst_off)
        if jst == "member":
            g.lines.append(_jst_flush(jst_members[-1:], tail_sync=True))
            jst_members.clear()
        hcls = mem.get("hcls", {})  # compressed-set module: pair -> (class, position, class size)
        for seed in range(k):
            t = pc._tangents(g, v, seed)
            col = pc._slot_sums(g, pc._adjoint_tangents(g, v, adj, t))
            j = seed
            for i in range(j, k):
                expr = R(col[i])
                dup = i != j and pc.slot_struct[i][0] == pc.slot_struct[j][0]
                if dup:
                    expr = f"({cnames[m][i]} == {cnames[m][j]} ? {expr} * 2.0 : {expr})"
                pair = i * (i + 1) // 2 + j
                if relax and _zero_const(col[i]):  # structural zero: +0.0, no weight
                    # (compressed-set module with a compressed Hessian: the
                    # segmented sum skips known +0.0 slots, nothing to write;
                    # an entry holding only this group's zeros is written here)
                    guard = "(MODE & EXA_M_HESS) && !A.Hc" if mem.get("cmp") else "MODE & EXA_M_HESS"
                    early.append(f"  if ({guard}) Hout[{T}.hess0 + {pair}LL * {T}.nrec + r] = 0.0;")
                    if pair in hcls and hcls[pair][1] == hcls[pair][2] - 1:
                        c = hcls[pair][0]
                        early.append(f"  if ((MODE & EXA_M_HESS) && hq{c} >= 0) __stcs(A.Hc + hq{c}, 0.0);")
                    continue
                if pair in hcls:
                    # group-local compressed entry: its slots are this thread's
                    # (one per member, members in raw-slot order): fold them in
                    # np.bincount's order and store the entry; records where the
                    # entry has other slots (hq < 0) write the raw slot instead
                    c, q, size, _zero = hcls[pair]
                    acc = "0.0 + hv_" if q == 0 else f"ha{c} + hv_"
                    g.lines.append(f"  if (MODE & EXA_M_HESS) {{ const double hv_ = wgt{m} * {expr}; ha{c} = {acc}; "
                                   f"if (hq{c} < 0) Hout[{T}.hess0 + {pair}LL * {T}.nrec + r] = hv_; }}")
                    if q == size - 1:
                        g.lines.append(f"  if ((MODE & EXA_M_HESS) && hq{c} >= 0) __stcs(A.Hc + hq{c}, ha{c});")
                    continue
                dst = early if (const(col[i]) and not dup) else g.lines
                dst.append(f"  if (MODE & EXA_M_HESS) Hout[{T}.hess0 + {pair}LL * {T}.nrec + r] = wgt{m} * {expr};")
    if jst_members:  # "group": one flush of every member's entries after the group's work
        g.lines.append(_jst_flush(jst_members, tail_sync=False))
    # attached augments: their J slots in the jac/set kernels, H in hess/set
    aug_late = []
    for k, aug in enumerate(augs):
        apc, off, m, s_ = aug[:4]
        rowsrc = aug[4] if len(aug) > 4 else None
        xs = vsyms[m][s_].name
        if relax and getattr(apc, "termx_hzero", False):
            # structural-zero Hessian entry: written as +0.0 (the reference's
            # w * 0.0 carries the multiplier's sign; IEEE-equal, see the zero-sign
            # relaxation) -- saves a two-load chain per record
            post.append(f"  const double wa{k} = 0.0;")
        elif rowsrc is not None:  # row = constant + a group index column: one load
            post.append(f"  const double wa{k} = !(MODE & EXA_M_HESS) ? 0.0 : __ldg(A.y + ({rowsrc[1]}LL + i{rowsrc[0]}));")
        else:
            post.append(f"  const double wa{k} = !(MODE & EXA_M_HESS) ? 0.0 : __ldg(A.y + __ldg(U{k}.rows + {off} + r));")
        dst = early if getattr(apc, "termx_const", False) else aug_late
        dst.append(f"  if (MODE & (EXA_M_JAC | EXA_M_HESS)) {{ double jv, hv; exa_termx_{apc.pid}({xs}, wa{k}, jv, hv); "
                   f"if (MODE & EXA_M_JAC) Jout[U{k}.jac0 + {off}LL + r] = jv; "
                   f"if (MODE & EXA_M_HESS) Hout[U{k}.hess0 + {off}LL + r] = hv; }}")
    g.lines.extend(aug_late)
    args = ", ".join([f"const ExaTerm& T{m}" for m in range(M)] + [f"const ExaTerm& U{k}" for k in range(len(augs))])
    ranks = ", ".join(f"int rank{m}" for m in range(M))
    out = [f"template <int MODE, int LDH = 1>\n__device__ __forceinline__ void exa_grp_{gid}({args}, int r, const ExaArgs& A, {ranks}) {{",
           "  double* __restrict__ Cout = A.c;", "  double* __restrict__ Jout = A.J;",
           "  double* __restrict__ Hout = A.H;", "  int rank = rank0;"]
    out.extend(pre)
    if jst_size:  # this warp's stage of direct Jacobian entries (32 records x k slots per member)
        out.append(f"  __shared__ double exa_jst_[EXA_JST_WARPS * {jst_size}];")
        out.append(f"  double* const EXA_JST = exa_jst_ + (threadIdx.x >> 5) * {jst_size};")
    # compressed-set module: positions of the group-local compressed H entries
    # (plan data, loaded before the grid dependency) and their running folds
    for c, off in sorted({c: off for _, mem in entries for (c, _q, _s, off) in mem.get("hcls_pos", [])}.items()):
        out.append(f"  const int hq{c} = A.hpos ? __ldg(A.hpos + {int(off)}LL + r) : -1;  // -1: raw slots")
        out.append(f"  double ha{c} = 0.0;")
    out.append(f"  EXA_TP(0, i{min(u_src)});" if u_src else "  EXA_TP(0, 0.0);")
    out.append("  EXA_GRID_WAIT();")
    out.extend(post)
    out.extend(early)
    if xkey:
        out.append("  EXA_TP(1, " + " + ".join(f"xg{n}" for n in range(len(xkey))) + ");")
    out.append("  EXA_GRID_RELEASE_MID(1);")
    # phase stamp 2 after the first sin/cos
    lines = list(g.lines)
    for i, ln in enumerate(lines):
        m_ = re.search(r"exa_sincos\(.*?&(\w+), &(\w+)\)", ln)
        if m_:
            lines.insert(i + 1, f"  EXA_TP(2, {m_.group(1)} + {m_.group(2)});")
            lines.insert(i + 2, "  EXA_GRID_RELEASE_MID(2);")
            break

    out.extend(lines)
    out.append("}")
    return "\n".join(out)
