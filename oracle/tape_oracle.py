"""CPU oracle for the callback set -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product package never imports it.

This is a numpy restatement of the reference's per-term tape passes
(``/root/reference/pkg/src/simdnlp/autodiff.py``):

* :meth:`Passes.values`            follows ``TermTape.values``          (127-168)
* :meth:`Passes.adjoints`          follows ``TermTape.adjoints``        (173-218)
* :meth:`Passes.slot_sums`         follows ``TermTape.slot_sums``       (220-226)
* :meth:`Passes.tangents`          follows ``TermTape.tangents``        (231-297)
* :meth:`Passes.adjoint_tangents`  follows ``TermTape.adjoint_tangents`` (302-382)
* ``_acc`` / ``_accd``             follow ``autodiff.py:385-396``
* ``eval_*``                       follow ``autodiff.py:536-652``
* ``compress``                     follows ``compress_coordinates``      (677-689)

Structural zeros are Python floats equal to 0.0 (``_is_zero``,
``autodiff.py:69-70``); everything data-dependent is an ndarray.  The oracle
operates on the host plan built by :mod:`paper_2510_12897_b200.plan` (whose
COO layout is pinned separately against the reference's goldens), so its
only job is the arithmetic.  It is pinned against golden vectors produced by
the reference itself (``tests/golden/``, ``tools/make_goldens.py``).
"""

from __future__ import annotations

import numpy as np


class OracleDomainError(ArithmeticError):
    def __init__(self, op, record, kind="?", block_index=-1):
        super().__init__(op, record)
        self.op, self.record, self.kind, self.block_index = op, record, kind, block_index


def _structural_zero(v) -> bool:
    return isinstance(v, float) and v == 0.0


def _first(mask) -> int:
    m = np.asarray(mask)
    return -1 if m.ndim == 0 else int(np.flatnonzero(m)[0])


def _need_positive(a, op):
    bad = ~(np.asarray(a) > 0.0)
    if np.any(bad):
        raise OracleDomainError(op, _first(bad))


def _need_nonzero(a, op):
    bad = np.asarray(a) == 0.0
    if np.any(bad):
        raise OracleDomainError(op, _first(bad))


def _acc(store, at, val):
    store[at] = val if store[at] is None else store[at] + val


def _accd(store, at, d_parent, partial, a_parent, partial_dot):
    contrib = 0.0 if _structural_zero(d_parent) else d_parent * partial
    if not _structural_zero(partial_dot):
        contrib = contrib + a_parent * partial_dot
    store[at] = contrib if store[at] is None else store[at] + contrib


class Passes:
    """The four passes over one tape (list of instruction tuples).

    ``trig`` selects the array sin/cos: ``None`` = numpy (glibc, i.e. the
    reference), or a ``(sin, cos)`` pair -- the tests pass the correctly
    rounded pair from :mod:`oracle.crtrig` to show that the only source of
    CUDA-vs-reference differences is glibc's (rare) misrounding.  Scalars
    always use numpy, as the generator folds them with numpy too.
    """

    def __init__(self, instr, k, trig=None):
        self.instr = instr
        self.k = k
        self.root = len(instr) - 1
        self.trig = trig

    def _sin(self, a):
        if self.trig is None or np.ndim(a) == 0:
            return np.sin(a)
        return self.trig[0](a)

    def _cos(self, a):
        if self.trig is None or np.ndim(a) == 0:
            return np.cos(a)
        return self.trig[1](a)

    # ---------------------------------------------------------------- values
    def values(self, x, reals, cols):
        v = [None] * len(self.instr)
        for p, ins in enumerate(self.instr):
            op = ins[0]
            if op == "const":
                v[p] = ins[1]
            elif op == "field":
                v[p] = reals[ins[1]]
            elif op == "var":
                v[p] = x[cols[ins[1]]]
            elif op == "neg":
                v[p] = -v[ins[1]]
            elif op == "sin":
                v[p] = self._sin(v[ins[1]])
            elif op == "cos":
                v[p] = self._cos(v[ins[1]])
            elif op == "exp":
                v[p] = np.exp(v[ins[1]])
            elif op in ("log", "sqrt"):
                _need_positive(v[ins[1]], op)
                v[p] = getattr(np, op)(v[ins[1]])
            elif op == "add":
                v[p] = v[ins[1]] + v[ins[2]]
            elif op == "sub":
                v[p] = v[ins[1]] - v[ins[2]]
            elif op == "mul":
                v[p] = v[ins[1]] * v[ins[2]]
            elif op == "div":
                _need_nonzero(v[ins[2]], "div")
                v[p] = v[ins[1]] / v[ins[2]]
            elif op == "ipow":
                base, n = v[ins[1]], ins[2]
                if n < 0:
                    _need_nonzero(base, "pow")
                v[p] = base * base if n == 2 else np.power(base, n)
            elif op == "pow":
                _need_positive(v[ins[1]], "pow")
                v[p] = np.power(v[ins[1]], v[ins[2]])
            else:
                raise ValueError(op)
        return v

    # ---------------------------------------------------------------- reverse
    def adjoints(self, v, nrec):
        adj = [None] * len(self.instr)
        adj[self.root] = np.ones(nrec)
        for p in range(self.root, -1, -1):
            g = adj[p]
            ins = self.instr[p]
            op = ins[0]
            if g is None or op in ("const", "field", "var"):
                continue
            a = ins[1]
            if op == "neg":
                _acc(adj, a, -g)
            elif op == "sin":
                _acc(adj, a, g * self._cos(v[a]))
            elif op == "cos":
                _acc(adj, a, -g * self._sin(v[a]))
            elif op == "exp":
                _acc(adj, a, g * v[p])
            elif op == "log":
                _acc(adj, a, g / v[a])
            elif op == "sqrt":
                _acc(adj, a, g / (2.0 * v[p]))
            elif op == "add":
                _acc(adj, a, g)
                _acc(adj, ins[2], g)
            elif op == "sub":
                _acc(adj, a, g)
                _acc(adj, ins[2], -g)
            elif op == "mul":
                _acc(adj, a, g * v[ins[2]])
                _acc(adj, ins[2], g * v[a])
            elif op == "div":
                b = ins[2]
                _acc(adj, a, g / v[b])
                _acc(adj, b, -g * v[p] / v[b])
            elif op == "ipow":
                n = ins[2]
                if n != 0:
                    if n - 1 < 0:
                        _need_nonzero(v[a], "pow")
                    _acc(adj, a, g * n * np.power(v[a], n - 1))
            else:  # pow
                b = ins[2]
                _acc(adj, a, g * v[b] * v[p] / v[a])
                _acc(adj, b, g * v[p] * np.log(v[a]))
        return adj

    def slot_sums(self, per_node, nrec):
        out = [np.zeros(nrec) for _ in range(self.k)]
        for p, ins in enumerate(self.instr):
            if ins[0] == "var" and per_node[p] is not None:
                out[ins[1]] = out[ins[1]] + per_node[p]
        return out

    # ------------------------------------------------------ forward tangents
    def tangents(self, v, seed):
        Z = _structural_zero
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
                t[p] = 0.0 if Z(ta) else -ta
            elif op == "sin":
                t[p] = 0.0 if Z(ta) else self._cos(v[ins[1]]) * ta
            elif op == "cos":
                t[p] = 0.0 if Z(ta) else -self._sin(v[ins[1]]) * ta
            elif op == "exp":
                t[p] = 0.0 if Z(ta) else v[p] * ta
            elif op == "log":
                t[p] = 0.0 if Z(ta) else ta / v[ins[1]]
            elif op == "sqrt":
                t[p] = 0.0 if Z(ta) else ta / (2.0 * v[p])
            elif op == "add":
                tb = t[ins[2]]
                t[p] = tb if Z(ta) else (ta if Z(tb) else ta + tb)
            elif op == "sub":
                tb = t[ins[2]]
                t[p] = ta if Z(tb) else (-tb if Z(ta) else ta - tb)
            elif op == "mul":
                tb = t[ins[2]]
                lhs = 0.0 if Z(ta) else ta * v[ins[2]]
                rhs = 0.0 if Z(tb) else v[ins[1]] * tb
                t[p] = 0.0 if (Z(lhs) and Z(rhs)) else lhs + rhs
            elif op == "div":
                tb = t[ins[2]]
                if Z(ta) and Z(tb):
                    t[p] = 0.0
                else:
                    lhs = 0.0 if Z(ta) else ta / v[ins[2]]
                    rhs = 0.0 if Z(tb) else v[p] * tb / v[ins[2]]
                    t[p] = lhs - rhs
            elif op == "ipow":
                n = ins[2]
                t[p] = 0.0 if (Z(ta) or n == 0) else n * np.power(v[ins[1]], n - 1) * ta
            else:  # pow
                tb = t[ins[2]]
                if Z(ta) and Z(tb):
                    t[p] = 0.0
                else:
                    base, ex = v[ins[1]], v[ins[2]]
                    d = 0.0 if Z(ta) else ex * ta / base
                    if not Z(tb):
                        d = d + np.log(base) * tb
                    t[p] = v[p] * d
        return t

    # ------------------------------------------- second-order reverse sweep
    def adjoint_tangents(self, v, adj, t):
        Z = _structural_zero
        dot = [None] * len(self.instr)
        dot[self.root] = 0.0
        for p in range(self.root, -1, -1):
            g, dg = adj[p], dot[p]
            ins = self.instr[p]
            op = ins[0]
            if g is None or op in ("const", "field", "var"):
                continue
            a = ins[1]
            if op == "neg":
                _accd(dot, a, dg, -1.0, g, 0.0)
            elif op == "sin":
                ta = t[a]
                pd = 0.0 if Z(ta) else -self._sin(v[a]) * ta
                _accd(dot, a, dg, self._cos(v[a]), g, pd)
            elif op == "cos":
                ta = t[a]
                pd = 0.0 if Z(ta) else -self._cos(v[a]) * ta
                _accd(dot, a, dg, -self._sin(v[a]), g, pd)
            elif op == "exp":
                _accd(dot, a, dg, v[p], g, t[p])
            elif op == "log":
                ta = t[a]
                pd = 0.0 if Z(ta) else -ta / (v[a] * v[a])
                _accd(dot, a, dg, 1.0 / v[a], g, pd)
            elif op == "sqrt":
                pd = 0.0 if Z(t[p]) else -t[p] / (2.0 * v[p] * v[p])
                _accd(dot, a, dg, 1.0 / (2.0 * v[p]), g, pd)
            elif op in ("add", "sub"):
                _accd(dot, a, dg, 1.0, g, 0.0)
                _accd(dot, ins[2], dg, 1.0 if op == "add" else -1.0, g, 0.0)
            elif op == "mul":
                b = ins[2]
                _accd(dot, a, dg, v[b], g, t[b])
                _accd(dot, b, dg, v[a], g, t[a])
            elif op == "div":
                b = ins[2]
                den = v[b]
                ta, tb = t[a], t[b]
                pda = 0.0 if Z(tb) else -tb / (den * den)
                if Z(ta) and Z(tb):
                    pdb = 0.0
                else:
                    pdb = -(0.0 if Z(ta) else ta / (den * den))
                    if not Z(tb):
                        pdb = pdb + 2.0 * v[p] * tb / (den * den)
                _accd(dot, a, dg, 1.0 / den, g, pda)
                _accd(dot, b, dg, -v[p] / den, g, pdb)
            elif op == "ipow":
                n = ins[2]
                if n == 0:
                    continue
                base, ta = v[a], t[a]
                part = n * np.power(base, n - 1)
                pd = 0.0 if (n <= 1 or Z(ta)) else n * (n - 1) * np.power(base, n - 2) * ta
                _accd(dot, a, dg, part, g, pd)
            else:  # pow
                b = ins[2]
                base, ex = v[a], v[b]
                ta, tb, tp = t[a], t[b], t[p]
                pa = ex * v[p] / base
                pb = v[p] * np.log(base)
                pda = 0.0 if Z(tb) else tb * v[p] / base
                if not Z(tp):
                    pda = pda + ex * tp / base
                if not Z(ta):
                    pda = pda - ex * v[p] * ta / (base * base)
                pdb = 0.0 if Z(tp) else tp * np.log(base)
                if not Z(ta):
                    pdb = pdb + v[p] * ta / base
                _accd(dot, a, dg, pa, g, pda)
                _accd(dot, b, dg, pb, g, pdb)
        return dot


# ---------------------------------------------------------------------------
# callbacks over a host plan (paper_2510_12897_b200.plan.ModelPlan)
# ---------------------------------------------------------------------------

_TRIG = [None]


def use_trig(trig):
    """Set the array sin/cos used by subsequent oracle calls (None = numpy)."""
    _TRIG[0] = trig


def _passes(tp):
    return Passes(tp.tape.instr, tp.tape.k, _TRIG[0])


def _values(tp, x):
    try:
        return _passes(tp).values(x, tp.reals, tp.cols)
    except OracleDomainError as e:
        raise OracleDomainError(e.op, e.record, tp.kind, tp.block_index) from None


def eval_objective(plan, x) -> float:
    x = np.asarray(x, dtype=np.float64)
    total = 0.0
    for tp in plan.obj_terms:
        root = _values(tp, x)[tp.tape.root]
        total += float(root) * tp.nrec if np.ndim(root) == 0 else float(np.sum(root))
    return total


def eval_gradient(plan, x, out):
    x = np.asarray(x, dtype=np.float64)
    out[:] = 0.0
    for tp in plan.obj_terms:
        P = _passes(tp)
        v = _values(tp, x)
        for s, gs in enumerate(P.slot_sums(P.adjoints(v, tp.nrec), tp.nrec)):
            out += np.bincount(tp.cols[s], weights=gs, minlength=plan.nvar)


def eval_constraints(plan, x, out):
    x = np.asarray(x, dtype=np.float64)
    if plan.ncon == 0:
        return
    out[:] = 0.0
    for tp in plan.con_terms:
        root = _values(tp, x)[tp.tape.root]
        if np.ndim(root) == 0:
            root = np.full(tp.nrec, float(root))
        if tp.row_offset is not None:
            out[tp.row_offset : tp.row_offset + tp.nrec] += root
        else:
            np.add.at(out, tp.rows, root)


def eval_jacobian(plan, x, out):
    x = np.asarray(x, dtype=np.float64)
    for tp in plan.con_terms:
        P = _passes(tp)
        v = _values(tp, x)
        for s, gs in enumerate(P.slot_sums(P.adjoints(v, tp.nrec), tp.nrec)):
            lo, hi = tp.jac_slices[s]
            out[lo:hi] = gs


def eval_hessian(plan, x, mult, obj_weight, out):
    x = np.asarray(x, dtype=np.float64)
    mult = np.asarray(mult, dtype=np.float64)
    for tp in plan.obj_terms + plan.con_terms:
        k = tp.tape.k
        if k == 0:
            continue
        w = float(obj_weight) if tp.kind == "objective" else mult[tp.rows]
        P = _passes(tp)
        v = _values(tp, x)
        adj = P.adjoints(v, tp.nrec)
        by_seed = [P.slot_sums(P.adjoint_tangents(v, adj, P.tangents(v, s)), tp.nrec) for s in range(k)]
        for pair in tp.hess_pairs:
            val = by_seed[pair.j][pair.i]
            if pair.dup is not None:
                val = val * (1.0 + pair.dup)
            out[pair.start : pair.start + tp.nrec] = w * val


def compress(rows, cols):
    """(urows, ucols, slot_map) like ``compress_coordinates`` (677-689)."""
    if rows.size == 0:
        e = np.zeros(0, dtype=np.int64)
        return e, e.copy(), e.copy()
    u, inv = np.unique(np.stack([rows, cols], axis=1), axis=0, return_inverse=True)
    return u[:, 0].astype(np.int64), u[:, 1].astype(np.int64), inv.astype(np.int64).ravel()


def sum_values(slot_map, nnz, raw):
    return np.bincount(slot_map, weights=raw, minlength=nnz)


def eval_set(plan, x, y, w):
    """One callback set: (c, J, H) as fresh arrays."""
    c = np.empty(plan.ncon)
    J = np.empty(plan.n_jac_slots)
    H = np.empty(plan.n_hess_slots)
    eval_constraints(plan, x, c)
    eval_jacobian(plan, x, J)
    eval_hessian(plan, x, y, w, H)
    return c, J, H
