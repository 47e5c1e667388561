"""Host-side sparsity detection, run once per model.

Reproduces the reference's ``build_plan`` COO layout bit-exactly
(``autodiff.py:444-508``):

* B1  objective terms first in the Hessian, then ``con_terms`` in
  registration order (blocks and augments interleaved);
* B3  Jacobian: per constraint-side term, per slot, ``nrec`` consecutive
  entries ``(rows[r], cols[s][r])``;
* B4  Hessian: per term, ``for i < k: for j <= i``, ``nrec`` consecutive
  entries ``(max(ci, cj), min(ci, cj))``;
* B5  records where two distinct slots hit the same variable are doubled;
* B9  k = 0 terms emit nothing.

Everything here is x-independent integer work on the host; the device only
ever sees the per-term *starts* of these layouts (:mod:`.device`).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .tape import TermTape


@dataclass(eq=False)
class HessPair:
    i: int
    j: int
    start: int
    dup: np.ndarray | None  # records where slots i and j hit the same variable


@dataclass(eq=False)
class TermPlan:
    tape: TermTape
    reals: dict
    cols: list  # per slot: global variable ids, int64[nrec]
    nrec: int
    kind: str  # "objective" | "constraint" | "augment"
    block_index: int
    table: object = None
    slot_blocks: list = field(default_factory=list)
    rows: np.ndarray | None = None
    row_offset: int | None = None
    target_index: int | None = None  # augments: index of the target block in core.constraints
    jac_slices: list | None = None
    hess_pairs: list | None = None
    hess_start: int = 0


@dataclass(eq=False)
class ModelPlan:
    obj_terms: list
    con_terms: list
    jac_rows: np.ndarray
    jac_cols: np.ndarray
    hess_rows: np.ndarray
    hess_cols: np.ndarray
    nvar: int = 0
    ncon: int = 0

    @property
    def n_jac_slots(self) -> int:
        return int(self.jac_rows.shape[0])

    @property
    def n_hess_slots(self) -> int:
        return int(self.hess_rows.shape[0])


def _term(kernel, table, kind: str, index: int) -> TermPlan:
    tape = TermTape(kernel)
    cols = [blk.offset + table.indices[ix] for blk, ix in tape.slots]
    return TermPlan(
        tape=tape,
        reals=dict(table.reals),
        cols=cols,
        nrec=table.nrec,
        kind=kind,
        block_index=index,
        table=table,
        slot_blocks=[blk for blk, _ in tape.slots],
    )


def build_plan(core) -> ModelPlan:
    from .core import ConstraintBlock

    obj_terms = [_term(b.kernel, b.table, "objective", i) for i, b in enumerate(core.objectives)]
    con_index = {id(c): i for i, c in enumerate(core.constraints)}
    aug_index = {id(a): i for i, a in enumerate(core.augments)}
    con_terms = []
    for term in core.con_terms:
        if isinstance(term, ConstraintBlock):
            tp = _term(term.kernel, term.table, "constraint", con_index[id(term)])
            tp.row_offset = term.row_offset
            tp.rows = term.rows()
        else:
            tp = _term(term.kernel, term.table, "augment", aug_index[id(term)])
            tp.rows = term.table.indices["row"].copy()
            tp.target_index = con_index[id(term.target)]
        con_terms.append(tp)

    jr, jc = [], []
    at = 0
    for tp in con_terms:
        tp.jac_slices = []
        for c in tp.cols:
            jr.append(tp.rows)
            jc.append(c)
            tp.jac_slices.append((at, at + tp.nrec))
            at += tp.nrec

    hr, hc = [], []
    at = 0
    for tp in obj_terms + con_terms:
        tp.hess_pairs = []
        tp.hess_start = at
        for i in range(tp.tape.k):
            ci = tp.cols[i]
            for j in range(i + 1):
                cj = tp.cols[j]
                hr.append(np.maximum(ci, cj))
                hc.append(np.minimum(ci, cj))
                dup = None
                if i != j:
                    same = ci == cj
                    if same.any():
                        dup = same
                tp.hess_pairs.append(HessPair(i, j, at, dup))
                at += tp.nrec

    none = np.zeros(0, dtype=np.int64)
    return ModelPlan(
        obj_terms=obj_terms,
        con_terms=con_terms,
        jac_rows=np.concatenate(jr).astype(np.int64) if jr else none,
        jac_cols=np.concatenate(jc).astype(np.int64) if jc else none.copy(),
        hess_rows=np.concatenate(hr).astype(np.int64) if hr else none.copy(),
        hess_cols=np.concatenate(hc).astype(np.int64) if hc else none.copy(),
        nvar=core.nvar,
        ncon=core.ncon,
    )
