"""Lower a host plan onto one B200: device layout, segment tables, JIT module.

HBM layout (one plan, read-only after creation):

* ``f64`` blob -- every real field column of every term, SoA, each column
  256-byte aligned (reference ``DataTable.reals``, ``core.py:36-64``);
* ``i32`` blob -- index columns as int32 in-block positions, augment row
  columns, the per-row contribution lists of augment-target blocks;
* term table -- one :c:type:`ExaTerm` per term (blob offsets, per-slot block
  offsets, output starts in the raw J/H layouts);
* per-callback segment tables -- CTA -> (term, records) so that each
  callback is ONE launch of the model's generated kernel.

Outputs are caller buffers: raw Jacobian ``[term][slot][record]`` and raw
Hessian ``[term][pair][record]`` exactly as the reference lays them out
(``autodiff.py:471-498``), so every warp store is a coalesced 256-byte run.

:class:`HostLayout` is pure host work (no GPU) so that ``build()`` can
pre-compile the exact module a model will use; :class:`DevicePlan` uploads it.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import _lib
from .codegen import _DERIV_ZERO_ELISION, PatternCode
from .core import ModelError
from .jit import PDL, PERSIST, SM_COUNT, THREADS_ENV, THREADS_HEAVY, choose_threads, compile_module, module_source

ALIGN = 32  # elements: 256 B for fp64, 128 B for int32

KIND = {"objective": 0, "constraint": 1, "augment": 2}
OP_LEAF, OP_ADD, OP_CONST, OP_ZERO_PLUS, OP_TOTAL_ADD = range(5)
SEG_TERM, SEG_ROW, SEG_FOLD, SEG_GROUP, SEG_BUCKET = 0, 1, 2, 3, 4
# Row buckets (specialised modules): augment-target rows whose augments are
# all single-variable and field-free are evaluated one thread per row, rows
# grouped by contribution count so the count is a compile-time constant.
BUCKETS = os.environ.get("EXA_BUCKETS", "1") == "1"
BUCKET_SEL_BITS = 2                    # augment selector in the entry's top bits
BUCKET_GID_BITS = 29                   # global variable id bits
BUCKET_MAX_D = 31                      # at most this many augment contributions per row
BUCKET_WMAX = 8                        # wider rows: one warp per row (in-order shuffle fold)
BUCKET_MAX_N = 48                      # at most this many distinct counts per block

# Terms of one heavy pattern that share index columns (OPF: the 4 branch-flow
# blocks) are evaluated by one thread per record (see codegen.group_source).
# terms per group: "auto" = 4 for sets that fit one wave of 32-thread CTAs
# (OPF: all four flow blocks of a branch in one thread -- half the vm/va
# gathers; case13659 5.92 -> 5.65 us with the evict-first cache policy), 2 for
# many-wave sets (twice the threads hide more latency: MP96 39.4 vs 40.7 us)
GROUP_MAX_ENV = os.environ.get("EXA_GROUP_MAX", "auto")
ATTACH = os.environ.get("EXA_ATTACH", "1") == "1"  # light terms join heavy groups
# instance-window CTA order of many-wave batched sets (0 = natural order)
LOCALITY_W = int(os.environ.get("EXA_LOCALITY_W", "0"))
GROUP_RPT = int(os.environ.get("EXA_GROUP_RPT", "1"))  # records per thread of term groups (ILP)
ATTACH_AUGS = os.environ.get("EXA_ATTACH_AUGS", "1") == "1"  # groups write aligned augments' J/H
HALF_ROWS = os.environ.get("EXA_HALF_ROWS", "1") == "1"  # long bucket rows of <= 15 entries: half a warp each

# Models with at most this many terms get a *specialised* module (metadata
# compiled in as constants); larger ones (e.g. thousands of per-instance
# blocks) use the generic module with run-time term tables.
META_CONST_MAX_TERMS = 80
# periodic parameter columns of batched element-major models (plan.batch_period)
PERIODIC = os.environ.get("EXA_PERIODIC", "1") == "1"


def _periodic(tp, period):
    """Per-element parameter columns of a term of an element-major batched
    model (records of element e over instances / periods k), or None.

    The element of record r is ``r // period`` when every element has all
    ``period`` records (``kcol = -1``: MP models, r = e * T + t), else
    ``ix[kcol][r] // period - g0`` for an index column whose block position
    ``h(e) * period + k`` names the element (N-1 flows: the flow variable of
    a branch, whose instances skip the one with that branch out).  A field
    column constant per element is stored once per element (bit ``fi`` of
    fmask); an index column of the form ``g(e) * period + k`` (same instance
    k as the record) is stored as ``g(e) * period`` per element (bit ``c`` of
    imask).  Data-driven and exact: the stored tables reproduce every
    record's value.  Returns dict(per, fmask, imask, kcol, g0, fcols,
    icols) with the per-element tables, or None when nothing reduces."""
    n = tp.nrec
    if not period or period < 2 or n == 0:
        return None
    P = int(period)
    fields = [np.ascontiguousarray(tp.reals[nm], dtype=np.float64) for nm in tp.tape.field_names]
    idx = [np.asarray(tp.table.indices[nm], dtype=np.int64) for nm in tp.tape.index_names]

    def reduce_with(elem, first, kk, kcol):
        """first[g] = a record of element g (elem = element of each record)."""
        fmask = imask = 0
        fcols, icols = {}, {}
        for fi, col in enumerate(fields):
            bits = col.view(np.int64)
            tab = bits[first]
            if np.all(bits == tab[elem]):
                fmask |= 1 << fi
                fcols[fi] = tab.view(np.float64)
        for c, col in enumerate(idx):
            if c == kcol:
                continue
            base = col - kk
            tab = base[first]
            if np.all(base == tab[elem]) and np.all(tab % P == 0):
                imask |= 1 << c
                icols[c] = tab
        G = first.size  # per-element table length
        saved = (8 * bin(fmask).count("1") + 4 * bin(imask).count("1")) * (n - G)
        return saved, dict(per=P, fmask=fmask, imask=imask, kcol=kcol, fcols=fcols, icols=icols)

    best = None
    if n % P == 0:  # implicit element r // P
        r = np.arange(n, dtype=np.int64)
        cand = reduce_with(r // P, np.arange(0, n, P), r % P, -1)
        cand[1]["g0"] = 0
        if cand[0] > 0:
            best = cand
    for kc, key in enumerate(idx):  # element named by an index column
        q = key // P
        g0, g1 = int(q.min()), int(q.max())
        if g1 - g0 + 1 > n:  # tables no larger than the columns they replace
            continue
        elem = q - g0
        first = np.zeros(g1 - g0 + 1, dtype=np.int64)
        first[elem[::-1]] = np.arange(n - 1, -1, -1)  # first record of each element
        cand = reduce_with(elem, first, key % P, kc)
        cand[1]["g0"] = g0
        # a keyed load adds one dependent load: prefer the implicit form on ties
        if cand[0] > 4 * n and (best is None or cand[0] > best[0] + 4 * n):
            best = cand
    if best is None or not (best[1]["fmask"] or best[1]["imask"]):
        return None
    return best[1]


# Run heavy patterns in a separate concurrent kernel (measured slower on
# case13659: the fork/join costs more than the register specialisation wins).
SPLIT_HEAVY = os.environ.get("EXA_SPLIT", "0") == "1"


class _Blob:
    def __init__(self, dtype):
        self.dtype = dtype
        self.parts: list = []
        self.n = 0

    def add(self, arr) -> int:
        arr = np.ascontiguousarray(arr, dtype=self.dtype).ravel()
        pad = (-self.n) % ALIGN
        if pad:
            self.parts.append(np.zeros(pad, dtype=self.dtype))
            self.n += pad
        off = self.n
        self.parts.append(arr)
        self.n += arr.size
        return off

    def array(self):
        if not self.parts:
            return np.zeros(1, dtype=self.dtype)
        return np.concatenate(self.parts)


def _i32(a, what):
    a = np.asarray(a, dtype=np.int64)
    if a.size and (a.min() < -(2**31) or a.max() >= 2**31):
        raise ModelError(f"{what} exceeds the int32 device index range")
    return a.astype(np.int32)


def pairwise_program(nrec: int, scr0: int, leaves: list, prog: list) -> None:
    """Leaves and combine ops of numpy's pairwise sum over V[scr0:scr0+nrec]
    (numpy pairwise_sum: blocks <= 128, split at n/2 rounded down to 8)."""

    def rec(start, n):
        if n <= 128:
            prog.append((OP_LEAF, len(leaves), 0))
            leaves.append((start, n))
            return
        n2 = n // 2
        n2 -= n2 % 8
        rec(start, n2)
        rec(start + n2, n - n2)
        prog.append((OP_ADD, 0, 0))

    rec(scr0, nrec)


def _const_op(v: float):
    return (OP_CONST, int(np.float64(v).view(np.int64)), 0)


def collect_patterns(plan, relax: bool | None = None):
    """Distinct tape patterns of a plan (first-appearance order) and the
    pattern id of every term (objective terms first, then constraint-side);
    ``relax`` = zero-sign mode of the generated code (None = default)."""
    keys: dict = {}
    pcodes: list = []
    term_pid = []
    for tp in plan.obj_terms + plan.con_terms:
        tape = tp.tape
        if tape.k > _lib.MAXK or len(tape.field_names) > _lib.MAXF or len(tape.index_names) > _lib.MAXI:
            raise ModelError(
                f"kernel with k={tape.k}, {len(tape.field_names)} fields, "
                f"{len(tape.index_names)} index columns exceeds the device limits (16 each)")
        key = tape.pattern_key()
        pid = keys.get(key)
        if pid is None:
            pid = len(pcodes)
            keys[key] = pid
            pc = PatternCode(pid, tape, len(tape.field_names), len(tape.index_names), key[1], relax=relax)
            if pc.has_checks and len(tape.instr) > 4095:
                raise ModelError("domain-checked kernels are limited to 4095 instructions")
            pcodes.append(pc)
        term_pid.append(pid)
    return pcodes, term_pid


PRERESOLVE = 1 << 30  # fold slot flag: .y holds the global variable id, not a record


def _row_layout(base_tp, base_dev, augs, dev_index, valx=None):
    """Contributions per base row in reference order (base, then augments in
    registration order, records in order).  Returns ``(None, None, slots)`` for
    the warp-fold layout -- rows packed into 32-lane warps, slot =
    (term | position << 16, record), pad = (-1, 0) -- or ``(ptr, ent, None)``
    for the serial CSR layout when a row has more than 32 contributions."""
    n = base_tp.nrec
    lrows, terms_, recs = [], [], []
    for a in augs:
        lrows.append(np.asarray(a.rows, dtype=np.int64) - base_tp.row_offset)
        t_a = dev_index[id(a)]
        if valx is not None and t_a in valx:
            # single-variable, field-free augment (pg, -p, ...): pre-resolve the
            # gathered variable so the fold lane needs one dependent load, not two
            gid = a.slot_blocks[0].offset + np.asarray(a.table.indices[a.tape.slots[0][1]], dtype=np.int64)
            terms_.append(np.full(a.nrec, t_a | PRERESOLVE, dtype=np.int64))
            recs.append(gid)
        else:
            terms_.append(np.full(a.nrec, t_a, dtype=np.int64))
            recs.append(np.arange(a.nrec, dtype=np.int64))
    lrows = np.concatenate(lrows) if lrows else np.zeros(0, np.int64)
    terms_ = np.concatenate(terms_) if terms_ else np.zeros(0, np.int64)
    recs = np.concatenate(recs) if recs else np.zeros(0, np.int64)
    order = np.argsort(lrows, kind="stable")
    counts = np.bincount(lrows, minlength=n)
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    ent = np.stack([terms_[order], recs[order]], axis=1)
    if (counts.size and counts.max() + 1 > 32) or len(dev_index) >= 2**16:
        if valx:
            return _row_layout(base_tp, base_dev, augs, dev_index, None)
        return _i32(ptr, "row CSR"), _i32(ent, "row CSR entries"), None
    # greedy packing of rows (1 + augments each) into 32-lane warps
    length = (counts + 1).astype(np.int64)
    warp_of = np.zeros(n, dtype=np.int64)
    lane0 = np.zeros(n, dtype=np.int64)
    w, fill = 0, 0
    for r, L in enumerate(length.tolist()):
        if fill + L > 32:
            w += 1
            fill = 0
        warp_of[r] = w
        lane0[r] = fill
        fill += L
    n_warps = w + 1 if n else 0
    slots = np.zeros((n_warps * 32, 2), dtype=np.int64)
    slots[:, 0] = -1
    base_slot = warp_of * 32 + lane0
    slots[base_slot, 0] = base_dev
    slots[base_slot, 1] = np.arange(n)
    if ent.shape[0]:
        row_of = lrows[order]
        pos = np.arange(ent.shape[0]) - ptr[row_of] + 1  # 1-based position within the row
        at = base_slot[row_of] + pos
        slots[at, 0] = ent[:, 0] | (pos << 16)  # PRERESOLVE (bit 30) survives the OR
        slots[at, 1] = ent[:, 1]
    return None, None, _i32(slots, "fold slots")


def _bucket_layout(base_tp, augs, nvar):
    """Row buckets of an augment-target block (reference order per row: base,
    then augments in registration order, records in order, autodiff.py:573-580).

    Every augment must be single-variable and field-free (value = f(x[gid])).
    Rows are grouped by their number of augment contributions d into width
    classes W (W/2 < d <= W); within a class rows ascend.  Returns
    ``[(W, rows, ent, rec)]`` with ``rows`` the in-block row ids, ``ent`` a
    (W, n) array of ``gid | sel << 29`` in reference order (sel = index of the
    contributing augment in ``augs``) and ``rec`` the contributing augment
    records (the row thread also writes their Jacobian/Hessian slots in the
    fused set kernel), -1 past a row's d; or None when the block does not fit
    the encoding.  Rows with more than BUCKET_WMAX contributions form the
    classes W = 32 and 16 (listed first): one warp (half warp, for rows of at
    most 15 contributions) per row, arrays (n, W) row-major, lane 0 reserved
    for the base term."""
    if len(augs) > (1 << BUCKET_SEL_BITS) or nvar >= (1 << BUCKET_GID_BITS):
        return None
    n = base_tp.nrec
    lrows, ents, recs = [], [], []
    for sel, a in enumerate(augs):
        lrows.append(np.asarray(a.rows, dtype=np.int64) - base_tp.row_offset)
        gid = a.slot_blocks[0].offset + np.asarray(a.table.indices[a.tape.slots[0][1]], dtype=np.int64)
        ents.append(gid | (sel << BUCKET_GID_BITS))
        recs.append(np.arange(a.nrec, dtype=np.int64))
    lrows = np.concatenate(lrows) if lrows else np.zeros(0, np.int64)
    ents = np.concatenate(ents) if ents else np.zeros(0, np.int64)
    recs = np.concatenate(recs) if recs else np.zeros(0, np.int64)
    order = np.argsort(lrows, kind="stable")  # per row: registration order, then record order
    lrows, ents, recs = lrows[order], ents[order], recs[order]
    counts = np.bincount(lrows, minlength=n)
    if counts.size and (counts.max() > BUCKET_MAX_D or np.unique(counts).size > BUCKET_MAX_N):
        return None
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    # width classes W = 0, 1, 2, 4, 8, ...: rows with W/2 < d <= W, entries
    # padded with -1 (skipped), so the code is unrolled once per class
    width = np.where(counts == 0, 0, 1 << np.ceil(np.log2(np.maximum(counts, 1))).astype(np.int64))
    out = []
    # long rows (d > BUCKET_WMAX): one warp per row, lane l > 0 holds entry l-1
    # (class W = 32, entries laid out row-major so each warp reads 128 B)
    long_ = width > BUCKET_WMAX
    if long_.any():
        lrows_ = np.flatnonzero(long_)
        # rows with <= 15 contributions take half a warp (two rows per warp)
        split = [(32, lrows_[counts[lrows_] > 15]), (16, lrows_[counts[lrows_] <= 15])] if HALF_ROWS \
            else [(32, lrows_)]
        for LW, rows in split:
            if rows.size == 0:
                continue
            ent = np.full((rows.size, LW), -1, dtype=np.int64)
            rec = np.full((rows.size, LW), -1, dtype=np.int64)
            for q, rr in enumerate(rows.tolist()):
                dd = int(counts[rr])
                ent[q, 1:dd + 1] = ents[ptr[rr]:ptr[rr] + dd]
                rec[q, 1:dd + 1] = recs[ptr[rr]:ptr[rr] + dd]
            out.append((LW, rows, ent, rec))
        width = np.where(long_, -1, width)
    for W in np.unique(width).tolist():
        if W < 0:
            continue
        rows = np.flatnonzero(width == W)
        ent = np.full((W, rows.size), -1, dtype=np.int64)
        rec = np.full((W, rows.size), -1, dtype=np.int64)
        for k in range(W):
            has = counts[rows] > k
            ent[k, has] = ents[ptr[rows[has]] + k]
            rec[k, has] = recs[ptr[rows[has]] + k]
        out.append((W, rows, ent, rec))
    return out


class HostLayout:
    """Everything the device needs for one plan, built on the host only."""

    def __init__(self, plan, group_max: int | None = None, exact_zero_sign: bool | None = None):
        self.plan = plan
        self.env_sig = (THREADS_ENV, THREADS_HEAVY, PDL)
        self.group_max_req = group_max
        # zero-sign mode: exact = the reference's signs of zero and w * 0
        # NaN propagation, bit for bit; relaxed = +0.0 structural zeros
        self.relax = _DERIV_ZERO_ELISION if exact_zero_sign is None else not exact_zero_sign
        self.exact_zero_sign = not self.relax
        terms = plan.obj_terms + plan.con_terms
        self.terms = terms
        n_obj = len(plan.obj_terms)
        self.n_obj = n_obj
        self.patterns, self.term_pid = collect_patterns(plan, relax=self.relax)
        self.has_checks = any(pc.has_checks for pc in self.patterns)
        pcs = self.patterns

        dev_index = {id(tp): t for t, tp in enumerate(terms)}
        targets: dict = {}
        for tp in plan.con_terms:
            if tp.kind == "augment":
                targets.setdefault(tp.target_index, []).append(tp)
        self._members: dict = {}
        self.specialised_ok = len(terms) <= META_CONST_MAX_TERMS

        f64 = _Blob(np.float64)
        i32 = _Blob(np.int32)
        descs = []
        self.fold_slots: dict = {}
        self.buckets: dict = {}
        scr = 0
        self.scr0 = []
        period = getattr(plan, "batch_period", None) if (PERIODIC and self.specialised_ok) else None
        for t, tp in enumerate(terms):
            red = _periodic(tp, period) or {"per": 0, "fmask": 0, "imask": 0, "kcol": -1, "g0": 0,
                                            "fcols": {}, "icols": {}}
            d = {
                "f_off": [f64.add(red["fcols"].get(fi, tp.reals[nm])) for fi, nm in enumerate(tp.tape.field_names)],
                "ix_off": [i32.add(_i32(red["icols"].get(c, tp.table.indices[nm]), f"index column {nm!r}"))
                           for c, nm in enumerate(tp.tape.index_names)],
                "per": red["per"], "fmask": red["fmask"], "imask": red["imask"], "kcol": red["kcol"],
                "g0": red["g0"],
                "voff": [blk.offset for blk in tp.slot_blocks],
                "rows_off": i32.add(_i32(tp.rows, "augment rows")) if tp.kind == "augment" else -1,
                "row_ptr_off": -1, "row_ent_off": -1,
                "nrec": tp.nrec, "pattern": self.term_pid[t], "kind": KIND[tp.kind],
                "order": t if tp.kind == "objective" else t - n_obj,
                "row_offset": tp.row_offset if tp.row_offset is not None else 0,
                "cons_direct": int(tp.kind == "constraint" and tp.block_index not in targets),
                "k": tp.tape.k,
                "jac0": tp.jac_slices[0][0] if (tp.kind != "objective" and tp.tape.k) else 0,
                "hess0": tp.hess_start,
                "scr0": scr if tp.kind == "objective" else 0,
            }
            self.scr0.append(d["scr0"])
            if tp.kind == "objective":
                scr += max(tp.tape.k, 1) * tp.nrec
            if tp.kind == "constraint" and tp.block_index in targets:
                augs = targets[tp.block_index]
                self._members[t] = [t] + [dev_index[id(a)] for a in augs]
                bk = None
                if (BUCKETS and self.specialised_ok and not pcs[self.term_pid[t]].has_checks
                        and all(pcs[self.term_pid[dev_index[id(a)]]].valx_ok for a in augs)):
                    bk = _bucket_layout(tp, augs, plan.nvar)
                if bk is not None:
                    lst = []
                    for (dd, rows, ent, rec) in bk:
                        # (entry, record) int2 pairs: one 8-byte load per contribution;
                        # kept writable until the blob is finalised (group attachment
                        # below marks records whose J/H a term group writes: rec = -1)
                        pairs = _i32(np.stack([ent, rec], axis=-1).reshape(-1), "bucket entries")
                        lst.append({
                            "d": dd, "n": int(rows.size), "pairs": pairs,
                            "rows_off": i32.add(_i32(rows, "bucket rows")),
                            "pair_off": i32.add(pairs) if dd else -1,
                            "f_off": [f64.add(np.asarray(tp.reals[nm])[rows]) for nm in tp.tape.field_names],
                            "ix_off": [i32.add(_i32(np.asarray(tp.table.indices[nm])[rows], f"index column {nm!r}"))
                                       for nm in tp.tape.index_names],
                        })
                    self.buckets[t] = {"buckets": lst, "augs": [dev_index[id(a)] for a in augs],
                                       "base_k": tp.tape.k}
                    descs.append(d)
                    continue
                valx = {dev_index[id(a)] for a in augs
                        if self.patterns[self.term_pid[dev_index[id(a)]]].valx_ok} if self.specialised_ok else None
                ptr, ent, slots = _row_layout(tp, t, augs, dev_index, valx)
                if slots is not None:  # int2 entries: ALIGN keeps offsets 8-byte aligned
                    d["row_ent_off"] = i32.add(slots)
                    self.fold_slots[t] = slots.shape[0]
                else:
                    d["row_ptr_off"] = i32.add(ptr)
                    d["row_ent_off"] = i32.add(ent)
            descs.append(d)
        self.descs = descs
        self.n_scr = scr

        # ---- term groups (specialised modules only) ---------------------------
        self.groups = []  # (pid, [term ids], members meta)
        self.group_of: dict = {}
        self.group_augs: dict = {}  # group id -> [(aug term, record offset, member, slot)]
        self.group_max = self._group_max(terms)
        if len(terms) <= META_CONST_MAX_TERMS and self.group_max > 1:
            self._make_groups(terms, descs)
            if ATTACH_AUGS:
                self._attach_augs(terms)
        self.f64 = f64.array()
        self.i32 = i32.array()

        # ---- segments per callback -----------------------------------------
        segs = {m: [] for m in range(_lib.NMODES)}

        def seg(m, t, kind, nrec):
            if nrec > 0:
                segs[m].append((t, kind, nrec))

        # set kernel: row threads of bucketed blocks also write the base term's
        # and their augments' Jacobian/Hessian slots
        fused_set = set()
        for t, info in self.buckets.items():
            fused_set.add(t)
            fused_set.update(info["augs"])
        for t, tp in enumerate(terms):
            k = tp.tape.k
            chk = pcs[self.term_pid[t]].has_checks
            if t in self.group_of and self.groups[self.group_of[t]][1][0] != t:
                continue  # evaluated by its group's first member
            if tp.kind == "objective":
                if k:
                    seg(_lib.MODE_SET, t, SEG_TERM, tp.nrec)
                    seg(_lib.MODE_HESS, t, SEG_TERM, tp.nrec)
                if k or chk:
                    seg(_lib.MODE_GRAD, t, SEG_TERM, tp.nrec)
                if pcs[self.term_pid[t]].root_const is None or chk:
                    seg(_lib.MODE_OBJV, t, SEG_TERM, tp.nrec)
                continue
            direct = bool(descs[t]["cons_direct"])
            if (k or direct) and t not in fused_set:
                seg(_lib.MODE_SET, t, SEG_TERM, tp.nrec)
            if direct:
                seg(_lib.MODE_CONS, t, SEG_TERM, tp.nrec)
            # bucketed blocks and their augments: the row threads write their
            # J/H slots in the set, jac and hess kernels alike
            if (k or chk) and t not in fused_set:
                seg(_lib.MODE_JAC, t, SEG_TERM, tp.nrec)
            if k and t not in fused_set:
                seg(_lib.MODE_HESS, t, SEG_TERM, tp.nrec)
            if tp.kind == "constraint" and not direct:
                if t in self.buckets:
                    for bi, bk in enumerate(self.buckets[t]["buckets"]):
                        nth = bk["n"] * (bk["d"] if bk["d"] >= 16 else 1)  # long rows: a (half) warp per row
                        for mode in (_lib.MODE_SET, _lib.MODE_CONS, _lib.MODE_JAC, _lib.MODE_HESS):
                            seg(mode, t, SEG_BUCKET + 16 * bi, nth)
                elif t in self.fold_slots:
                    seg(_lib.MODE_SET, t, SEG_FOLD, self.fold_slots[t])
                    seg(_lib.MODE_CONS, t, SEG_FOLD, self.fold_slots[t])
                else:
                    seg(_lib.MODE_SET, t, SEG_ROW, tp.nrec)
                    seg(_lib.MODE_CONS, t, SEG_ROW, tp.nrec)
        # CTA order of the segments = dispatch and first-load order.  One-wave
        # sets put the row buckets first (their chain -- entry loads, random
        # gathers, in-order adds -- is the longest; dispatched last they
        # finished last): case13659 6.96 -> 6.68 us.  Many-wave sets keep the
        # natural order (MP96: buckets first 41.5 -> 42.1 us).
        order = os.environ.get("EXA_SEG_ORDER")
        if order is None and choose_threads(sum(sg[2] for sg in segs[_lib.MODE_SET])) == 32:
            order = "BOG"
        if order:
            flags = order[3:]

            def prio(sg):  # order[:3] = permutation of "BGO": buckets, groups, other terms
                t, kind, _ = sg
                if (kind & 15) == SEG_BUCKET:
                    d = self.buckets[t]["buckets"][kind >> 4]["d"]
                    return (order.index("B"), -d if "d" in flags else 0, -t if "t" in flags else 0)
                if t in self.group_of:
                    return (order.index("G"), -t if "r" in flags else 0, 0)
                return (order.index("O"), 0, 0)
            for m in segs:
                segs[m] = sorted(segs[m], key=prio)
        # experiment knob: keep only heavy (k > 2) or only light segments
        filt = os.environ.get("EXA_SEG_FILTER")
        if filt:
            def keep(sg):
                t, kind = sg[0], sg[1]
                heavy = kind == SEG_TERM and terms[t].tape.k > 2
                if filt == "heavy":
                    return heavy
                if filt == "light":
                    return not heavy
                if filt == "fold":
                    return (kind & 15) in (SEG_FOLD, SEG_ROW, SEG_BUCKET)
                if filt == "aug":
                    return kind == SEG_TERM and terms[t].kind == "augment"
                if filt == "other":
                    return kind == SEG_TERM and not heavy and terms[t].kind != "augment"
                return True
            for m in segs:
                segs[m] = [sg for sg in segs[m] if keep(sg)]
        # Each callback -> a heavy kernel (patterns with transcendentals or > 2
        # slots, small CTAs so the few heavy CTAs spread evenly over the 148
        # SMs) and a light kernel (everything else, big CTAs, few registers);
        # kernel id = 2 * mode + {0 heavy, 1 light}.  They run concurrently.
        self.threads = (THREADS_HEAVY, choose_threads(sum(sg[2] for sg in segs[_lib.MODE_SET])))
        self.segs = {}
        self.n_ctas = []
        for m in range(_lib.NMODES):
            for half in (0, 1):
                kid = 2 * m + half
                th = self.threads[half]
                cta = 0
                lst = []
                for (t, kind, nrec) in segs[m]:
                    if kind == SEG_TERM and t in self.group_of:
                        kind = SEG_GROUP
                    heavy = SPLIT_HEAVY and kind in (SEG_TERM, SEG_GROUP) and pcs[self.term_pid[t]].heavy
                    if heavy != (half == 0):
                        continue
                    rpt = pcs[self.term_pid[t]].rpt if kind == SEG_TERM else (GROUP_RPT if kind == SEG_GROUP else 1)
                    if kind == SEG_GROUP:  # segment names the group, not the term
                        t = self.group_of[t]
                    lst.append((t, kind, cta, nrec, rpt))
                    cta += (nrec + th * rpt - 1) // (th * rpt)
                self.segs[kid] = lst
                self.n_ctas.append(cta)

        # ---- objective program ---------------------------------------------
        leaves: list = []
        prog: list = []
        for t, tp in enumerate(plan.obj_terms):
            rc = pcs[self.term_pid[t]].root_const
            if rc is not None:
                prog.append(_const_op(float(rc) * tp.nrec))
            elif tp.nrec == 0:
                prog.append(_const_op(0.0))
                prog.append((OP_ZERO_PLUS, 0, 0))
            else:
                pairwise_program(tp.nrec, self.scr0[t], leaves, prog)
                prog.append((OP_ZERO_PLUS, 0, 0))
            prog.append((OP_TOTAL_ADD, 0, 0))
        self.leaves = np.array(leaves, dtype=np.int64).reshape(-1, 2)
        self.prog = np.array(prog, dtype=np.int64).reshape(-1, 3)
        self.grad_ptr, self.grad_ent = self._grad_csr(plan.nvar)
        self.fill_jac, self.fill_hess = self._host_fill(terms)

        # ---- module source ---------------------------------------------------
        self.specialised = len(terms) <= META_CONST_MAX_TERMS
        # persistent kernels (specialised modules): PERSIST virtual CTAs per real CTA
        self.persist = [PERSIST if (self.specialised and self.n_ctas[kid]) else 0 for kid in range(_lib.NKERN)]
        self.pdl = PDL
        # CTA dispatch order of the many-wave set kernel for batched models
        # whose variables are (element, instance) element-major: CTAs sorted by
        # the instance window their records gather from, so the x / y rows of
        # one window stay in L2 while all of its terms and rows are evaluated
        self.cta_perm_off = None
        period = getattr(plan, "batch_period", None)
        if (self.specialised and LOCALITY_W > 0 and period and period >= 2 * LOCALITY_W
                and self.threads[1] > 32 and not any(self.persist)):
            perm = self._locality_order(terms, int(period))
            if perm is not None:
                self.cta_perm_off = int(self.i32.size)
                self.i32 = np.concatenate([self.i32, perm.astype(np.int32)])
        self.source = module_source(self.patterns, layout=self if self.specialised else None,
                                    threads=self.threads[1])

    def jac_direct(self, jp):
        """Term-group members whose Jacobian entries the compressed-set
        kernels write directly: ({term: jc0}, uint8 mask of their raw J slots).

        A member is direct when every one of its records' rows holds exactly
        that record's k slots, one raw slot per compressed entry, with
        distinct columns: the row's entries are then its slots in column
        order, and slot s of record r lands at ``jc0 + k r + rank`` (rank = how
        many of the record's other columns are smaller), ``jc0`` = the row
        block's first entry in ``jp`` (np.unique order of
        ``compress_coordinates``, reference autodiff.py:677-689).  OPF: the
        four flow blocks, thermal limits and angle differences -- every
        Jacobian row but the bus balances.  The result is kept on the layout
        (``jdirect``) for :meth:`compressed_source`."""
        jdir, mask = {}, np.zeros(jp.slot_map.size, dtype=np.uint8)
        if jp.nnz:
            counts = np.bincount(jp.slot_map, minlength=jp.nnz)
            for t in sorted(self.group_of):
                tp = self.terms[t]
                k, n = tp.tape.k, tp.nrec
                if tp.kind != "constraint" or tp.row_offset is None or not k or not n:
                    continue
                raw = np.stack([np.arange(lo, lo + n, dtype=np.int64) for lo, _ in tp.jac_slices[:k]])
                e = jp.slot_map[raw]
                if not np.all(counts[e] == 1):
                    continue
                cols = np.stack([np.asarray(c, dtype=np.int64) for c in tp.cols[:k]])
                srt = np.sort(cols, axis=0)
                if k > 1 and np.any(srt[1:] == srt[:-1]):
                    continue
                rank = (cols[None, :, :] < cols[:, None, :]).sum(axis=1)
                jc0 = int(np.searchsorted(jp.rows, tp.row_offset))
                if not np.array_equal(e, jc0 + k * np.arange(n, dtype=np.int64)[None, :] + rank):
                    continue
                jdir[t] = jc0
                mask[raw.ravel()] = 1
        self.jdirect = jdir
        return jdir, mask

    def hess_local(self, hp):
        """Group-local compressed Hessian entries: (hlocal, hpos, mask).

        A *class* is a set of one H pair per term-group member (members in
        raw-slot order) whose slots, for a record, are ALL the non-known
        slots of one compressed entry of ``hp`` -- e.g. H(vm_f, va_t) of a
        branch, to which exactly its four flow terms contribute.  The group
        thread then folds the class in np.bincount's order (0.0 + the first
        member's value + the next ...) and stores the entry itself.  Classes
        are found on a sample of records (columns with equal entries) and
        validated on every record; ``hpos[off + r]`` is the entry of record r,
        or -1 where the entry has other slots too (parallel branches): that
        record writes its raw slots for the segmented sum.  ``hlocal[gid][m]
        = {pair: (class, position, size, off)}``; ``mask`` flags the raw H
        slots folded in-thread (left out of the segmented sum)."""
        known = np.zeros(hp.slot_map.size, dtype=bool)
        for a, n_, _ in self.fill_hess:
            known[a:a + n_] = True
        cnt = np.bincount(hp.slot_map[~known], minlength=hp.nnz)
        cnt_all = np.bincount(hp.slot_map, minlength=hp.nnz)
        hlocal, pos, mask = {}, [], np.zeros(hp.slot_map.size, dtype=np.uint8)
        at = ncls = 0
        for gid, (_pid, grp, _members) in enumerate(self.groups):
            n = self.terms[grp[0]].nrec
            for zero in ((False, True) if os.environ.get("EXA_HLOCAL_ZERO", "1") == "1" else (False,)):
                # value classes (slots that are not known +0.0), then classes of
                # known +0.0 slots whose entries hold nothing else: the thread
                # writes +0.0 there instead of the segmented sum
                cols = []  # (member, pair, raw slot of record 0)
                for m, u in enumerate(grp):
                    tp = self.terms[u]
                    if not tp.tape.k or tp.nrec != n:
                        continue
                    for pr in tp.hess_pairs:
                        if bool(known[pr.start]) == zero:
                            cols.append((m, (pr.start - tp.hess_start) // n, pr.start))
                if not cols or n == 0:
                    continue
                at, ncls = self._local_classes(hp, gid, n, cols, cnt_all if zero else cnt, zero, hlocal, pos,
                                               mask, at, ncls)
        self.hlocal = hlocal
        hpos = np.concatenate(pos) if pos else np.zeros(0, dtype=np.int32)
        return hlocal, hpos, mask

    def _local_classes(self, hp, gid, n, cols, cnt, zero, hlocal, pos, mask, at, ncls):
        """Classes among ``cols`` of group ``gid`` (see :meth:`hess_local`)."""
        E = np.stack([hp.slot_map[st:st + n] for _, _, st in cols])
        samp = E[:, :: max(1, n // 4096)]
        parent = list(range(len(cols)))

        def find(a):
            while parent[a] != a:
                parent[a] = parent[parent[a]]
                a = parent[a]
            return a

        for a in range(len(cols)):
            for b in range(a + 1, len(cols)):
                if np.mean(samp[a] == samp[b]) > 0.5:
                    parent[find(b)] = find(a)
        classes: dict = {}
        for a in range(len(cols)):
            classes.setdefault(find(a), []).append(a)
        for members in classes.values():
            members.sort(key=lambda a: cols[a][2])  # raw-slot (fold) order
            ms = [cols[a][0] for a in members]
            if len(set(ms)) != len(ms) or ms != sorted(ms):
                continue  # one slot per member, members in fold order
            e0 = E[members[0]]
            valid = cnt[e0] == len(members)
            for a in members[1:]:
                valid &= E[a] == e0
            if valid.mean() < 0.5:
                continue
            off = at
            pos.append(np.where(valid, e0, -1).astype(np.int32))
            at += n
            for q, a in enumerate(members):
                m, pair, st = cols[a]
                hlocal.setdefault(gid, {}).setdefault(m, {})[pair] = (ncls, q, len(members), off, zero)
                mask[st:st + n][valid] = 1
            ncls += 1
        return at, ncls

    def compressed_source(self) -> str:
        """CUDA source of the compressed-set module (set kernels
        ``exa_k_setc_h`` / ``_l``; needs :meth:`jac_direct` first)."""
        return module_source(self.patterns, layout=self, threads=self.threads[1], compressed=True)

    def _locality_order(self, terms, period: int):
        """Real CTA -> virtual CTA of the set kernel (light half): virtual CTAs
        sorted by (instance window of their first record, virtual index).  A
        record's instance is the first gathered variable's index modulo the
        model's ``batch_period`` (element-major batched layouts: variable
        (i, k) at i * period + k); row buckets use their row's base term."""
        kid = 2 * _lib.MODE_SET + 1
        th = self.threads[1]
        n = self.n_ctas[kid]
        if n == 0:
            return None
        key = np.zeros(n, dtype=np.int64)
        for (t, kind, cta0, nrec, rpt) in self.segs[kid]:
            nc = (nrec + th * rpt - 1) // (th * rpt)
            r0 = np.arange(nc, dtype=np.int64) * th * rpt
            col = None
            if kind == SEG_GROUP:
                u = self.groups[t][1][0]
                col = np.asarray(terms[u].cols[0], dtype=np.int64)[r0]
            elif kind == SEG_TERM and terms[t].tape.k:
                col = np.asarray(terms[t].cols[0], dtype=np.int64)[r0]
            elif (kind & 15) == SEG_BUCKET:
                bk = self.buckets[t]["buckets"][kind >> 4]
                q = r0 // (bk["d"] if bk["d"] >= 16 else 1)
                rows = self.i32[bk["rows_off"]:bk["rows_off"] + bk["n"]].astype(np.int64)[np.minimum(q, bk["n"] - 1)]
                col = (np.asarray(terms[t].cols[0], dtype=np.int64)[rows] if terms[t].tape.k else rows)
            if col is None:
                col = np.minimum(r0, nrec - 1)
            key[cta0:cta0 + nc] = (col % period) // LOCALITY_W
        return np.lexsort((np.arange(n), key))

    def _group_max(self, terms) -> int:
        if self.group_max_req is not None:
            return int(self.group_max_req)
        if GROUP_MAX_ENV != "auto":
            return int(GROUP_MAX_ENV)
        # threads of the set kernel with groups of 4 heavy terms (an estimate:
        # light constraint terms counted as if ungrouped)
        est = sum(tp.nrec / 4 if self.patterns[self.term_pid[t]].heavy else tp.nrec
                  for t, tp in enumerate(terms) if tp.kind != "augment")
        if choose_threads(int(est)) != 32:
            return 2  # many-wave sets
        # one-wave sets: groups of four halve the voltage gathers (case13659
        # 5.65 us); a set too small to give every SM a warp of groups of four
        # needs the parallelism of groups of two (case1354 3.37 -> 3.19 us)
        heavy = sum(tp.nrec for t, tp in enumerate(terms)
                    if tp.kind != "augment" and self.patterns[self.term_pid[t]].heavy)
        return 4 if heavy / 4 >= SM_COUNT * 32 else 2

    def _make_groups(self, terms, descs):
        import hashlib

        def col_hash(arr):
            return hashlib.blake2b(np.ascontiguousarray(arr, dtype=np.int64).tobytes(), digest_size=16).digest()

        sig = {}
        for t, tp in enumerate(terms):
            pc = self.patterns[self.term_pid[t]]
            if not pc.heavy or tp.nrec == 0:
                continue
            key = (self.term_pid[t], tp.nrec, tp.kind, descs[t]["cons_direct"])
            sig.setdefault(key, []).append(t)
        hashes = {t: [col_hash(tp.table.indices[nm]) for nm in tp.tape.index_names]
                  for t, tp in enumerate(terms) if tp.nrec}
        groups = []
        for key, cand in sig.items():
            free = list(cand)
            while free:
                t0 = free.pop(0)
                grp = [t0]
                cols = set(hashes[t0])
                for u in list(free):
                    if len(grp) >= self.group_max:
                        break
                    if cols & set(hashes[u]):
                        grp.append(u)
                        cols |= set(hashes[u])
                        free.remove(u)
                if len(grp) >= 2:
                    groups.append(grp)
        # Light constraint terms over the same records that gather some of the
        # same variables (OPF: thermal limits and angle differences of the
        # branches) join the heavy group with which they share most gathers;
        # their loads and gathers are then shared (fewer random L2 sectors).
        if ATTACH and groups:
            def keys(t):
                tp = terms[t]
                hs = hashes[t]
                ss = self.patterns[self.term_pid[t]].slot_struct
                return {(id(tp.slot_blocks[s_]), hs[ic]) for s_, (_, ic) in enumerate(ss)}

            def attachable(t):
                tp = terms[t]
                pc = self.patterns[self.term_pid[t]]
                return (tp.kind == "constraint" and descs[t]["cons_direct"] and tp.tape.k > 0
                        and not pc.heavy and not pc.has_checks and tp.nrec > 0)

            in_grp = {t for grp in groups for t in grp}
            gkeys = [set().union(*(keys(t) for t in grp)) for grp in groups]
            for t in range(len(terms)):
                if t in in_grp or not attachable(t):
                    continue
                kt = keys(t)
                best, score = None, 0
                for gi, grp in enumerate(groups):
                    t0 = grp[0]
                    if terms[t0].nrec != terms[t].nrec or terms[t0].kind != "constraint" or not descs[t0]["cons_direct"]:
                        continue
                    sc = len(kt & gkeys[gi])
                    if sc > score or (sc == score and sc and len(grp) < len(groups[best])):
                        best, score = gi, sc
                if best is not None:
                    groups[best].append(t)
                    gkeys[best] |= kt
        for grp in groups:
            t0 = grp[0]
            uid: dict = {}
            bid: dict = {}
            members = []
            for t in grp:
                members.append({
                    "cols": [uid.setdefault(h, len(uid)) for h in hashes[t]],
                    "blocks": [bid.setdefault(id(b), len(bid)) for b in terms[t].slot_blocks],
                })
            gi = len(self.groups)
            self.groups.append((self.term_pid[t0], grp, members))
            for t in grp:
                self.group_of[t] = gi

    def _attach_augs(self, terms):
        """Bucketed augments (single-variable, field-free: pg, -p, -q ...) whose
        records ``[off, off + n)`` gather, record for record, the same variable
        as a slot of a term group over n records: the group thread writes
        those records' J/H slots (coalesced, the variable already gathered)
        instead of the row thread (scattered).  OPF: the -p/-q balance
        augments of the from- and to-ends ride on the two flow groups."""
        for gi, (_, grp, _) in enumerate(self.groups):
            n = terms[grp[0]].nrec
            slot_gids = []
            for m, u in enumerate(grp):
                for s_ in range(terms[u].tape.k):
                    slot_gids.append((m, s_, np.asarray(terms[u].cols[s_], dtype=np.int64)))
            for t, info in self.buckets.items():
                for sel, u in enumerate(info["augs"]):
                    a = terms[u]
                    if a.nrec < n or a.nrec % n:
                        continue
                    gid = np.asarray(a.cols[0], dtype=np.int64)
                    for off in range(0, a.nrec, n):
                        if any(x[1] == off for x in self.group_augs.get(gi, []) if x[0] == u):
                            continue
                        hit = next(((m, s_) for (m, s_, g) in slot_gids if np.array_equal(g, gid[off:off + n])), None)
                        if hit is None:
                            continue
                        self.group_augs.setdefault(gi, []).append((u, off, hit[0], hit[1]))
                        for bk in info["buckets"]:  # the row thread no longer writes them
                            pr = bk["pairs"].reshape(-1, 2)
                            e, rc = pr[:, 0], pr[:, 1]
                            mine = (e >= 0) & ((e >> BUCKET_GID_BITS) == sel) & (rc >= off) & (rc < off + n)
                            rc[mine] = -1

    # accessors used by the specialised-kernel generator (jit.py)
    def term_descs(self):
        return self.descs

    def row_members(self):
        return self._members

    def mode_segments(self, m):
        return self.segs[m]

    def _host_fill(self, terms):
        """Runs of raw J / H slots the host path writes on the host instead of
        copying them from the device (the kernels still write them: device
        callers get every slot).

        * constant runs, int64 triples (first slot, length, value bits):
          constant Jacobian slots and -- under the zero-sign relaxation -- the
          structural-zero Hessian pairs (+0.0); adjacent equal runs merged;
        * exact zero-sign mode: *weighted-zero* runs, int64 quadruples (first
          H slot, length, offset into ``wz_rows`` or -1 for the objective
          weight, bits of the structural constant z): slot i of the run is
          ``mult[wz_rows[off + i]] * z`` (or ``obj_weight * z``), the
          reference's ``weight * 0.0`` with its sign and NaN propagation
          (autodiff.py:652), computed from the caller's host multipliers.
        """
        runs_j, runs_h, runs_w = [], [], []
        rows_pool, rows_off = [], {}
        at = 0
        for t, tp in enumerate(terms):
            pc = self.patterns[self.term_pid[t]]
            d, n = self.descs[t], tp.nrec
            if n == 0 or not pc.k:
                continue
            if tp.kind != "objective":
                for s_, v in pc.jconst.items():
                    runs_j.append((d["jac0"] + s_ * n, n, int(np.float64(v).view(np.int64))))
            for pr in pc.hzero:
                runs_h.append((d["hess0"] + pr * n, n, 0))
            for pr, z in pc.hzero_w:
                if tp.kind == "objective":
                    off = -1
                else:
                    off = rows_off.get(t)
                    if off is None:
                        off = rows_off[t] = at
                        rows_pool.append(np.asarray(tp.rows, dtype=np.int32))
                        at += n
                runs_w.append((d["hess0"] + pr * n, n, off, int(np.float64(z).view(np.int64))))

        def merge(runs):
            out = []
            for a, n, v in sorted(runs):
                if out and out[-1][0] + out[-1][1] == a and out[-1][2] == v:
                    out[-1][1] += n
                else:
                    out.append([a, n, v])
            return np.array(out, dtype=np.int64).reshape(-1, 3)

        self.fill_wzero = np.array(sorted(runs_w), dtype=np.int64).reshape(-1, 4)
        self.wz_rows = (np.concatenate(rows_pool) if rows_pool else np.zeros(0, dtype=np.int32)).astype(np.int32)
        return merge(runs_j), merge(runs_h)

    def _grad_csr(self, nvar):
        plan = self.plan
        vars_, gidx, grp = [], [], []
        g = 0
        for t, tp in enumerate(plan.obj_terms):
            for s in range(tp.tape.k):
                vars_.append(np.asarray(tp.cols[s], dtype=np.int64))
                gidx.append(self.scr0[t] + s * tp.nrec + np.arange(tp.nrec, dtype=np.int64))
                grp.append(np.full(tp.nrec, g, dtype=np.int64))
                g += 1
        if not vars_:
            return None, None
        vars_ = np.concatenate(vars_)
        gidx = np.concatenate(gidx)
        grp = np.concatenate(grp)
        order = np.argsort(vars_, kind="stable")
        sv, sg, si = vars_[order], grp[order], gidx[order]
        new = np.ones(sv.size, dtype=bool)
        new[1:] = (sv[1:] != sv[:-1]) | (sg[1:] != sg[:-1])
        ent = si | (new.astype(np.int64) << 62)
        ptr = np.zeros(nvar + 1, dtype=np.int64)
        np.cumsum(np.bincount(sv, minlength=nvar), out=ptr[1:])
        return ptr, ent


def host_layout(plan, group_max: int | None = None, exact_zero_sign: bool | None = None) -> HostLayout:
    """The plan's device layout (cached on the plan); ``group_max`` overrides
    the automatic term-group size (the strided-batch plan uses 2),
    ``exact_zero_sign`` the default zero-sign mode."""
    exact = (not _DERIV_ZERO_ELISION) if exact_zero_sign is None else bool(exact_zero_sign)
    if group_max is None and exact == (not _DERIV_ZERO_ELISION):
        lay = getattr(plan, "_exa_layout", None)
        if lay is None or lay.env_sig != (THREADS_ENV, THREADS_HEAVY, PDL):
            lay = HostLayout(plan)
            plan._exa_layout = lay
        return lay
    cache = plan.__dict__.setdefault("_exa_layouts", {})
    key = (THREADS_ENV, THREADS_HEAVY, PDL, group_max, exact)
    if key not in cache:
        cache[key] = HostLayout(plan, group_max, exact_zero_sign=exact)
    return cache[key]


def precompile(plan) -> bytes:
    """JIT (or fetch from cache) the module for a host plan -- and the
    strided-batch variant when the plan groups more than two terms; no GPU
    needed."""
    lay = host_layout(plan)
    if lay.specialised and lay.group_max > 2:
        compile_module(host_layout(plan, 2).source)
    return compile_module(lay.source)


class DevicePlan:
    """The model's plan resident on one GPU, with its compiled kernels."""

    def __init__(self, model, device=None, group_max: int | None = None, exact_zero_sign: bool | None = None):
        import torch

        if not torch.cuda.is_available():
            raise _lib.ExaError("no CUDA device: the callback engine runs on B200 only (no CPU path)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        plan = model.plan
        self.model = model
        self.plan = plan
        lay = host_layout(plan, group_max, exact_zero_sign)
        self.layout = lay
        self.exact_zero_sign = lay.exact_zero_sign
        self.patterns = lay.patterns
        self.has_checks = lay.has_checks
        self.n_ctas = lay.n_ctas
        self.cubin = compile_module(lay.source)

        terms = lay.terms
        descs = (_lib.TermDesc * max(1, len(terms)))()
        for t, d in enumerate(lay.descs):
            td = descs[t]
            for i in range(_lib.MAXF):
                td.f_off[i] = d["f_off"][i] if i < len(d["f_off"]) else -1
            for i in range(_lib.MAXI):
                td.ix_off[i] = d["ix_off"][i] if i < len(d["ix_off"]) else -1
            for s, vo in enumerate(d["voff"]):
                td.voff[s] = vo
            for k in ("rows_off", "row_ptr_off", "row_ent_off", "nrec", "pattern", "kind", "order",
                      "row_offset", "cons_direct", "k", "jac0", "hess0", "scr0"):
                setattr(td, k, d[k])
        seg_arrays = []
        for m in range(_lib.NKERN):
            lst = lay.segs[m]
            arr = (_lib.SegDesc * max(1, len(lst)))()
            for s, (t, kind, cta0, nrec, rpt) in enumerate(lst):
                arr[s].term, arr[s].kind, arr[s].cta0, arr[s].nrec = t, (kind & 15) | (rpt << 8), cta0, nrec
            seg_arrays.append(arr)

        desc = _lib.PlanDesc()
        desc.abi_version = _lib.ABI_VERSION
        desc.device = self.device
        desc.nvar, desc.ncon = model.nvar, model.ncon
        desc.n_jac, desc.n_hess = plan.n_jac_slots, plan.n_hess_slots
        desc.f64 = lay.f64.ctypes.data_as(C.POINTER(C.c_double))
        desc.n_f64 = lay.f64.size
        desc.i32 = lay.i32.ctypes.data_as(C.POINTER(C.c_int32))
        desc.n_i32 = lay.i32.size
        desc.terms = C.cast(descs, C.POINTER(_lib.TermDesc))
        desc.n_terms = len(terms)
        desc.threads[0], desc.threads[1] = lay.threads
        for m in range(_lib.NKERN):
            desc.segs[m] = C.cast(seg_arrays[m], C.POINTER(_lib.SegDesc))
            desc.n_segs[m] = len(lay.segs[m])
            desc.n_ctas[m] = lay.n_ctas[m]
            desc.persist[m] = lay.persist[m]
        desc.pdl = int(lay.pdl)
        desc.batchable = int(lay.specialised and not any(lay.persist))
        self._fill = np.ascontiguousarray(np.concatenate([lay.fill_jac, lay.fill_hess]).reshape(-1), dtype=np.int64)
        desc.host_fill = self._fill.ctypes.data_as(C.POINTER(C.c_int64))
        desc.n_fill_jac, desc.n_fill_hess = len(lay.fill_jac), len(lay.fill_hess)
        self._wz = np.ascontiguousarray(lay.fill_wzero.reshape(-1), dtype=np.int64)
        self._wz_rows = np.ascontiguousarray(lay.wz_rows, dtype=np.int32)
        desc.host_wzero = self._wz.ctypes.data_as(C.POINTER(C.c_int64))
        desc.n_wzero = len(lay.fill_wzero)
        desc.host_wzero_rows = self._wz_rows.ctypes.data_as(C.POINTER(C.c_int32))
        desc.n_wzero_rows = self._wz_rows.size
        n_obj, n_con = len(plan.obj_terms), len(plan.con_terms)
        bases = {
            _lib.MODE_SET: (n_con, 0), _lib.MODE_CONS: (0, 0), _lib.MODE_JAC: (0, 0),
            _lib.MODE_HESS: (0, n_obj), _lib.MODE_OBJV: (0, 0), _lib.MODE_GRAD: (0, 0),
        }
        for m, (ob, cb) in bases.items():
            desc.err_base[m][0] = ob
            desc.err_base[m][1] = cb
        desc.n_vscr = desc.n_gscr = lay.n_scr
        desc.leaves = lay.leaves.ctypes.data_as(C.POINTER(C.c_int64))
        desc.n_leaves = lay.leaves.shape[0]
        desc.obj_prog = lay.prog.ctypes.data_as(C.POINTER(C.c_int64))
        desc.n_prog = lay.prog.shape[0]
        if lay.grad_ptr is not None:
            desc.grad_ptr = lay.grad_ptr.ctypes.data_as(C.POINTER(C.c_int64))
            desc.grad_ent = lay.grad_ent.ctypes.data_as(C.POINTER(C.c_int64))
            desc.n_grad_ent = lay.grad_ent.size
        cub = C.create_string_buffer(self.cubin, len(self.cubin))
        desc.cubin = C.cast(cub, C.c_void_p)
        desc.cubin_size = len(self.cubin)
        desc.has_domain_checks = int(self.has_checks)
        lib = _lib.load()
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(lib.exa_plan_create(C.byref(desc), C.byref(handle)), "exa_plan_create")
        self.handle = handle
        self._lib = lib
        self.device_bytes = int(lay.f64.nbytes + lay.i32.nbytes)
        self._tls = threading.local()
        self._ws_lock = threading.Lock()
        self._workspaces: list = []

    def compressed_masks(self):
        """(J mask, H mask): raw slots the compressed-set kernels fold into
        their compressed entries themselves -- whole-row Jacobian blocks
        (``HostLayout.jac_direct``) and group-local Hessian entries
        (``HostLayout.hess_local``) -- after compiling and attaching the
        plan's compressed-set module (once per plan); (None, None) for
        generic modules, nothing eligible, or ``EXA_JDIRECT=0``."""
        if hasattr(self, "_cmp_masks"):
            return self._cmp_masks
        self._cmp_masks = (None, None)
        lay = self.layout
        if not lay.specialised or os.environ.get("EXA_JDIRECT", "1") != "1":
            return self._cmp_masks
        from .autodiff import model_patterns

        jp, hp = model_patterns(self.model)
        jdir, jmask = lay.jac_direct(jp)
        hloc, hpos, hmask = lay.hess_local(hp) if os.environ.get("EXA_HLOCAL", "1") == "1" else ({}, None, None)
        if not jdir and not hloc:
            return self._cmp_masks
        if not hloc:
            lay.hlocal, hpos = {}, np.zeros(0, dtype=np.int32)
        cubin = compile_module(lay.compressed_source())
        buf = C.create_string_buffer(cubin, len(cubin))
        hpos = np.ascontiguousarray(hpos, dtype=np.int32)
        import torch

        with torch.cuda.device(self.device):
            _lib.check(self._lib.exa_plan_attach_compressed(self.handle, C.cast(buf, C.c_void_p), len(cubin),
                                                            hpos.ctypes.data if hpos.size else None, hpos.size),
                       "exa_plan_attach_compressed")
        self._cmp_masks = (jmask if jdir else None, hmask if hloc else None)
        return self._cmp_masks

    def workspace(self) -> C.c_void_p:
        """The calling thread's workspace (objective / gradient scratch,
        domain-error word, host-path staging, the aux stream of the light
        kernels).  The plan itself is immutable, so one model is shareable
        across threads (reference ``core.py:301-305``): every Python thread
        evaluates through its own workspace, created on first use and
        destroyed with the plan."""
        ws = getattr(self._tls, "ws", None)
        if ws is None:
            import torch

            ws = C.c_void_p()
            with torch.cuda.device(self.device):
                _lib.check(self._lib.exa_workspace_create(self.handle, C.byref(ws)), "exa_workspace_create")
            with self._ws_lock:
                self._workspaces.append(ws)
            self._tls.ws = ws
        return ws

    def info(self):
        b, r = C.c_int64(), C.c_int32()
        _lib.check(self._lib.exa_plan_info(self.handle, C.byref(b), C.byref(r)), "plan_info")
        return {"device_bytes": b.value, "regs_set_kernel": r.value, "patterns": len(self.patterns),
                "specialised": self.layout.specialised,
                "ctas": {f"{m}_{h}": self.n_ctas[2 * i + j]
                         for i, m in enumerate(("set", "cons", "jac", "hess", "objv", "grad"))
                         for j, h in enumerate(("h", "l"))}}

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                for ws in getattr(self, "_workspaces", ()):
                    self._lib.exa_workspace_destroy(ws)
                self._lib.exa_plan_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self.handle = None
