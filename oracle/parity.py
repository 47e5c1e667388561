"""Parity comparator of SURVEY §8(c) -- TEST INFRASTRUCTURE ONLY.

Used by ``tests/`` and ``tools/parity_report.py`` to judge the CUDA outputs
against the oracle (numpy = the reference's arithmetic, pinned bit-exact to
the reference's goldens) and against the oracle with correctly-rounded
sin/cos (``oracle/crtrig``).  Never imported by the product package.

Comparator (SURVEY §8c "Parity comparator (recommended)"):

* per element: ``ref == 0`` requires ``gpu == 0`` (IEEE, -0.0 == 0.0), else
  ``|gpu - ref| <= 1e-12 |ref|`` -- a *strict violation* otherwise;
* per array and per family (term block): max relative deviation, the count
  of strict violations, the count of IEEE-unequal elements, the count of
  zero-sign mismatches (both zero, sign bits differ), and the
  *conditioning-scaled* max ``|gpu - ref| / scale``.  For the polar flow
  family (F3, reference ``opf.py:318-350``) the scale of
  an element is the sum of the magnitudes of the terms it is computed from:
  ``|a2 cos d| + |a3 sin d|`` for A-entries, ``|a2 sin d| + |a3 cos d|`` for
  B-entries, times ``|vi vj|`` / ``|vi|`` / ``|vj|`` and ``|w|`` as the entry
  carries them; every other element's scale is ``|ref|`` (its relative
  deviation).
"""

from __future__ import annotations

import numpy as np

RTOL = 1e-12  # north_star: values within 1e-12 relative (fp64)


def ieee_equal(a, b) -> bool:
    """Element-wise IEEE equality (-0.0 == +0.0; NaN matches NaN)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and bool(np.all((a == b) | (np.isnan(a) & np.isnan(b))))


def bit_equal(a, b) -> bool:
    """Identical IEEE-754 bit patterns (signs of zero included); NaNs match
    any NaN (IEEE leaves the payload unspecified: x86 and the GPU produce
    different default NaNs)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    same = a.view(np.uint64) == b.view(np.uint64)
    return bool(np.all(same | (np.isnan(a) & np.isnan(b))))


def strict_mask(gpu, ref, rtol=RTOL):
    gpu, ref = np.asarray(gpu, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    zero = ref == 0.0
    bad = np.zeros(ref.shape, dtype=bool)
    bad[zero] = gpu[zero] != 0.0
    nz = ~zero
    bad[nz] = ~(np.abs(gpu[nz] - ref[nz]) <= rtol * np.abs(ref[nz]))
    return bad


def strict_violations(gpu, ref, rtol=RTOL):
    return np.flatnonzero(strict_mask(gpu, ref, rtol))


def zero_sign_mismatches(gpu, ref) -> int:
    gpu, ref = np.asarray(gpu, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    both = (gpu == 0.0) & (ref == 0.0)
    return int(np.count_nonzero(both & (np.signbit(gpu) != np.signbit(ref))))


# ---------------------------------------------------------------------------
# families and conditioning scales
# ---------------------------------------------------------------------------

def _is_flow(tp) -> bool:
    ops = {ins[0] for ins in tp.tape.instr}
    return tp.tape.k == 5 and {"sin", "cos"} <= ops and {"a1", "a2", "a3"} <= set(tp.tape.field_names)


def family_name(tp) -> str:
    ops = {ins[0] for ins in tp.tape.instr}
    if _is_flow(tp):
        short = "flow"
    elif tp.kind == "objective":
        short = "objective"
    elif tp.kind == "augment":
        short = "augment"
    elif ops & {"sin", "cos", "exp", "log", "sqrt", "pow", "div"}:
        short = "nonlinear"
    else:
        short = f"k{tp.tape.k}"
    return f"{tp.kind}[{tp.block_index}]:{short}"


def families(plan):
    """Per-output family ids: (names, cons_fam[ncon], jac_fam[n_jac], hess_fam[n_hess]).

    A constraint row belongs to its base block (augments add into rows of
    their target block); J / H slots belong to the term that writes them."""
    names = []
    cf = np.full(plan.ncon, -1, dtype=np.int32)
    jf = np.full(plan.n_jac_slots, -1, dtype=np.int32)
    hf = np.full(plan.n_hess_slots, -1, dtype=np.int32)
    for tp in plan.obj_terms + plan.con_terms:
        fid = len(names)
        names.append(family_name(tp))
        if tp.kind == "constraint":
            cf[tp.row_offset: tp.row_offset + tp.nrec] = fid
        for lo, hi in tp.jac_slices or []:
            jf[lo:hi] = fid
        for pr in tp.hess_pairs or []:
            hf[pr.start: pr.start + tp.nrec] = fid
    return names, cf, jf, hf


def _flow_scales(tp, x, mult, obj_weight):
    """Per-record condition scales of one F3 term."""
    a1, a2, a3 = (tp.reals[n] for n in ("a1", "a2", "a3"))
    # slot order [vm_i, vm_j, va_i, va_j, flow_d] (post-order DFS of the kernel)
    vi, vj, ti, tj, yd = (x[c] for c in tp.cols)
    d = ti - tj
    cA = np.abs(a2 * np.cos(d)) + np.abs(a3 * np.sin(d))
    cB = np.abs(a2 * np.sin(d)) + np.abs(a3 * np.cos(d))
    w = np.abs(mult[tp.rows]) if tp.kind != "objective" else np.full(tp.nrec, abs(obj_weight))
    avij = np.abs(vi * vj)
    cons = np.abs(a1 * vi * vi) + avij * cA + np.abs(yd)
    jac = [np.abs(2 * a1 * vi) + np.abs(vj) * cA, np.abs(vi) * cA, avij * cB, avij * cB, np.ones(tp.nrec)]
    z = np.zeros(tp.nrec)
    hess = {(0, 0): np.abs(2 * a1) * w, (1, 0): cA * w, (1, 1): z, (2, 0): np.abs(vj) * cB * w,
            (2, 1): np.abs(vi) * cB * w, (2, 2): avij * cA * w, (3, 0): np.abs(vj) * cB * w,
            (3, 1): np.abs(vi) * cB * w, (3, 2): avij * cA * w, (3, 3): avij * cA * w}
    return cons, jac, hess


def condition_scales(plan, x, mult, obj_weight, ref):
    """Scale arrays (cons, jac, hess) for the conditioning-scaled deviation."""
    c_ref, j_ref, h_ref = ref
    cs, js, hs = np.abs(c_ref).copy(), np.abs(j_ref).copy(), np.abs(h_ref).copy()
    for tp in plan.obj_terms + plan.con_terms:
        if not _is_flow(tp):
            continue
        cons, jac, hess = _flow_scales(tp, x, mult, obj_weight)
        if tp.kind == "constraint":
            cs[tp.row_offset: tp.row_offset + tp.nrec] = np.maximum(cs[tp.row_offset: tp.row_offset + tp.nrec], cons)
        for s, (lo, hi) in enumerate(tp.jac_slices or []):
            js[lo:hi] = jac[s]
        for pr in tp.hess_pairs or []:
            sc = hess.get((pr.i, pr.j))
            if sc is not None:
                hs[pr.start: pr.start + tp.nrec] = sc
    return cs, js, hs


def _stats(gpu, ref, cr, scale):
    gpu, ref = np.asarray(gpu, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    n = int(gpu.size)
    if n == 0:
        return {"n": 0, "strict_violations": 0, "ieee_unequal": 0, "zero_sign_mismatch": 0, "max_rel": 0.0,
                "cond_scaled_max": 0.0, "cr_oracle_unequal": 0, "violations_equal_cr_oracle": True}
    bad = strict_mask(gpu, ref)
    nz = ref != 0.0
    rel = np.zeros(n)
    rel[nz] = np.abs(gpu[nz] - ref[nz]) / np.abs(ref[nz])
    rel[~nz] = np.where(gpu[~nz] == 0.0, 0.0, np.inf)
    dev = np.abs(gpu - ref)
    with np.errstate(divide="ignore", invalid="ignore"):
        sc = np.where(dev == 0.0, 0.0, dev / np.asarray(scale, dtype=np.float64))
    out = {
        "n": n,
        "strict_violations": int(bad.sum()),
        "ieee_unequal": int(np.count_nonzero(~((gpu == ref) | (np.isnan(gpu) & np.isnan(ref))))),
        "zero_sign_mismatch": zero_sign_mismatches(gpu, ref),
        "max_rel": float(rel.max()),
        "cond_scaled_max": float(np.nanmax(sc)),
    }
    if cr is not None:
        cr = np.asarray(cr, dtype=np.float64)
        out["cr_oracle_unequal"] = int(np.count_nonzero(~((gpu == cr) | (np.isnan(gpu) & np.isnan(cr)))))
        out["violations_equal_cr_oracle"] = bool(np.all(gpu[bad] == cr[bad]))
    return out


def report(plan, x, mult, obj_weight, got, ref, cr=None, with_families=True):
    """Per-array and per-family statistics of got = (c, J, H) against
    ref (numpy oracle = reference arithmetic) and cr (CR-trig oracle)."""
    scales = condition_scales(plan, x, mult, obj_weight, ref)
    out = {"arrays": {}, "families": []}
    for i, label in enumerate(("cons", "jac", "hess")):
        out["arrays"][label] = _stats(got[i], ref[i], None if cr is None else cr[i], scales[i])
    if with_families:
        names, cf, jf, hf = families(plan)
        for i, (label, fam) in enumerate((("cons", cf), ("jac", jf), ("hess", hf))):
            for fid, name in enumerate(names):
                sel = np.flatnonzero(fam == fid)
                if sel.size == 0:
                    continue
                st = _stats(got[i][sel], ref[i][sel], None if cr is None else cr[i][sel], scales[i][sel])
                st.update(array=label, family=name)
                out["families"].append(st)
    return out


def scalar_stats(gpu, ref, cr=None):
    return _stats(np.atleast_1d(gpu), np.atleast_1d(ref), None if cr is None else np.atleast_1d(cr),
                  np.abs(np.atleast_1d(ref)))
