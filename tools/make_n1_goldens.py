"""Golden N-1 batch composed from the REFERENCE (SURVEY §8c "N-1 config").

Run in the build container (where /root/reference exists):

    python tools/make_n1_goldens.py

The reference has no N-1 model (``SPEC.md:374``), so the oracle is composed
from its public API exactly as SURVEY §8(c) prescribes:

* instance 0 is ``opf_model(case)``; instance k >= 1 is ``opf_model(case_k)``
  with ``case_k = deepcopy(case)`` and ``branches[cont[k-1]].status = 0``
  (the reference drops inactive branches, ``opf.py:205``);
* the linking rows ``pg_k - pg_0`` are a reference ``ModelCore`` with the
  ramp tape of ``opf.py:470-479`` (``pg["i1"] - pg["i0"]``) over records
  (generator g, instance k >= 1), element-major like the batched model.

Every reference instance is evaluated at its slice of ONE evaluation point of
this repo's batched model (``scopf.scopf_model``): ``x_k = x[var_map_k]``,
``y_k = y[row_map_k]``, objective weight ``w`` for instance 0 and 0 for the
others (the batched objective is the base-case cost).  The maps from the
reference's per-instance indices to the batched model's are committed with
the values:

* ``var_map_k``  reference variable -> batched variable, by block name,
  element and instance; the reference's branch-direction index ``d'`` of the
  reduced branch list maps to the ORIGINAL branch's direction (the batched
  model keeps the outaged branch's p/q variables: they appear in no row,
  J or H slot of that instance, which the test asserts);
* ``row_map_k``, ``jac_map_k``, ``hess_map_k``  reference row / raw J slot /
  raw H slot -> batched one.  Records are matched by the (mapped) variables
  they read, term by term in registration order (both models register the
  same blocks and augments in the same order); rows of a base block follow
  its records.

The test (``tests/test_n1_composed.py``) asserts that the batched model's
outputs at these maps equal the reference's values bit for bit (CPU oracle)
and within the parity comparator (CUDA path), and that the maps are
injective and cover every batched row / slot of the owned instances except
the linking rows (compared against the linking model) and the objective of
the contingency instances (which the batched model does not have).
"""

from __future__ import annotations

import copy
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden" / "n1_syn60.npz"
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import simdnlp as ref  # noqa: E402
from simdnlp import autodiff as rad  # noqa: E402

from make_goldens import ref_case_from_ours  # noqa: E402
from paper_2510_12897_b200 import synth  # noqa: E402
from paper_2510_12897_b200.casearrays import case_to_arrays  # noqa: E402
from paper_2510_12897_b200.scopf import scopf_model  # noqa: E402

CASE_ARGS = dict(n_bus=60, n_gen=12, n_branch=90, seed=13, name="syn60n1")
CONTINGENCIES = list(range(0, 60, 3))  # 20 single-branch outages


def evaluate(model, x, y, w):
    g = np.empty(model.nvar)
    c = np.empty(model.ncon)
    J = np.empty(model.plan.n_jac_slots)
    H = np.empty(model.plan.n_hess_slots)
    f = rad.eval_objective(model, x)
    rad.eval_gradient(model, x, g)
    rad.eval_constraints(model, x, c)
    rad.eval_jacobian(model, x, J)
    rad.eval_hessian(model, x, y, w, H)
    return f, g, c, J, H


def var_maps(ours, rm, k, S, nbr, out_branch):
    """Reference instance-k variable -> batched variable."""
    ob = {blk.name: blk for blk in ours.variables}
    vm = np.full(rm.nvar, -1, dtype=np.int64)
    active = [b for b in range(nbr) if b != out_branch]  # reference's reduced branch list
    nbr_k = len(active)
    for blk in rm.variables:
        n = blk.size
        if blk.name in ("p", "q"):
            orig = np.array([active[d] if d < nbr_k else nbr + active[d - nbr_k] for d in range(n)], dtype=np.int64)
        else:
            orig = np.arange(n, dtype=np.int64)
        vm[blk.offset: blk.offset + n] = ob[blk.name].offset + orig * S + k
    assert (vm >= 0).all()
    return vm


def term_record_map(ref_tp, our_tp, vmap):
    """Reference record -> batched record of the corresponding term, matched
    by the (mapped) variable ids the record reads."""
    if ref_tp.tape.k == 0:
        return None
    keys: dict = {}
    for r, key in enumerate(zip(*[np.asarray(c) for c in our_tp.cols])):
        keys.setdefault(tuple(int(v) for v in key), []).append(r)
    # records reading the same variables (parallel branches' angle-difference
    # rows) are matched in element order, the order both models list them in
    taken: dict = {}
    out = np.empty(ref_tp.nrec, dtype=np.int64)
    for r, key in enumerate(zip(*[vmap[np.asarray(c)] for c in ref_tp.cols])):
        key = tuple(int(v) for v in key)
        j = taken.get(key, 0)
        out[r] = keys[key][j]
        taken[key] = j + 1
    return out


def slot_maps(rm, ours, vmap, with_objective, k=0, S=1):
    """row / raw J / raw H maps of one reference model onto the batched model."""
    rp, op = rm.plan, ours.plan
    row_map = np.full(rm.ncon, -1, dtype=np.int64)
    jac_map = np.full(rp.n_jac_slots, -1, dtype=np.int64)
    hess_map = np.full(rp.n_hess_slots, -1, dtype=np.int64)
    pairs = []
    if with_objective:
        pairs += list(zip(rp.obj_terms, op.obj_terms))
    pairs += list(zip(rp.con_terms, op.con_terms[: len(rp.con_terms)]))
    for rt, ot in pairs:
        assert rt.tape.instr == ot.tape.instr and rt.kind == ot.kind
        rec = term_record_map(rt, ot, vmap)
        if rec is None:
            # k = 0 base block (a balance without shunts reads no variable): its
            # records are (bus, instance) pairs over every bus, element-major
            if rt.kind != "constraint" or ot.nrec != rt.nrec * S:
                continue
            rec = np.arange(rt.nrec, dtype=np.int64) * S + k
        if rt.kind == "constraint":
            row_map[rt.rows] = ot.rows[rec]
        for s, (lo, hi) in enumerate(rt.jac_slices or []):
            olo = ot.jac_slices[s][0]
            jac_map[lo:hi] = olo + rec
        for rpair, opair in zip(rt.hess_pairs, ot.hess_pairs):
            assert (rpair.i, rpair.j) == (opair.i, opair.j)
            hess_map[rpair.start: rpair.start + rt.nrec] = opair.start + rec
    return row_map, jac_map, hess_map


def link_model(ng, S):
    """Linking rows pg_k - pg_0 with the reference's ModelCore and the ramp
    tape of opf.py:470-479 (records (g, k >= 1), element-major)."""
    core = ref.ModelCore()
    pg = core.add_variable((ng, S), name="pg")
    g = np.repeat(np.arange(ng, dtype=np.int64), S - 1)
    k = np.tile(np.arange(1, S, dtype=np.int64), ng)
    core.add_constraint(pg["i1"] - pg["i0"], ref.DataTable({"i0": g * S, "i1": g * S + k}), lb=0.0, ub=0.0)
    return core.compile()


def main():
    case = synth.synthetic_case(**CASE_ARGS)
    rcase = ref_case_from_ours(case)
    ours = scopf_model(case, CONTINGENCIES, lower_to_gpu=False)[0]
    S = len(CONTINGENCIES) + 1
    nbr = len([b for b in case.branches if b.status == 1])
    ng = len([g for g in case.gens if g.status == 1])
    rng = np.random.default_rng(11)
    x = synth.random_interior_point(ours, rng)
    y = rng.uniform(-1.0, 1.0, ours.ncon)
    w = 1.0
    arrays = {f"case_{k}": v for k, v in case_to_arrays(case).items()}
    arrays.update(contingencies=np.array(CONTINGENCIES, dtype=np.int64), x=x, y=y, w=w,
                  nvar=ours.nvar, ncon=ours.ncon, n_jac=ours.plan.n_jac_slots, n_hess=ours.plan.n_hess_slots)
    for k in range(S):
        kcase = copy.deepcopy(rcase)
        out_b = -1 if k == 0 else CONTINGENCIES[k - 1]
        if k:
            kcase.branches[out_b].status = 0
        rm = ref.opf_model(kcase, form="polar")[0]
        vmap = var_maps(ours, rm, k, S, nbr, out_b)
        row_map, jac_map, hess_map = slot_maps(rm, ours, vmap, with_objective=(k == 0), k=k, S=S)
        # rows of the reference model not produced by a base block (none in OPF)
        assert (row_map >= 0).all()
        xk = x[vmap]
        yk = y[row_map]
        f, g, c, J, H = evaluate(rm, xk, yk, w if k == 0 else 0.0)
        keep_h = hess_map >= 0  # objective slots of contingency instances are not in the batch
        arrays.update({f"var_map{k}": vmap, f"row_map{k}": row_map, f"jac_map{k}": jac_map,
                       f"hess_map{k}": hess_map[keep_h], f"obj{k}": f, f"grad{k}": g, f"cons{k}": c,
                       f"jac{k}": J, f"hess{k}": H[keep_h]})
        print(f"instance {k:2d}: out={out_b:3d} nvar={rm.nvar} ncon={rm.ncon} jac={rm.plan.n_jac_slots} "
              f"hess={int(keep_h.sum())}")
    lm = link_model(ng, S)
    pg_off = next(b.offset for b in ours.variables if b.name == "pg")
    xl = x[pg_off: pg_off + ng * S]
    sec = ours.plan.con_terms[-1]
    assert sec.tape.instr == lm.plan.con_terms[0].tape.instr
    vmap_l = pg_off + np.arange(ng * S, dtype=np.int64)
    rec = term_record_map(lm.plan.con_terms[0], sec, vmap_l)
    row_l = sec.rows[rec]
    jac_l = np.concatenate([sec.jac_slices[s][0] + rec for s in range(2)])
    hess_l = np.concatenate([p.start + rec for p in sec.hess_pairs])
    yl = y[row_l]
    f, g, c, J, H = evaluate(lm, xl, yl, 0.0)
    arrays.update(link_var_map=vmap_l, link_row_map=row_l, link_jac_map=jac_l, link_hess_map=hess_l,
                  link_cons=c, link_jac=J, link_hess=H, n_instances=S)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB): batched nvar={ours.nvar} ncon={ours.ncon} "
          f"jac={ours.plan.n_jac_slots} hess={ours.plan.n_hess_slots}")


if __name__ == "__main__":
    main()
