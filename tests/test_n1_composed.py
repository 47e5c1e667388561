"""Batched N-1 model vs the oracle COMPOSED FROM THE REFERENCE.

``tests/golden/n1_syn60.npz`` (``tools/make_n1_goldens.py``) holds, for a
60-bus synthetic case with 20 single-branch contingencies, the reference's
own ``opf_model(case_k)`` outputs per instance (branch k out of service,
``opf.py:205``) plus the linking rows ``pg_k - pg_0`` built with the
reference's ``ModelCore`` and the ramp tape of ``opf.py:470-479``, all
evaluated at slices of one evaluation point of the batched model, together
with the committed maps from each instance's variables / rows / raw J and H
slots to the batched model's.

CPU: the batched model's structure covers exactly the composed instances and
its oracle values equal the reference's bit for bit.  GPU: the CUDA set
kernel equals the CR-trig oracle bit for bit and the reference within the
parity comparator.
"""

import numpy as np
import pytest

from fixture_models import GOLDEN
from oracle import crtrig
from oracle import tape_oracle as O
from oracle.parity import bit_equal, ieee_equal, strict_violations

_G = {}


def golden():
    if not _G:
        with np.load(GOLDEN / "n1_syn60.npz") as z:
            _G.update({k: z[k] for k in z.files})
    return _G


def batched_model(lower_to_gpu=False):
    from paper_2510_12897_b200.casearrays import arrays_to_case
    from paper_2510_12897_b200.scopf import scopf_model

    g = golden()
    case = arrays_to_case({k[5:]: v for k, v in g.items() if k.startswith("case_")})
    return scopf_model(case, g["contingencies"].tolist(), lower_to_gpu=lower_to_gpu)[0]


def _instances(g):
    return range(int(g["n_instances"]))


def _check_against_composed(c, J, H, g, cmp):
    for k in _instances(g):
        assert cmp(c[g[f"row_map{k}"]], g[f"cons{k}"]), f"instance {k}: cons"
        assert cmp(J[g[f"jac_map{k}"]], g[f"jac{k}"]), f"instance {k}: jac"
        assert cmp(H[g[f"hess_map{k}"]], g[f"hess{k}"]), f"instance {k}: hess"
    assert cmp(c[g["link_row_map"]], g["link_cons"]), "linking rows: cons"
    assert cmp(J[g["link_jac_map"]], g["link_jac"]), "linking rows: jac"
    assert cmp(H[g["link_hess_map"]], g["link_hess"]), "linking rows: hess"


def test_batched_structure_covers_composed_instances():
    g = golden()
    m = batched_model()
    plan = m.plan
    assert (m.nvar, m.ncon, plan.n_jac_slots, plan.n_hess_slots) == (
        int(g["nvar"]), int(g["ncon"]), int(g["n_jac"]), int(g["n_hess"]))
    S = int(g["n_instances"])
    # every batched row / raw J slot / raw H slot belongs to exactly one
    # instance of the composition (or to the linking model)
    for what, n, key in (("rows", m.ncon, "row_map"), ("jac", plan.n_jac_slots, "jac_map"),
                         ("hess", plan.n_hess_slots, "hess_map")):
        hit = np.zeros(n, dtype=np.int64)
        for k in range(S):
            np.add.at(hit, g[f"{key}{k}"], 1)
        np.add.at(hit, g[f"link_{key}"], 1)
        assert (hit == 1).all(), f"{what}: {np.count_nonzero(hit != 1)} batched entries not covered exactly once"
    # variables: the maps are injective; the batched model additionally keeps
    # the outaged branch's p / q variables of each contingency instance, and
    # those appear in no Jacobian column or Hessian entry
    seen = np.zeros(m.nvar, dtype=np.int64)
    for k in range(S):
        np.add.at(seen, g[f"var_map{k}"], 1)
    assert seen.max() == 1
    extra = np.flatnonzero(seen == 0)
    blocks = {b.name: b for b in m.variables}
    nbr = blocks["p"].size // (2 * S)
    want = []
    for k, b in enumerate(g["contingencies"].tolist(), start=1):
        for name in ("p", "q"):
            for d in (b, nbr + b):
                want.append(blocks[name].offset + d * S + k)
    assert np.array_equal(np.sort(extra), np.sort(np.array(want)))
    assert not np.isin(extra, plan.jac_cols).any()
    assert not np.isin(extra, plan.hess_rows).any() and not np.isin(extra, plan.hess_cols).any()
    # the COO structure itself maps: batched (row, col) of a mapped slot =
    # (row_map[ref row], var_map[ref col]) is implied by bitwise values below;
    # here the instance slices of jac_cols are variables of that instance
    for k in range(S):
        assert np.isin(plan.jac_cols[g[f"jac_map{k}"]], g[f"var_map{k}"]).all()
        assert np.isin(plan.hess_cols[g[f"hess_map{k}"]], g[f"var_map{k}"]).all()


def test_batched_oracle_equals_reference_instances_bitwise():
    g = golden()
    m = batched_model()
    x, y, w = g["x"], g["y"], float(g["w"])
    c, J, H = O.eval_set(m.plan, x, y, w)
    _check_against_composed(c, J, H, g, bit_equal)
    # objective = base-case cost (instance 0), gradient only on its variables
    assert O.eval_objective(m.plan, x) == float(g["obj0"])
    gr = np.empty(m.nvar)
    O.eval_gradient(m.plan, x, gr)
    assert bit_equal(gr[g["var_map0"]], g["grad0"])
    rest = np.ones(m.nvar, dtype=bool)
    rest[g["var_map0"]] = False
    assert (gr[rest] == 0.0).all()


@pytest.mark.gpu
def test_batched_gpu_equals_reference_instances():
    from paper_2510_12897_b200 import eval_callback_set, eval_gradient, eval_objective

    g = golden()
    m = batched_model(lower_to_gpu=True)
    x, y, w = g["x"], g["y"], float(g["w"])
    c, J, H = np.empty(m.ncon), np.empty(m.plan.n_jac_slots), np.empty(m.plan.n_hess_slots)
    eval_callback_set(m, x, y, w, c, J, H)
    O.use_trig(crtrig.TRIG)
    try:
        cr = O.eval_set(m.plan, x, y, w)
    finally:
        O.use_trig(None)
    for a, o in zip((c, J, H), cr):
        assert ieee_equal(a, o)

    def within(a, r):
        bad = strict_violations(a, r)
        return bad.size == 0

    # the composed reference values: every element within 1e-12 (zeros exact)
    _check_against_composed(c, J, H, g, within)
    assert eval_objective(m, x) == float(g["obj0"])
    gr = np.empty(m.nvar)
    eval_gradient(m, x, gr)
    assert bit_equal(gr[g["var_map0"]], g["grad0"])
