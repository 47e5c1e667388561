"""Batched N-1 model (CPU): per-instance agreement with standalone opf_model
instances built from the reference-style API, and instance-shard reassembly."""

import copy

import numpy as np
import pytest

from oracle import tape_oracle as O
from paper_2510_12897_b200 import opf_model, synthetic_case
from paper_2510_12897_b200.scopf import attach_instance_maps, instance_windows, scopf_model
from paper_2510_12897_b200.synth import evaluation_point


def _case():
    return synthetic_case(30, 6, 45, seed=11)


def _instance_view(model, v, k, S):
    """x-vector positions of instance k's variables (block-wise, element-major)."""
    out = {}
    for name in ("va", "vm", "pg", "qg", "p", "q"):
        blk = getattr(v, name)
        n = blk.shape[0]
        out[name] = blk.offset + np.arange(n) * S + k
    return out


@pytest.mark.parametrize("k", [0, 3])
def test_instance_matches_standalone_opf(k):
    case = _case()
    cont = [2, 5, 7, 11, 20]
    gm, gv, gc = scopf_model(case, cont, lower_to_gpu=False)
    S = len(cont) + 1
    x, y, w = evaluation_point(gm, 2)
    c = np.empty(gm.ncon)
    O.eval_constraints(gm.plan, x, c)
    ck = copy.deepcopy(case)
    nbr = len(case.branches)
    keep = np.arange(nbr)
    if k > 0:
        ck.branches[cont[k - 1]].status = 0
        keep = np.delete(keep, cont[k - 1])
    sm, sv, sc = opf_model(ck, lower_to_gpu=False)
    view = _instance_view(gm, gv, k, S)
    xs = np.empty(sm.nvar)
    for name in ("va", "vm", "pg", "qg"):
        blk = getattr(sv, name)
        xs[blk.offset:blk.offset + blk.size] = x[view[name]]
    for name in ("p", "q"):
        blk = getattr(sv, name)
        dirs = np.concatenate([keep, nbr + keep])
        xs[blk.offset:blk.offset + blk.size] = x[view[name][dirs]]
    cs = np.empty(sm.ncon)
    O.eval_constraints(sm.plan, xs, cs)
    # balance rows (bus order) and flow rows (active-branch order) agree bitwise
    for blk_name in ("c_active_power_balance", "c_reactive_power_balance"):
        gb, sb = getattr(gc, blk_name), getattr(sc, blk_name)
        rows_g = gb.row_offset + np.arange(case.n_bus) * S + k
        assert np.all(c[rows_g] == cs[sb.row_offset:sb.row_offset + sb.nrows])
    gb, sb = gc.c_from_active_power_flow, sc.c_from_active_power_flow
    act = np.ones((nbr, S), dtype=bool)
    act[cont, np.arange(1, S)] = False
    recs = np.flatnonzero(act.ravel())  # element-major (branch, instance) records
    inst_rows = gb.row_offset + np.flatnonzero((recs % S) == k)
    assert np.all(c[inst_rows] == cs[sb.row_offset:sb.row_offset + sb.nrows])


@pytest.mark.parametrize("n", [2, 3])
def test_instance_shards_reassemble_bitwise(n):
    case = _case()
    cont = list(range(0, 40, 4))
    gm = scopf_model(case, cont, lower_to_gpu=False)[0]
    S = len(cont) + 1
    x, y, w = evaluation_point(gm, 4)
    gc, gJ, gH = O.eval_set(gm.plan, x, y, w)
    c = np.full(gm.ncon, np.nan)
    J = np.full(gm.plan.n_jac_slots, np.nan)
    H = np.full(gm.plan.n_hess_slots, np.nan)
    f = 0.0
    for r, (c0, c1) in enumerate(instance_windows(S, n)):
        sm = scopf_model(case, cont, owned=(c0, c1), lower_to_gpu=False)[0]
        vm, owned, rm, jm, hm = attach_instance_maps(sm, gm, (c0, c1))
        sc, sJ, sH = O.eval_set(sm.plan, x[vm], y[rm], w)
        assert np.all(np.isnan(c[rm]))
        c[rm], J[jm], H[hm] = sc, sJ, sH
        f += O.eval_objective(sm.plan, x[vm])
    for a, b in ((c, gc), (J, gJ), (H, gH)):
        assert not np.isnan(a).any() and np.all(a == b)
    assert f == O.eval_objective(gm.plan, x)  # base cost lives on one shard only
