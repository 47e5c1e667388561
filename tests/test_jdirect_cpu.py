"""Direct compressed-Jacobian entries (no GPU): the term blocks
``HostLayout.jac_direct`` selects write slot s of record r straight to
compressed entry ``jc0 + k r + rank`` -- checked here against
``compress_coordinates``'s own slot map (reference autodiff.py:677-689) and
against the oracle's ``sum_values`` of the raw Jacobian (``0.0 + value`` is
the single-slot fold); the compressed-set module compiles for sm_100a and
exports ``exa_k_setc_h`` / ``exa_k_setc_l``."""

import numpy as np
import pytest

from fixture_models import build, load
from oracle import tape_oracle as O
from paper_2510_12897_b200.autodiff import compress_coordinates
from paper_2510_12897_b200.device import host_layout


def _direct(model):
    plan = model.plan
    lay = host_layout(plan)
    jp = compress_coordinates(plan.jac_rows, plan.jac_cols)
    jdir, mask = lay.jac_direct(jp)
    return lay, jp, jdir, mask


@pytest.mark.parametrize("name", ["case14_polar", "case14_rect", "case5_strg_mp4_polar", "syn30_mp6_polar", "dupvar",
                                  "augments", "lv10"])
def test_direct_entries_match_the_slot_map(name):
    model = build(name, data=load(name))
    lay, jp, jdir, mask = _direct(model)
    g = load(name)
    J = np.empty(model.plan.n_jac_slots)
    O.eval_jacobian(model.plan, g["x0"], J)
    Jc = O.sum_values(jp.slot_map, jp.nnz, J)
    counts = np.bincount(jp.slot_map, minlength=jp.nnz)
    for t, jc0 in jdir.items():
        tp = lay.terms[t]
        k, n = tp.tape.k, tp.nrec
        cols = np.stack([np.asarray(c, dtype=np.int64) for c in tp.cols[:k]])
        rank = (cols[None, :, :] < cols[:, None, :]).sum(axis=1)
        for s in range(k):
            lo = tp.jac_slices[s][0]
            e = jc0 + k * np.arange(n) + rank[s]
            assert np.array_equal(jp.slot_map[lo:lo + n], e)
            assert np.all(counts[e] == 1)
            # what the kernel stores: 0.0 + raw (bit for bit the bincount fold)
            assert np.array_equal((0.0 + J[lo:lo + n]).view(np.int64), Jc[e].view(np.int64))
    # the mask flags exactly the direct blocks' raw slots
    assert int(mask.sum()) == sum(lay.terms[t].tape.k * lay.terms[t].nrec for t in jdir)


def test_polar_opf_direct_blocks():
    """case14 polar: the four flow blocks, both thermal limits and the angle
    differences are direct; the bus balances (augment targets) are not."""
    model = build("case14_polar", data=load("case14_polar"))
    lay, jp, jdir, mask = _direct(model)
    assert len(jdir) >= 4
    for t in jdir:
        assert lay.terms[t].kind == "constraint" and t in lay.group_of
    # no direct slot shares its entry with another slot
    assert np.all(np.bincount(jp.slot_map[mask.astype(bool)], minlength=jp.nnz) <= 1)


def test_compressed_module_compiles():
    from paper_2510_12897_b200.jit import compile_module
    from paper_2510_12897_b200.workloads import build_workload

    model = build_workload("case1354", lower_to_gpu=False)
    lay, jp, jdir, mask = _direct(model)
    assert jdir
    src = lay.compressed_source()
    assert "exa_k_setc_l" in src and "exa_k_setc_h" in src and "A.Jc + " in src
    cubin = compile_module(src)
    assert len(cubin) > 1000


def _model_point(name):
    if name.startswith("case13659"):
        from paper_2510_12897_b200.workloads import build_workload, eval_inputs

        model = build_workload("case13659", lower_to_gpu=False)
        return model, eval_inputs(model, 0)
    g = load(name)
    return build(name, data=g), (g["x0"], g["y0"], float(g["w0"]))


@pytest.mark.parametrize("name", ["syn30_mp6_polar", "case5_strg_mp4_polar", "case13659"])
def test_group_local_hessian_classes(name):
    """``HostLayout.hess_local``: for every valid (class, record) the class's
    slots are exactly the compressed entry's slots other than known +0.0, in
    raw-slot order, and folding the oracle's raw values in that order
    (0.0 + v1 + v2 ...) is the oracle's sum_values bit for bit.  case13659
    (groups of all four flows of a branch) has four-slot classes."""
    model, (x, y, w) = _model_point(name)
    plan = model.plan
    lay = host_layout(plan)
    hp = compress_coordinates(plan.hess_rows, plan.hess_cols)
    hloc, hpos, mask = lay.hess_local(hp)
    assert hloc
    H = np.empty(plan.n_hess_slots)
    O.eval_hessian(plan, x, y, w, H)
    order_ = np.argsort(hp.slot_map, kind="stable")
    ptr = np.zeros(hp.nnz + 1, dtype=np.int64)
    np.cumsum(np.bincount(hp.slot_map, minlength=hp.nnz), out=ptr[1:])
    Hc = O.sum_values(hp.slot_map, hp.nnz, H)
    known = np.zeros(plan.n_hess_slots, dtype=bool)
    for a, n, _ in lay.fill_hess:
        known[a:a + n] = True
    classes = {}
    for gid, ms in hloc.items():
        grp = lay.groups[gid][1]
        for m, pairs in ms.items():
            tp = lay.terms[grp[m]]
            for pair, (c, q, size, off, zero) in pairs.items():
                classes.setdefault(c, {"off": off, "size": size, "zero": zero, "slots": {}})["slots"][q] = (tp, pair)
    if name == "case13659":
        assert max(info["size"] for info in classes.values()) == 4
    for c, info in classes.items():
        order = [info["slots"][q] for q in range(info["size"])]
        n = order[0][0].nrec
        pos = hpos[info["off"]:info["off"] + n]
        for r in np.flatnonzero(pos >= 0)[:200]:
            raws = [tp.hess_start + pair * n + r for tp, pair in order]
            assert raws == sorted(raws)
            e = int(pos[r])
            if info["zero"]:  # the entry holds exactly these known +0.0 slots
                assert {int(t) for t in order_[ptr[e]:ptr[e + 1]]} == set(raws) and all(known[s] for s in raws)
                assert Hc[e] == 0.0 and not np.signbit(Hc[e])
                continue
            own = {int(t) for t in order_[ptr[e]:ptr[e + 1]] if not known[t]}
            assert own == set(raws)
            acc = 0.0
            for s in raws:
                acc = acc + H[s]
            assert np.float64(acc).view(np.int64) == Hc[e].view(np.int64)
            assert all(mask[s] for s in raws)
