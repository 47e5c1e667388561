"""Host-side device layouts (no GPU): the row-bucket layout of augment-target
blocks reproduces the reference's constraint accumulation order bit for bit
(autodiff.py:573-580), and every module variant compiles for sm_100a."""

import numpy as np

from oracle import tape_oracle as O
from paper_2510_12897_b200 import DataTable, ModelCore, cos, field, sin
from paper_2510_12897_b200.device import BUCKET_GID_BITS, host_layout, precompile
from paper_2510_12897_b200.workloads import build_workload, eval_inputs


def _bucket_cons(model, x):
    """Constraint rows of bucketed blocks, summed from the bucket layout in
    its stated order with the oracle's per-term values."""
    lay = host_layout(model.plan)
    terms = lay.terms
    vals = [np.broadcast_to(O._values(tp, x)[tp.tape.root], (tp.nrec,)) for tp in terms]
    out = {}
    for t, info in lay.buckets.items():
        tp = terms[t]
        # value of augment `sel` as a function of its global variable id
        by_gid = []
        for u in info["augs"]:
            a = terms[u]
            gid = a.slot_blocks[0].offset + np.asarray(a.table.indices[a.tape.slots[0][1]])
            by_gid.append(dict(zip(gid.tolist(), vals[u].tolist())))
        for bk in info["buckets"]:
            W, n = bk["d"], bk["n"]
            rows = lay.i32[bk["rows_off"]:bk["rows_off"] + n]
            pairs = lay.i32[bk["pair_off"]:bk["pair_off"] + 2 * W * n] if W else np.zeros(0, np.int32)
            ent = pairs[0::2].reshape(W, n) if W else np.zeros((0, n), np.int32)
            if W >= 16:  # long rows: (n, W) row-major, lane 0 = base
                ent = pairs[0::2].reshape(n, W).T
            for q in range(n):
                r = int(rows[q])
                acc = 0.0 + float(vals[t][r])
                for k in range(W):
                    e = int(ent[k, q])
                    if e < 0:
                        continue
                    sel, gid = e >> BUCKET_GID_BITS, e & ((1 << BUCKET_GID_BITS) - 1)
                    acc = acc + by_gid[sel][gid]
                out[tp.row_offset + r] = acc
    return out


def test_bucket_layout_reproduces_reference_row_order():
    model = build_workload("case1354", lower_to_gpu=False)
    lay = host_layout(model.plan)
    assert lay.buckets, "balance blocks should use row buckets"
    x, _, _ = eval_inputs(model, 3)
    ref = np.empty(model.ncon)
    O.eval_constraints(model.plan, x, ref)
    got = _bucket_cons(model, x)
    rows = np.array(sorted(got))
    vals = np.array([got[r] for r in rows])
    assert rows.size == sum(lay.terms[t].nrec for t in lay.buckets)
    assert np.array_equal(vals, ref[rows])  # bitwise (== treats -0.0 == 0.0 ...)
    assert np.array_equal(np.signbit(vals), np.signbit(ref[rows]))
    # the fused set kernel writes every augment record's J/H slot exactly once
    for t, info in lay.buckets.items():
        seen = {u: [] for u in info["augs"]}
        for bk in info["buckets"]:
            W, n = bk["d"], bk["n"]
            if not W:
                continue
            pairs = lay.i32[bk["pair_off"]:bk["pair_off"] + 2 * W * n]
            ent, rec = pairs[0::2], pairs[1::2]
            assert np.all(rec[ent < 0] < 0)
            for sel, u in enumerate(info["augs"]):
                r_ = rec[(ent >= 0) & ((ent >> BUCKET_GID_BITS) == sel)]
                seen[u].append(r_[r_ >= 0])
        # records whose J/H a term group writes instead (aligned augments)
        for gi, lst in lay.group_augs.items():
            n_g = lay.terms[lay.groups[gi][1][0]].nrec
            for (u, off, m, s_) in lst:
                if u in seen:
                    seen[u].append(np.arange(off, off + n_g))
                    # the group's slot gathers exactly the augment's variable
                    g_term = lay.terms[lay.groups[gi][1][m]]
                    assert np.array_equal(np.asarray(g_term.cols[s_]), np.asarray(lay.terms[u].cols[0])[off:off + n_g])
        for u, parts in seen.items():
            assert np.array_equal(np.sort(np.concatenate(parts)), np.arange(lay.terms[u].nrec))


def test_generic_module_compiles():
    """> 80 terms -> generic module with run-time metadata (NVRTC, sm_100a)."""
    core = ModelCore()
    x = core.add_variable(20, lower=0.1, upper=2.0, start=1.0)
    rng = np.random.default_rng(0)
    for _ in range(45):
        n = 5
        t = DataTable({"i": rng.integers(0, 20, n), "j": rng.integers(0, 20, n), "a": rng.normal(size=n)})
        core.add_constraint(field("a") * sin(x["i"] - x["j"]), t)
        core.add_objective(x["i"] * x["i"], DataTable({"i": rng.integers(0, 20, n)}))
    blk = core.add_constraint(cos(x["i"]), DataTable({"i": np.arange(4)}))
    core.modify_constraint(blk, x["k"], DataTable({"k": np.arange(4), "row": blk.row_offset + np.arange(4)}))
    model = core.compile(lower_to_gpu=False)
    lay = host_layout(model.plan)
    assert not lay.specialised
    assert precompile(model.plan)[:4] == b"\x7fELF"


def test_bucket_layout_width_classes_and_fallbacks():
    """Host replay of the bucket layout on a model with every width class and
    warp rows; > 4 distinct augments -> no buckets."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_gpu_edge import _bucket_model

    model = _bucket_model().compile(lower_to_gpu=False)
    lay = host_layout(model.plan)
    x = np.random.default_rng(2).uniform(0.2, 1.2, model.nvar)
    ref = np.empty(model.ncon)
    O.eval_constraints(model.plan, x, ref)
    got = _bucket_cons(model, x)
    rows = np.array(sorted(got))
    assert rows.size == model.ncon
    vals = np.array([got[r] for r in rows])
    assert np.array_equal(vals, ref[rows]) and np.array_equal(np.signbit(vals), np.signbit(ref[rows]))
