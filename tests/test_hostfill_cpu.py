"""Host-path constant runs (no GPU): every raw J / H slot that
``HostLayout._host_fill`` declares constant -- and which ``exa_eval_*_host``
therefore writes on the host instead of copying it from the device -- holds
exactly that value in the oracle's outputs (autodiff.py:588-652 restated in
oracle/tape_oracle.py) at several random points and multipliers.  Relaxed
zero-sign layouts: structural Hessian zeros compare IEEE-equal (+0.0).  Exact
layouts: the weighted-zero runs (weight * z, computed on the host from the
caller's multipliers) equal the oracle bit for bit, signs of zero and NaN
propagation included."""

import numpy as np
import pytest

from fixture_models import build, load
from oracle import tape_oracle as O
from oracle.parity import bit_equal
from paper_2510_12897_b200.device import host_layout


@pytest.mark.parametrize("name", ["case14_polar", "case14_rect", "case5_strg_mp4_polar", "lv10", "augments",
                                  "dupvar", "syn30_mp6_polar"])
def test_constant_runs_hold_in_the_oracle(name):
    model = build(name, data=load(name))
    plan = model.plan
    lay = host_layout(plan)
    rng = np.random.default_rng(3)
    g = load(name)
    for k in range(3):
        x = g["x0"] + (0.0 if k == 0 else 0.05 * rng.standard_normal(model.nvar))
        y = rng.standard_normal(model.ncon) * (1.0 + k)
        w = float(rng.uniform(0.5, 2.0))
        _, J, H = O.eval_set(plan, x, y, w)
        for runs, out in ((lay.fill_jac, J), (lay.fill_hess, H)):
            for a, n, bits in runs:
                v = np.int64(bits).view(np.float64)
                seg = out[a:a + n]
                assert np.all(seg == v), f"{name}: run at {a} (+{n}) is not the constant {v}"
    # runs are sorted, disjoint and inside the raw arrays
    for runs, total in ((lay.fill_jac, plan.n_jac_slots), (lay.fill_hess, plan.n_hess_slots)):
        if len(runs):
            assert np.all(runs[1:, 0] >= runs[:-1, 0] + runs[:-1, 1])
            assert runs[-1, 0] + runs[-1, 1] <= total and runs[0, 0] >= 0


def test_case13659_fill_is_a_third_of_the_outputs():
    from paper_2510_12897_b200.workloads import build_workload

    model = build_workload("case13659", lower_to_gpu=False)
    lay = host_layout(model.plan)
    filled = int(lay.fill_jac[:, 1].sum() + lay.fill_hess[:, 1].sum())
    total = model.plan.n_jac_slots + model.plan.n_hess_slots
    # constant J slots (-1 of the flow definitions, +-1 of the balance augments)
    # and structural-zero H pairs
    assert 0.3 < filled / total < 0.5


@pytest.mark.parametrize("name", ["case14_polar", "case5_strg_mp4_polar", "lv10", "augments", "dupvar",
                                  "syn30_mp6_polar"])
def test_weighted_zero_runs_exact_mode(name):
    model = build(name, data=load(name))
    plan = model.plan
    lay = host_layout(plan, exact_zero_sign=True)
    assert len(lay.fill_hess) == 0  # exact mode: no +0.0 runs
    rng = np.random.default_rng(5)
    g = load(name)
    x = g["x0"]
    for y, w in ((rng.standard_normal(model.ncon), 0.75), (-np.abs(rng.standard_normal(model.ncon)), -1.5),
                 (np.where(rng.random(model.ncon) < 0.3, np.nan, 1.0), np.inf)):
        _, _, H = O.eval_set(plan, x, y, w)
        filled = np.zeros(plan.n_hess_slots, dtype=bool)
        for a, n, off, zbits in lay.fill_wzero:
            z = np.int64(zbits).view(np.float64)
            want = (w * z) * np.ones(n) if off < 0 else y[lay.wz_rows[off:off + n]] * z
            assert bit_equal(H[a:a + n], want), f"{name}: weighted run at {a}"
            assert not filled[a:a + n].any()
            filled[a:a + n] = True
    # every structural zero of the relaxed layout is a weighted run here
    relaxed = host_layout(plan, exact_zero_sign=False)
    n_rel = int(relaxed.fill_hess[:, 1].sum()) if len(relaxed.fill_hess) else 0
    assert int(lay.fill_wzero[:, 1].sum() if len(lay.fill_wzero) else 0) == n_rel
