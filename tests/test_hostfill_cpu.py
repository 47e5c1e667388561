"""Host-path constant runs (no GPU): every raw J / H slot that
``HostLayout._host_fill`` declares constant -- and which ``exa_eval_*_host``
therefore writes on the host instead of copying it from the device -- holds
exactly that value in the oracle's outputs (autodiff.py:588-652 restated in
oracle/tape_oracle.py) at several random points and multipliers.  Structural
Hessian zeros compare IEEE-equal (the zero-sign relaxation writes +0.0)."""

import numpy as np
import pytest

from fixture_models import build, load
from oracle import tape_oracle as O
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
