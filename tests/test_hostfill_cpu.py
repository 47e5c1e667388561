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


def _mirror_holds(out, runs, exact):
    """Exact layouts: bit for bit.  Relaxed layouts derive the relation from
    the kernel's own expressions, which drop the reference's derivative-space
    ``0 + x`` normalisations: there the oracle (the reference's bits) is held
    to IEEE equality, the kernel's outputs to bits (GPU tests)."""
    for a, n, src, sg in runs:
        want = out[src:src + n] * float(sg)
        got = out[a:a + n]
        nan = np.isnan(want)
        assert np.array_equal(np.isnan(got), nan), f"mirror run at {a}: NaN pattern differs"
        ok = bit_equal(got[~nan], want[~nan]) if exact else np.array_equal(got[~nan], want[~nan])
        assert ok, f"mirror run at {a} (+{n}) != {sg} x run at {src}"


@pytest.mark.parametrize("name", ["case14_polar", "case14_rect", "case5_strg_mp4_polar", "lv10", "augments",
                                  "dupvar", "allops", "syn30_mp6_polar"])
@pytest.mark.parametrize("exact", [False, True])
def test_mirror_runs_hold_in_the_oracle(name, exact):
    """Host mirrors (``HostLayout._host_mirrors``): every run the host path
    writes as sign x another run is that, bit for bit (signs of zero
    included), in the oracle's J / H -- at the start point (flat angles:
    sin 0 = +0 products), perturbed points, and with NaN / inf / negative
    multipliers and weights."""
    model = build(name, data=load(name))
    plan = model.plan
    lay = host_layout(plan, exact_zero_sign=exact)
    rng = np.random.default_rng(11)
    g = load(name)
    cases = [(g["x0"], rng.standard_normal(model.ncon), 1.0),
             (g["x0"] + 0.05 * rng.standard_normal(model.nvar), -np.abs(rng.standard_normal(model.ncon)), -2.0),
             (g["x0"] + 0.1 * rng.standard_normal(model.nvar), np.where(rng.random(model.ncon) < 0.3, np.nan, 1.0),
              np.inf),
             (np.zeros(model.nvar), np.zeros(model.ncon), 0.0)]
    for x, y, w in cases:
        with np.errstate(all="ignore"):
            try:
                _, J, H = O.eval_set(plan, x, y, w)
            except Exception:  # domain error at an all-zero point (log / div models)
                continue
        _mirror_holds(J, lay.mirror_jac, exact)
        _mirror_holds(H, lay.mirror_hess, exact)
    # mirror runs are disjoint from each other and from the constant runs, and
    # their sources are copied (neither constant nor mirrored)
    for mir, fills, total in ((lay.mirror_jac, [lay.fill_jac], plan.n_jac_slots),
                              (lay.mirror_hess, [lay.fill_hess, lay.fill_wzero[:, :2]], plan.n_hess_slots)):
        mark = np.zeros(total, dtype=np.int8)
        for f in fills:
            for a, n in f[:, :2]:
                mark[a:a + n] += 1
        for a, n, _, _ in mir:
            mark[a:a + n] += 1
        assert mark.max(initial=0) <= 1
        for _, n, src, _ in mir:
            assert not mark[src:src + n].any()


def test_case13659_mirrors():
    from paper_2510_12897_b200.workloads import build_workload

    model = build_workload("case13659", lower_to_gpu=False)
    lay = host_layout(model.plan)
    mj = int(lay.mirror_jac[:, 1].sum())
    mh = int(lay.mirror_hess[:, 1].sum())
    # polar flows: dp/dva_t = -dp/dva_f (4 x 20,467 J slots); H (va_f, vm) / (va_t, vm)
    # pairs and the thermal terms' equal diagonal pairs
    assert mj == 4 * 20467
    assert 8 * (mj + mh) > 2.2e6
