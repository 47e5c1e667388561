"""The reference's acceptance criterion 1 on the GPU callbacks (B200 only):
central finite differences of the CUDA objective / constraints / Lagrangian
gradient agree with the CUDA gradient, Jacobian and Hessian
(pkg/tests/test_acceptance.py:45-62: grad/jac <= 1e-6, hess <= 1e-5, relative
to max(1, |fd|)).  The FD driver follows simdnlp/derivcheck.py:28-189; only
the GPU callbacks are evaluated, so this checks derivative correctness
independently of the oracle."""

import numpy as np
import pytest

from fixture_models import build, load

pytestmark = pytest.mark.gpu

STEP = 1e-6  # derivcheck.DEFAULT_STEP


def _interior(model, rng):
    """derivcheck.random_interior_point (28-44)."""
    lo, hi = model.lower, model.upper
    u = rng.uniform(-1.0, 1.0, size=model.nvar)
    x = np.empty(model.nvar)
    width = hi - lo
    both = np.isfinite(lo) & np.isfinite(hi)
    x[both] = 0.5 * (lo[both] + hi[both]) + 0.3 * u[both] * width[both]
    loose = ~both
    x[loose] = (model.start + 0.3 * u)[loose]
    return np.clip(x, lo, hi)


def _rel_err(ad, fd):
    if ad.size == 0:
        return 0.0
    return float(np.abs(ad - fd).max()) / max(1.0, float(np.abs(fd).max()))


@pytest.mark.parametrize("name", ["lv10", "case3_polar", "case3_rect", "case5_polar", "case5_rect",
                                  "case14_polar", "case14_rect"])
def test_fd_suite_on_gpu_callbacks(name):
    from paper_2510_12897_b200 import (compress_coordinates, eval_constraints, eval_gradient, eval_hessian,
                                       eval_jacobian, eval_objective, hessian_structure, jacobian_structure)

    model = build(name, lower_to_gpu=True, data=load(name))
    rng = np.random.default_rng(0)
    jp = compress_coordinates(*jacobian_structure(model))
    hp = compress_coordinates(*hessian_structure(model))
    n, m = model.nvar, model.ncon

    def jac_dense(x):
        raw = np.empty(model.plan.n_jac_slots)
        eval_jacobian(model, x, raw)
        D = np.zeros((m, n))
        D[jp.rows, jp.cols] = jp.sum_values(raw)
        return D

    def lag_grad(x, mult):
        g = np.empty(n)
        eval_gradient(model, x, g)
        if m:
            g = g + jac_dense(x).T @ mult
        return g

    for _ in range(2):
        x = _interior(model, rng)
        mult = rng.uniform(-1.0, 1.0, size=m)
        g = np.empty(n)
        eval_gradient(model, x, g)
        fg, fj, fh = np.empty(n), np.zeros((m, n)), np.zeros((n, n))
        cp, cm = np.empty(m), np.empty(m)
        for i in range(n):
            h = STEP * (1.0 + abs(x[i]))
            xp, xm = x.copy(), x.copy()
            xp[i] += h
            xm[i] -= h
            fg[i] = (eval_objective(model, xp) - eval_objective(model, xm)) / (2 * h)
            if m:
                eval_constraints(model, xp, cp)
                eval_constraints(model, xm, cm)
                fj[:, i] = (cp - cm) / (2 * h)
            fh[:, i] = (lag_grad(xp, mult) - lag_grad(xm, mult)) / (2 * h)
        fh = 0.5 * (fh + fh.T)
        raw_h = np.empty(model.plan.n_hess_slots)
        eval_hessian(model, x, mult, 1.0, raw_h)
        H = np.zeros((n, n))
        H[hp.rows, hp.cols] = hp.sum_values(raw_h)
        H = H + H.T - np.diag(np.diag(H))
        assert _rel_err(g, fg) <= 1e-6
        assert _rel_err(jac_dense(x), fj) <= 1e-6
        assert _rel_err(H, fh) <= 1e-5
