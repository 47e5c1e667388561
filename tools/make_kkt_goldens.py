"""Golden KKT matrices captured from the REFERENCE solver (build container only).

    python tools/make_kkt_goldens.py

Runs ``simdnlp.solve`` (``/root/reference/pkg/src``, read-only) on bundled
cases with ``lapack.dsytrf`` wrapped to record the first KKT matrix it
factors (iteration 1, delta_w = delta_c = 0), and reconstructs that
iteration's inputs with the reference's own helpers (``_push_interior``, the
compressed J/H values from ``_Scratch``, sigma as ``solver.py:421-424``).
Writes ``tests/golden/kkt_<case>.npz``: inputs + the reference's Kt.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_DATA = Path("/root/reference/pkg/data")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
sys.path.insert(0, str(REF_SRC))

import simdnlp as ref  # noqa: E402
from simdnlp import solver as rs  # noqa: E402


def capture(model):
    seen = {}
    orig = rs.lapack.dsytrf

    def rec(K, *a, **kw):
        if "Kt" not in seen:
            seen["Kt"] = np.array(K, copy=True)
        return orig(K, *a, **kw)

    hv, jv = [], []
    orig_h, orig_j = rs._Scratch.hess, rs._Scratch.jac

    def hess(self, x, y):
        v = orig_h(self, x, y)
        hv.append(np.array(v, copy=True))
        return v

    def jac(self, x):
        v = orig_j(self, x)
        jv.append(np.array(v, copy=True))
        return v

    rs.lapack.dsytrf, rs._Scratch.hess, rs._Scratch.jac = rec, hess, jac
    try:
        rs.solve(model, rs.SolverOptions(max_iter=1))
    finally:
        rs.lapack.dsytrf, rs._Scratch.hess, rs._Scratch.jac = orig, orig_h, orig_j
    return seen["Kt"], hv[0], jv[0]


def first_iteration_sigma(model):
    """solver.py:302-324 (initial point) and 379-380, 421-424 (sigma)."""
    nx, m = model.nvar, model.ncon
    zlo = np.concatenate([model.lower, model.con_lower])
    zhi = np.concatenate([model.upper, model.con_upper])
    fixed = zlo == zhi
    has_lo = np.isfinite(zlo) & ~fixed
    has_up = np.isfinite(zhi) & ~fixed
    x = rs._push_interior(model.start, model.lower, model.upper)
    c0 = np.empty(m)
    ref.eval_constraints(model, x, c0)
    s = rs._push_interior(c0, model.con_lower, model.con_upper)
    s[fixed[nx:]] = model.con_lower[fixed[nx:]]
    z = np.concatenate([x, s])
    zl = np.where(has_lo, 1.0, 0.0)
    zu = np.where(has_up, 1.0, 0.0)

    def masked_div(num, den, mask):
        out = np.zeros_like(den)
        out[mask] = num[mask] / den[mask]
        return out

    sigma = masked_div(zl, z - zlo, has_lo) + masked_div(zu, zhi - z, has_up)
    return sigma, fixed


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    for case in ("case3", "case5", "case14"):
        model = ref.opf_model(str(REF_DATA / f"{case}.m"))[0]
        Kt, hvals, jvals = capture(model)
        sigma, fixed = first_iteration_sigma(model)
        jp = ref.compress_coordinates(*ref.jacobian_structure(model))
        hp = ref.compress_coordinates(*ref.hessian_structure(model))
        np.savez_compressed(
            OUT / f"kkt_{case}.npz", nx=model.nvar, m=model.ncon, hrows=hp.rows, hcols=hp.cols, hvals=hvals,
            jrows=jp.rows, jcols=jp.cols, jvals=jvals, sigma=sigma, fixed=fixed, Kt=Kt)
        print(case, Kt.shape, int(fixed.sum()), "fixed")


if __name__ == "__main__":
    main()
