"""The CPU oracle reproduces the reference's golden vectors bit-for-bit (CPU).

This pins the oracle before it is used to judge the CUDA path.
"""

import numpy as np
import pytest

from fixture_models import NAMES, build, load
from oracle import tape_oracle as O


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and bool(np.all((a == b) | (np.isnan(a) & np.isnan(b))))


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("point", [0, 1])
def test_oracle_bit_exact(name, point):
    g = load(name)
    m = build(name, data=g)
    plan = m.plan
    x, y, w = g[f"x{point}"], g[f"y{point}"], float(g[f"w{point}"])
    assert O.eval_objective(plan, x) == float(g[f"obj{point}"])
    gr = np.empty(m.nvar)
    O.eval_gradient(plan, x, gr)
    assert _same(gr, g[f"grad{point}"])
    c, J, H = O.eval_set(plan, x, y, w)
    assert _same(c, g[f"cons{point}"])
    assert _same(J, g[f"jac{point}"])
    assert _same(H, g[f"hess{point}"])
    r, cc, smap = O.compress(plan.jac_rows, plan.jac_cols)
    assert _same(r, g["jc_rows"]) and _same(cc, g["jc_cols"]) and _same(smap, g["jc_map"])
    assert _same(O.sum_values(smap, r.size, J), g[f"jacc{point}"])
    r, cc, smap = O.compress(plan.hess_rows, plan.hess_cols)
    assert _same(r, g["hc_rows"]) and _same(cc, g["hc_cols"]) and _same(smap, g["hc_map"])
    assert _same(O.sum_values(smap, r.size, H), g[f"hessc{point}"])
