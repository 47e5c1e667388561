"""Host plan vs the reference: model metadata and COO layouts bit-exact (CPU)."""

import json

import numpy as np
import pytest

from fixture_models import NAMES, build, load


@pytest.mark.parametrize("name", NAMES)
def test_model_and_coo_bit_exact(name):
    g = load(name)
    m = build(name, data=g)
    assert m.nvar == int(g["nvar"]) and m.ncon == int(g["ncon"])
    for k in ("lower", "upper", "start", "con_lower", "con_upper"):
        np.testing.assert_array_equal(getattr(m, k), g[k], err_msg=k)
    np.testing.assert_array_equal(m.plan.jac_rows, g["jac_rows"])
    np.testing.assert_array_equal(m.plan.jac_cols, g["jac_cols"])
    np.testing.assert_array_equal(m.plan.hess_rows, g["hess_rows"])
    np.testing.assert_array_equal(m.plan.hess_cols, g["hess_cols"])
    assert m.plan.jac_rows.dtype == np.int64 and m.plan.hess_cols.dtype == np.int64


@pytest.mark.parametrize("name", NAMES)
def test_tapes_match_reference(name):
    g = load(name)
    m = build(name, data=g)
    ref = json.loads(bytes(g["tapes_json"]).decode())
    ours = [[list(i) for i in tp.tape.instr] for tp in m.plan.obj_terms + m.plan.con_terms]
    assert ours == ref
