"""Per-element parameter columns of batched models (no GPU): the tables
``device._periodic`` stores reproduce every record's field and index value
exactly -- the generated kernels read a record's element at ``r / per``
(complete element runs, MP / scenario models) or through the key index
column (``ix[kcol][r] / per - g0``; N-1, whose branch runs skip the instance
with that branch out), and its instance at ``r % per`` / ``ix[kcol][r] %
per``."""

import numpy as np
import pytest

from fixture_models import build, load
from paper_2510_12897_b200.device import _periodic, host_layout


def _check_model(plan):
    P = getattr(plan, "batch_period", None)
    reduced = 0
    for tp in plan.obj_terms + plan.con_terms:
        red = _periodic(tp, P)
        if red is None:
            continue
        reduced += 1
        n = tp.nrec
        r = np.arange(n, dtype=np.int64)
        if red["kcol"] < 0:
            elem, inst = r // red["per"], r % red["per"]
        else:
            key = np.asarray(tp.table.indices[tp.tape.index_names[red["kcol"]]], dtype=np.int64)
            elem, inst = key // red["per"] - red["g0"], key % red["per"]
        for fi, tab in red["fcols"].items():
            col = np.ascontiguousarray(tp.reals[tp.tape.field_names[fi]], dtype=np.float64)
            assert np.array_equal(tab[elem].view(np.int64), col.view(np.int64))
            assert tab.size < n
        for c, tab in red["icols"].items():
            col = np.asarray(tp.table.indices[tp.tape.index_names[c]], dtype=np.int64)
            assert np.array_equal(tab[elem] + inst, col)
            assert tab.size < n
    return reduced


@pytest.mark.parametrize("name", ["syn30_mp6_polar", "case5_strg_mp4_polar", "case5_strg_mp4_rect"])
def test_mp_fixture_columns_reconstruct(name):
    model = build(name, data=load(name))
    assert model.plan.batch_period > 1
    assert _check_model(model.plan) > 0
    lay = host_layout(model.plan)
    assert any(d.get("per") for d in lay.descs)


def test_n1_keyed_columns_reconstruct():
    from paper_2510_12897_b200.scopf import scopf_model
    from paper_2510_12897_b200.synth import pglib_shaped

    model = scopf_model(pglib_shaped("case1354", seed=1), list(range(12)), lower_to_gpu=False)[0]
    assert _check_model(model.plan) > 0
    lay = host_layout(model.plan)
    # the four flow blocks are keyed on their flow variable column
    assert sum(1 for d in lay.descs if d.get("per") and d["kcol"] >= 0) >= 4


def test_single_instance_models_are_untouched():
    model = build("case14_polar", data=load("case14_polar"))
    assert getattr(model.plan, "batch_period", None) in (None, 0, 1)
    assert not any(d.get("per") for d in host_layout(model.plan).descs)
