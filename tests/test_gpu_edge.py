"""Edge cases on the GPU path (B200): generic (run-time metadata) module for
models with many blocks, serial row sums (> 32 contributions), empty tables,
constant kernels, k = 0 terms, constraint-free models, domain errors."""

import numpy as np
import pytest

from oracle import crtrig
from oracle import tape_oracle as O
from paper_2510_12897_b200 import (DataTable, EvalDomainError, ModelCore, cos, eval_callback_set,
                                   eval_constraints, eval_gradient, eval_hessian, eval_jacobian,
                                   eval_objective, field, sin)
from oracle.parity import ieee_equal

pytestmark = pytest.mark.gpu


def _check_all(model, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.5, 1.5, model.nvar)
    y = rng.uniform(-1, 1, model.ncon)
    O.use_trig(crtrig.TRIG)
    try:
        c0, J0, H0 = O.eval_set(model.plan, x, y, 0.5)
        f0 = O.eval_objective(model.plan, x)
        g0 = np.empty(model.nvar)
        O.eval_gradient(model.plan, x, g0)
    finally:
        O.use_trig(None)
    c = np.empty(model.ncon)
    J = np.empty(model.plan.n_jac_slots)
    H = np.empty(model.plan.n_hess_slots)
    eval_callback_set(model, x, y, 0.5, c, J, H)
    assert ieee_equal(c, c0) and ieee_equal(J, J0) and ieee_equal(H, H0)
    c2 = np.empty(model.ncon)
    if model.ncon:
        eval_constraints(model, x, c2)
        assert ieee_equal(c2, c0)
    J2 = np.empty(model.plan.n_jac_slots)
    eval_jacobian(model, x, J2)
    assert ieee_equal(J2, J0)
    H2 = np.empty(model.plan.n_hess_slots)
    eval_hessian(model, x, y, 0.5, H2)
    assert ieee_equal(H2, H0)
    g = np.empty(model.nvar)
    eval_gradient(model, x, g)
    assert ieee_equal(g, g0)
    assert eval_objective(model, x) == f0


def test_generic_module_many_blocks():
    """> 80 terms: run-time term/segment tables from global memory."""
    core = ModelCore()
    x = core.add_variable(50, lower=0.1, upper=2.0, start=1.0)
    rng = np.random.default_rng(1)
    blocks = []
    for b in range(45):
        n = int(rng.integers(1, 40))
        i = rng.integers(0, 50, n)
        j = rng.integers(0, 50, n)
        blk = core.add_constraint(field("a") * sin(x["i"] - x["j"]) + x["i"] * x["j"],
                                  DataTable({"i": i, "j": j, "a": rng.normal(size=n)}))
        blocks.append(blk)
        core.add_objective(field("c") * x["i"] ** 2, DataTable({"i": i, "c": rng.uniform(size=n)}))
    for blk in blocks[:10]:
        rows = blk.row_offset + rng.integers(0, blk.nrows, 7)
        core.modify_constraint(blk, cos(x["k"]), DataTable({"k": rng.integers(0, 50, 7), "row": rows}))
    model = core.compile()
    assert len(model.plan.obj_terms) + len(model.plan.con_terms) > 80
    assert not model.device_plan.layout.specialised
    _check_all(model)


def test_serial_rows_more_than_32_contributions():
    core = ModelCore()
    x = core.add_variable(200, start=0.5)
    base = core.add_constraint(-field("d"), DataTable({"d": np.arange(5, dtype=float)}))
    # row 2 gets 70 contributions, others a few
    rows = np.concatenate([np.full(70, 2), np.arange(5), np.arange(5)])
    core.modify_constraint(base, x["k"] * x["k"], DataTable({"k": np.arange(rows.size) % 200, "row": rows}))
    model = core.compile()
    lay = model.device_plan.layout
    assert not lay.fold_slots  # serial CSR layout chosen
    _check_all(model)


def test_empty_tables_constant_kernels_and_k0_terms():
    core = ModelCore()
    x = core.add_variable(4, start=0.3)
    core.add_constraint(x["i"] * 2.0, DataTable({"i": np.zeros(0, dtype=np.int64)}))  # empty
    core.add_constraint(-field("c"), DataTable({"c": np.array([1.0, -2.0, 0.0])}))  # k = 0
    core.add_objective(field("w") * 3.0, DataTable({"w": np.array([1.5, 2.5])}))  # k = 0 objective
    blk = core.add_constraint(x["i"] ** 2, DataTable({"i": np.array([0, 1, 2, 3])}))
    core.modify_constraint(blk, -field("e"), DataTable({"e": np.array([0.5, 0.25]), "row": np.array([3, 4])}))
    model = core.compile()
    _check_all(model)


def test_model_without_constraints():
    core = ModelCore()
    x = core.add_variable(6, start=0.7)
    core.add_objective((x["a"] - x["b"]) ** 2 + sin(x["a"]),
                       DataTable({"a": np.arange(5), "b": np.arange(1, 6)}))
    model = core.compile()
    assert model.ncon == 0
    _check_all(model)


def test_domain_error_in_augment_row_sum():
    from paper_2510_12897_b200 import log

    core = ModelCore()
    x = core.add_variable(3, start=1.0)
    base = core.add_constraint(x["i"] * 1.0, DataTable({"i": np.array([0, 1])}))
    core.modify_constraint(base, log(x["k"]), DataTable({"k": np.array([2, 1]), "row": np.array([0, 1])}))
    model = core.compile()
    out = np.empty(model.ncon)
    with pytest.raises(EvalDomainError) as exc:
        eval_constraints(model, np.array([1.0, -1.0, 2.0]), out)
    assert exc.value.op == "log" and exc.value.kind == "augment" and exc.value.record == 1


def _bucket_model(n_rows=40, seed=3):
    """Balance-like block with single-variable augments of two signs: rows
    with 0, 1..8, 9..15 and 16..31 contributions (every width class, half-warp
    and warp rows),
    a base term with a variable (J/H written by the row thread) and
    duplicate variables across a row's augments."""
    core = ModelCore()
    x = core.add_variable(60, start=0.4)
    y = core.add_variable(30, start=0.6)
    rng = np.random.default_rng(seed)
    base = core.add_constraint(-field("d") - field("g") * x["b"] * x["b"],
                               DataTable({"d": rng.normal(size=n_rows), "g": rng.normal(size=n_rows),
                                          "b": rng.integers(0, 60, n_rows)}))
    # 9, 12, 15: three half-warp rows (odd count: the last warp's second half
    # redoes a row); 31: a full warp row
    counts = np.concatenate([[0, 0, 1, 2, 3, 5, 8, 9, 12, 15, 31], rng.integers(0, 9, n_rows - 11)])
    rows = np.repeat(np.arange(n_rows), counts)
    rng.shuffle(rows)
    half = rows.size // 2
    core.modify_constraint(base, x["k"], DataTable({"k": rng.integers(0, 60, half), "row": base.row_offset + rows[:half]}))
    core.modify_constraint(base, -y["m"], DataTable({"m": rng.integers(0, 30, rows.size - half),
                                                    "row": base.row_offset + rows[half:]}))
    return core


def test_row_buckets_all_width_classes():
    core = _bucket_model()
    model = core.compile()
    lay = model.device_plan.layout
    assert lay.buckets, "expected the row-bucket layout"
    widths = {bk["d"] for info in lay.buckets.values() for bk in info["buckets"]}
    assert 32 in widths and 16 in widths and 8 in widths and 0 in widths
    assert [bk["n"] for info in lay.buckets.values() for bk in info["buckets"] if bk["d"] == 16] == [3]
    _check_all(model)
    _check_all(model, seed=5)


def test_row_buckets_fall_back_to_folds():
    """> 31 contributions in a row or > 4 distinct augments: warp folds /
    serial rows, same results."""
    core = ModelCore()
    x = core.add_variable(80, start=0.3)
    base = core.add_constraint(-field("d"), DataTable({"d": np.arange(6, dtype=float)}))
    for a in range(5):  # five distinct augment terms
        core.modify_constraint(base, x["k"] * (1.0 + a), DataTable({"k": np.arange(6) + a, "row": np.arange(6)}))
    model = core.compile()
    assert not model.device_plan.layout.buckets
    _check_all(model)
