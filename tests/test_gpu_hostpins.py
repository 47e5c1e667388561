"""numpy buffers a caller reuses are page-locked in place (B200 only).

A solver allocates its callback buffers once and passes them every iteration
(reference ``solver.py:249-295``, ``_Scratch``).  ``autodiff._HostPins`` locks
such arrays on their second use (``exa_host_register``), so the host path
reads them by DMA and writes them through their device mapping instead of
staging.  The outputs must stay bitwise those of the pageable (staged) path
and of the device path, for arrays, views of a larger owner, the separate
callbacks and the compressed set; a lock must be dropped when its array is
freed, and one-shot arrays must never be locked.
"""

import gc

import numpy as np
import pytest

from oracle.parity import bit_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def model():
    from paper_2510_12897_b200.workloads import build_workload

    return build_workload("case1354", lower_to_gpu=True)


def _pins():
    from paper_2510_12897_b200 import autodiff

    return autodiff._PINS


def _reference(model, x, y, w):
    """The same set through device buffers (no host path at all)."""
    import torch

    from paper_2510_12897_b200 import eval_callback_set

    dev = torch.device("cuda", model.device_plan.device)
    c = torch.empty(model.ncon, dtype=torch.float64, device=dev)
    J = torch.empty(model.plan.n_jac_slots, dtype=torch.float64, device=dev)
    H = torch.empty(model.plan.n_hess_slots, dtype=torch.float64, device=dev)
    eval_callback_set(model, torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev), w, c, J, H)
    return c.cpu().numpy(), J.cpu().numpy(), H.cpu().numpy()


def test_reused_outputs_locked_on_second_use_and_bitwise(model):
    from paper_2510_12897_b200 import eval_callback_set
    from paper_2510_12897_b200.workloads import eval_inputs

    pins = _pins()
    assert pins.enabled
    c, J, H = np.empty(model.ncon), np.empty(model.plan.n_jac_slots), np.empty(model.plan.n_hess_slots)
    assert J.nbytes >= pins.MIN_BYTES and H.nbytes >= pins.MIN_BYTES
    for k in range(4):
        x, y, w = eval_inputs(model, 10 + k)
        c[:], J[:], H[:] = np.nan, np.nan, np.nan
        eval_callback_set(model, x, y, w, c, J, H)
        locked = pins.locked(J) and pins.locked(H)
        assert locked == (k >= 1), f"call {k}: outputs locked={locked}"
        rc, rJ, rH = _reference(model, x, y, w)
        for got, ref, what in ((c, rc, "cons"), (J, rJ, "jac"), (H, rH, "hess")):
            assert bit_equal(got, ref), f"call {k}: {what} differs from the device path"
    n_locked = len(pins._spans)
    del c, J, H, got
    gc.collect()
    assert len(pins._spans) <= n_locked - 2, "freed arrays must drop their page lock"


def test_one_shot_arrays_never_locked(model):
    from paper_2510_12897_b200 import eval_jacobian
    from paper_2510_12897_b200.workloads import eval_inputs

    pins = _pins()
    x, _, _ = eval_inputs(model, 3)
    before = dict(pins._spans)
    for _ in range(3):
        J = np.empty(model.plan.n_jac_slots)  # a fresh array every call
        eval_jacobian(model, x, J)
        assert not pins.locked(J)
        del J
    assert set(pins._spans) <= set(before)


def test_views_and_separate_callbacks_on_a_locked_owner(model):
    from paper_2510_12897_b200 import eval_constraints, eval_hessian, eval_jacobian
    from paper_2510_12897_b200.workloads import eval_inputs

    pins = _pins()
    nc, nj, nh = model.ncon, model.plan.n_jac_slots, model.plan.n_hess_slots
    owner = np.full(1 + nc + nj + nh, np.nan)  # one buffer, callback outputs are views into it
    c, J, H = owner[1:1 + nc], owner[1 + nc:1 + nc + nj], owner[1 + nc + nj:]
    for k in range(3):
        x, y, w = eval_inputs(model, 40 + k)
        owner[:] = np.nan
        eval_constraints(model, x, c)
        eval_jacobian(model, x, J)
        eval_hessian(model, x, y, w, H)
        assert pins.locked(owner)  # the owner's second use is the first iteration's eval_hessian
        rc, rJ, rH = _reference(model, x, y, w)
        assert bit_equal(c, rc) and bit_equal(J, rJ) and bit_equal(H, rH)
        assert np.isnan(owner[0]), "a view's call wrote outside the view"


def test_compressed_set_into_locked_buffers(model):
    from paper_2510_12897_b200 import eval_callback_set, eval_callback_set_compressed, model_patterns
    from paper_2510_12897_b200.workloads import eval_inputs

    pins = _pins()
    jp, hp = model_patterns(model)
    c, Jc, Hc = np.empty(model.ncon), np.empty(jp.nnz), np.empty(hp.nnz)
    cr, J, H = np.empty(model.ncon), np.empty(model.plan.n_jac_slots), np.empty(model.plan.n_hess_slots)
    for k in range(3):
        x, y, w = eval_inputs(model, 70 + k)
        eval_callback_set_compressed(model, x, y, w, c, Jc, Hc)
        eval_callback_set(model, x, y, w, cr, J, H)
        assert pins.locked(Hc) == (Hc.nbytes >= pins.MIN_BYTES and k >= 1)
        assert bit_equal(c, cr)
        assert bit_equal(Jc, jp.sum_values(J)) and bit_equal(Hc, hp.sum_values(H))


def test_disabled_by_environment(monkeypatch, model):
    from paper_2510_12897_b200 import autodiff, eval_jacobian
    from paper_2510_12897_b200.workloads import eval_inputs

    monkeypatch.setattr(autodiff._PINS, "enabled", False)
    x, _, _ = eval_inputs(model, 5)
    J = np.empty(model.plan.n_jac_slots)
    for _ in range(3):
        eval_jacobian(model, x, J)
    assert not autodiff._PINS.locked(J)
