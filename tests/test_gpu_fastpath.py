"""The all-device-tensor fast paths of ``eval_callback_set`` and
``eval_callback_set_compressed`` (B200 only): once primed by a first call
through the general path, a repeated call with device tensors goes straight to
the C ABI.  Its outputs must be bitwise the general path's, and anything the
fast path does not take (wrong length, dtype, non-contiguous, numpy) must
still get the general path's conversions and errors."""

import numpy as np
import pytest

from oracle.parity import bit_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def model():
    from paper_2510_12897_b200.workloads import build_workload

    return build_workload("case1354", lower_to_gpu=True)


def _dev(model, k):
    import torch

    from paper_2510_12897_b200.workloads import eval_inputs

    d = torch.device("cuda", model.device_plan.device)
    x, y, w = eval_inputs(model, k)
    return torch.from_numpy(x).to(d), torch.from_numpy(y).to(d), w, d


def test_set_fast_path_bitwise_and_checks(model):
    import torch

    from paper_2510_12897_b200 import eval_callback_set

    x, y, w, d = _dev(model, 1)
    nj, nh = model.plan.n_jac_slots, model.plan.n_hess_slots
    outs = [torch.full((n,), float("nan"), dtype=torch.float64, device=d) for n in (model.ncon, nj, nh)]
    eval_callback_set(model, x, y, w, *outs)  # general path (primes the plan's device object)
    first = [o.cpu().numpy().copy() for o in outs]
    for o in outs:
        o.fill_(float("nan"))
    eval_callback_set(model, x, y, w, *outs)  # fast path
    for a, b in zip(first, outs):
        assert bit_equal(a, b.cpu().numpy())
    # not taken by the fast path: still converted or rejected as before
    eval_callback_set(model, x.to(torch.float32), y, w, *outs)  # converted input
    with pytest.raises(ValueError, match="jacobian buffer has shape"):
        eval_callback_set(model, x, y, w, outs[0], outs[1][:-1], outs[2])
    with pytest.raises(ValueError, match="x has shape"):
        eval_callback_set(model, x[:-1], y, w, *outs)
    c, J, H = np.empty(model.ncon), np.empty(nj), np.empty(nh)
    eval_callback_set(model, x.cpu().numpy(), y.cpu().numpy(), w, c, J, H)  # numpy: host path
    assert bit_equal(J, first[1]) and bit_equal(H, first[2])


def test_compressed_fast_path_bitwise(model):
    import torch

    from paper_2510_12897_b200 import eval_callback_set, eval_callback_set_compressed, model_patterns

    jp, hp = model_patterns(model)
    x, y, w, d = _dev(model, 2)
    outs = [torch.empty(n, dtype=torch.float64, device=d) for n in (model.ncon, jp.nnz, hp.nnz)]
    raw = [torch.empty(n, dtype=torch.float64, device=d)
           for n in (model.ncon, model.plan.n_jac_slots, model.plan.n_hess_slots)]
    eval_callback_set(model, x, y, w, *raw)
    for k in range(3):  # first call general, then fast
        for o in outs:
            o.fill_(float("nan"))
        eval_callback_set_compressed(model, x, y, w, *outs)
        assert bit_equal(outs[0].cpu().numpy(), raw[0].cpu().numpy())
        assert bit_equal(outs[1].cpu().numpy(), jp.sum_values(raw[1]).cpu().numpy())
        assert bit_equal(outs[2].cpu().numpy(), hp.sum_values(raw[2]).cpu().numpy())
    assert model.device_plan.__dict__.get("_cmp_handles") is not None
    with pytest.raises(ValueError, match="compressed hessian buffer has shape"):
        eval_callback_set_compressed(model, x, y, w, outs[0], outs[1], outs[2][:-1])
