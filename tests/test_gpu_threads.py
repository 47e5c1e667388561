"""One compiled model shared by several Python threads (B200 only).

Reference contract: ``CompiledModel`` is immutable and safely shareable
across threads; all evaluation state lives in caller buffers
(``core.py:301-305``, ``SPEC.md:129,216``).  Every thread here evaluates the
same model concurrently -- numpy (host path) and torch (device path) buffers,
the fused set, the separate callbacks, objective and gradient -- and each
result must be bitwise the serial result for the same inputs.  A model with
domain-checked operations checks that an ``EvalDomainError`` is reported to
exactly the thread whose input caused it.
"""

import threading

import numpy as np
import pytest

from oracle.parity import bit_equal

pytestmark = pytest.mark.gpu

N_THREADS = 4
ITERS = 12


def _points(model, n):
    from paper_2510_12897_b200.workloads import eval_inputs

    return [eval_inputs(model, 100 + k) for k in range(n)]


def _numpy_eval(model, x, y, w):
    from paper_2510_12897_b200 import (eval_callback_set, eval_constraints, eval_gradient, eval_hessian,
                                       eval_jacobian, eval_objective)

    c, J, H = np.empty(model.ncon), np.empty(model.plan.n_jac_slots), np.empty(model.plan.n_hess_slots)
    eval_callback_set(model, x, y, w, c, J, H)
    c2, J2, H2 = np.empty_like(c), np.empty_like(J), np.empty_like(H)
    eval_constraints(model, x, c2)
    eval_jacobian(model, x, J2)
    eval_hessian(model, x, y, w, H2)
    g = np.empty(model.nvar)
    eval_gradient(model, x, g)
    return c, J, H, c2, J2, H2, g, np.array([eval_objective(model, x)])


def _run_threads(target, n):
    errors = []

    def wrap(k):
        try:
            target(k)
        except BaseException as e:  # noqa: BLE001 - reported to the main thread
            errors.append((k, e))

    ts = [threading.Thread(target=wrap, args=(k,)) for k in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_numpy_callbacks_concurrent_threads_bitwise_serial():
    from paper_2510_12897_b200.workloads import build_workload

    model = build_workload("case1354", lower_to_gpu=True)
    pts = _points(model, N_THREADS)
    serial = [_numpy_eval(model, *p) for p in pts]
    results = [[] for _ in range(N_THREADS)]

    def work(k):
        for it in range(ITERS):
            results[k].append(_numpy_eval(model, *pts[(k + it) % N_THREADS]))

    _run_threads(work, N_THREADS)
    for k in range(N_THREADS):
        for it, got in enumerate(results[k]):
            want = serial[(k + it) % N_THREADS]
            for a, b in zip(got, want):
                assert bit_equal(a, b), (k, it)
    # distinct threads got distinct workspaces
    assert len(model.device_plan._workspaces) >= N_THREADS


def test_torch_callbacks_concurrent_streams_bitwise_serial():
    import torch

    from paper_2510_12897_b200 import eval_callback_set, eval_objective
    from paper_2510_12897_b200.workloads import build_workload

    model = build_workload("case1354", lower_to_gpu=True)
    dev = torch.device("cuda", 0)
    pts = _points(model, N_THREADS)
    serial = [_numpy_eval(model, *p) for p in pts]
    results = [None] * N_THREADS

    def work(k):
        x, y, w = pts[k]
        st = torch.cuda.Stream(dev)
        with torch.cuda.stream(st):
            xt, yt = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
            outs = []
            for _ in range(ITERS):
                c = torch.empty(model.ncon, dtype=torch.float64, device=dev)
                J = torch.empty(model.plan.n_jac_slots, dtype=torch.float64, device=dev)
                H = torch.empty(model.plan.n_hess_slots, dtype=torch.float64, device=dev)
                eval_callback_set(model, xt, yt, w, c, J, H)
                f = eval_objective(model, xt)
                outs.append((c, J, H, f))
            st.synchronize()
            results[k] = [(c.cpu().numpy(), J.cpu().numpy(), H.cpu().numpy(), f) for c, J, H, f in outs]

    _run_threads(work, N_THREADS)
    for k in range(N_THREADS):
        want = serial[k]
        for c, J, H, f in results[k]:
            assert bit_equal(c, want[0]) and bit_equal(J, want[1]) and bit_equal(H, want[2])
            assert f == want[7][0]


def test_domain_errors_reported_to_the_right_thread():
    from paper_2510_12897_b200 import DataTable, EvalDomainError, ModelCore, eval_constraints, eval_objective, log

    core = ModelCore()
    x = core.add_variable(64, lower=-1.0, upper=2.0, start=1.0)
    idx = np.arange(64)
    core.add_objective(log(x["i"]), DataTable({"i": idx}))
    core.add_constraint(log(x["i"]) * x["i"], DataTable({"i": idx}), lb=0.0, ub=1.0)
    model = core.compile(lower_to_gpu=True)
    good = np.linspace(0.5, 1.5, 64)
    bad = good.copy()
    bad[37] = -0.25
    outcome = [[] for _ in range(N_THREADS)]

    def work(k):
        xk = bad if k % 2 else good
        for _ in range(ITERS):
            c = np.empty(model.ncon)
            try:
                eval_constraints(model, xk, c)
                f = eval_objective(model, xk)
                outcome[k].append(("ok", f))
            except EvalDomainError as e:
                outcome[k].append(("err", e.op, e.record, e.kind))

    _run_threads(work, N_THREADS)
    f_good = eval_objective(model, good)
    for k in range(N_THREADS):
        for o in outcome[k]:
            if k % 2:
                assert o == ("err", "log", 37, "constraint"), (k, o)
            else:
                assert o == ("ok", f_good), (k, o)
