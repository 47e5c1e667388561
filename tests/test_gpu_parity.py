"""CUDA callbacks vs the reference goldens and the CPU oracle (B200 only).

Two oracles judge every output:

* the reference itself (committed goldens, numpy + glibc sin/cos) -- strict
  |gpu - ref| <= 1e-12 |ref| per element, exact zeros where ref == 0;
* the oracle restatement with correctly-rounded array sin/cos -- the CUDA path
  must equal it BIT FOR BIT on every fixture whose kernels use only IEEE
  basic ops, sqrt, sin and cos.  Any element that differs from the reference
  beyond 1e-12 must be one where the CR oracle agrees with the GPU, i.e. the
  difference is glibc's own sin/cos misrounding amplified by cancellation.
"""

import numpy as np
import pytest

from fixture_models import INDEX, NAMES, build, load
from oracle import crtrig
from oracle import tape_oracle as O
from oracle.parity import RTOL, bit_equal, ieee_equal, strict_violations, zero_sign_mismatches  # noqa: F401

pytestmark = pytest.mark.gpu

_EXACT_OPS = {"const", "field", "var", "neg", "add", "sub", "mul", "div", "sin", "cos", "sqrt"}


def _exact_fixture(model) -> bool:
    for tp in model.plan.obj_terms + model.plan.con_terms:
        for ins in tp.tape.instr:
            if ins[0] == "ipow" and ins[2] in (-1, 0, 1, 2):
                continue
            if ins[0] not in _EXACT_OPS:
                return False
    return True


def oracle_cr(model, x, y, w):
    O.use_trig(crtrig.TRIG)
    try:
        plan = model.plan
        f = O.eval_objective(plan, x)
        g = np.empty(model.nvar)
        O.eval_gradient(plan, x, g)
        c, J, H = O.eval_set(plan, x, y, w)
        return f, g, c, J, H
    finally:
        O.use_trig(None)


def gpu_all(model, x, y, w):
    from paper_2510_12897_b200 import autodiff as A

    f = A.eval_objective(model, x)
    g = np.empty(model.nvar)
    A.eval_gradient(model, x, g)
    c = np.empty(model.ncon)
    A.eval_constraints(model, x, c)
    J = np.empty(model.plan.n_jac_slots)
    A.eval_jacobian(model, x, J)
    H = np.empty(model.plan.n_hess_slots)
    A.eval_hessian(model, x, y, w, H)
    return f, g, c, J, H


_models: dict = {}


def gpu_model(name):
    if name not in _models:
        _models[name] = (build(name, lower_to_gpu=True), load(name))
    return _models[name]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("point", [0, 1])
def test_callbacks_match_reference(name, point):
    model, g = gpu_model(name)
    x, y, w = g[f"x{point}"], g[f"y{point}"], float(g[f"w{point}"])
    got = gpu_all(model, x, y, w)
    ref = (float(g[f"obj{point}"]), g[f"grad{point}"], g[f"cons{point}"], g[f"jac{point}"], g[f"hess{point}"])
    cr = oracle_cr(model, x, y, w)
    exact = _exact_fixture(model)
    for label, a, r, o in zip(("obj", "grad", "cons", "jac", "hess"), got, ref, cr):
        a, r, o = np.atleast_1d(a), np.atleast_1d(r), np.atleast_1d(o)
        if exact:
            assert ieee_equal(a, o), f"{name}/{label}: GPU differs from CR-trig oracle"
        bad = strict_violations(a, r)
        if exact:
            # every > 1e-12 deviation from the reference is explained by glibc sin/cos rounding
            assert ieee_equal(a[bad], o[bad]), f"{name}/{label}: unexplained deviations {bad[:10]}"
            # recorded: no golden fixture has a strict violation (zero budget)
            assert bad.size == 0, f"{name}/{label}: {bad.size} deviations"
        else:
            assert bad.size == 0, f"{name}/{label}: {bad.size} elements beyond 1e-12: {bad[:10]}"
        if model.device_plan.exact_zero_sign:
            # exact zero-sign mode: the reference's signs of zero too
            assert zero_sign_mismatches(a, r) == 0, f"{name}/{label}: zero signs differ"


@pytest.mark.parametrize("name", ["case14_polar", "syn60_polar", "case5_strg_mp4_polar", "syn30_mp6_polar"])
def test_zero_sign_modes(name):
    """Both code-generation modes, whatever the default: exact = the
    reference's bit patterns (signs of zero; NaN / inf multipliers give NaN
    in the structural-zero slots like weight * 0.0, autodiff.py:652);
    relaxed = IEEE-equal for finite weights, +0.0 structural zeros."""
    from paper_2510_12897_b200 import eval_callback_set
    from paper_2510_12897_b200.device import DevicePlan

    model, g = gpu_model(name)
    x, y, w = g["x0"], g["y0"].copy(), -0.75
    y[::3] = -np.abs(y[::3])
    default = model.device_plan
    try:
        for exact in (True, False):
            model.device_plan = DevicePlan(model, 0, exact_zero_sign=exact)
            for yy, ww in ((y, w), (np.where(np.arange(model.ncon) % 5 == 0, np.nan, y), np.inf)):
                outs = [np.empty(model.ncon), np.empty(model.plan.n_jac_slots), np.empty(model.plan.n_hess_slots)]
                eval_callback_set(model, x, yy, ww, *outs)
                dev = [np.empty_like(o) for o in outs]
                import torch

                d = torch.device("cuda", 0)
                td = [torch.empty(o.size, dtype=torch.float64, device=d) for o in outs]
                eval_callback_set(model, torch.from_numpy(x).to(d), torch.from_numpy(yy).to(d), ww, *td)
                dev = [t.cpu().numpy() for t in td]
                ref = oracle_cr(model, x, yy, ww)[2:]
                for label, a, b, r in zip(("cons", "jac", "hess"), outs, dev, ref):
                    if exact:
                        # host path (weighted zeros filled on the host) and device path
                        assert bit_equal(a, r), f"{name}/{label}: host path not bit-equal (exact mode)"
                        assert bit_equal(b, r), f"{name}/{label}: device path not bit-equal (exact mode)"
                    elif np.isfinite(yy).all() and np.isfinite(ww):
                        assert ieee_equal(a, r) and ieee_equal(b, r)
    finally:
        model.device_plan = default


@pytest.mark.parametrize("name", NAMES)
def test_fused_set_equals_separate_callbacks(name):
    from paper_2510_12897_b200 import autodiff as A

    model, g = gpu_model(name)
    x, y, w = g["x0"], g["y0"], float(g["w0"])
    _, _, c, J, H = gpu_all(model, x, y, w)
    c2 = np.empty_like(c)
    J2 = np.empty_like(J)
    H2 = np.empty_like(H)
    A.eval_callback_set(model, x, y, w, c2, J2, H2)
    assert ieee_equal(c, c2) and ieee_equal(J, J2) and ieee_equal(H, H2)


@pytest.mark.parametrize("name", ["case14_polar", "syn60_polar", "case5_strg_mp4_rect", "lv10"])
def test_zero_copy_torch_path_and_determinism(name):
    import torch

    from paper_2510_12897_b200 import autodiff as A

    model, g = gpu_model(name)
    x, y, w = g["x0"], g["y0"], float(g["w0"])
    f, gr, c, J, H = gpu_all(model, x, y, w)
    dev = torch.device("cuda", 0)
    xt = torch.from_numpy(x).to(dev)
    yt = torch.from_numpy(y).to(dev)
    ct = torch.empty(model.ncon, dtype=torch.float64, device=dev)
    Jt = torch.empty(model.plan.n_jac_slots, dtype=torch.float64, device=dev)
    Ht = torch.empty(model.plan.n_hess_slots, dtype=torch.float64, device=dev)
    gt = torch.empty(model.nvar, dtype=torch.float64, device=dev)
    for _ in range(2):  # run-to-run bitwise determinism
        A.eval_callback_set(model, xt, yt, w, ct, Jt, Ht)
        A.eval_gradient(model, xt, gt)
        assert A.eval_objective(model, xt) == f
        assert ieee_equal(ct.cpu().numpy(), c)
        assert ieee_equal(Jt.cpu().numpy(), J)
        assert ieee_equal(Ht.cpu().numpy(), H)
        assert ieee_equal(gt.cpu().numpy(), gr)


@pytest.mark.parametrize("name", ["case14_polar", "syn60_polar", "syn30_mp6_polar", "case5_strg_mp4_polar"])
def test_compressed_sum_values_on_gpu(name):
    from paper_2510_12897_b200 import autodiff as A

    model, g = gpu_model(name)
    jp = A.compress_coordinates(*A.jacobian_structure(model))
    hp = A.compress_coordinates(*A.hessian_structure(model))
    np.testing.assert_array_equal(jp.rows, g["jc_rows"])
    np.testing.assert_array_equal(hp.cols, g["hc_cols"])
    np.testing.assert_array_equal(hp.slot_map, g["hc_map"])
    assert ieee_equal(jp.sum_values(g["jac0"]), g["jacc0"])
    assert ieee_equal(hp.sum_values(g["hess0"]), g["hessc0"])


def test_device_sincos_is_correctly_rounded_and_matches_host_build():
    import torch

    from paper_2510_12897_b200 import _lib

    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(-0.8, 0.8, 200000), rng.uniform(-50, 50, 50000),
                        [0.0, -0.0, 1e-300, -1e-20, np.pi / 4, 3.0, 1e5, 2e6, np.inf, np.nan]])
    xt = torch.from_numpy(x).cuda()
    s = torch.empty_like(xt)
    c = torch.empty_like(xt)
    _lib.check(_lib.load().exa_device_sincos(xt.data_ptr(), s.data_ptr(), c.data_ptr(), x.size, None))
    torch.cuda.synchronize()
    hs, hc = crtrig.sincos(x)
    # beyond |x| = 2^20 pi/2 both sides fall back to their platform libm
    dd = ~(np.abs(x) > float.fromhex("0x1.921fb54442d18p+20"))
    assert ieee_equal(s.cpu().numpy()[dd], hs[dd]) and ieee_equal(c.cpu().numpy()[dd], hc[dd])
    # vs glibc: only 1-ulp differences, on a small fraction of arguments
    fin = np.isfinite(x) & (np.abs(x) < 1e5)
    ds = s.cpu().numpy()[fin] != np.sin(x[fin])
    assert ds.mean() < 0.005
    ulp = np.abs(np.spacing(np.sin(x[fin])))
    assert np.all(np.abs(s.cpu().numpy()[fin] - np.sin(x[fin])) <= ulp)


def test_domain_error_location_matches_reference():
    from paper_2510_12897_b200 import DataTable, EvalDomainError, ModelCore, eval_objective, log

    core = ModelCore()
    x = core.add_variable(2, start=1.0)
    core.add_objective(log(x["i"]), DataTable({"i": np.array([0, 1])}))
    model = core.compile()
    with pytest.raises(EvalDomainError) as exc:
        eval_objective(model, np.array([1.0, -2.0]))
    err = exc.value
    assert err.op == "log" and err.kind == "objective" and err.record == 1 and err.block_index == 0


def test_domain_error_in_constraint_block_order():
    from paper_2510_12897_b200 import DataTable, EvalDomainError, ModelCore, eval_constraints, field, sqrt

    core = ModelCore()
    x = core.add_variable(3, start=1.0)
    core.add_constraint(x["i"] * 2.0, DataTable({"i": np.array([0, 1, 2])}))
    core.add_constraint(sqrt(x["i"]) + 1.0 / field("d"), DataTable({"i": np.array([0, 1, 2]),
                                                                      "d": np.array([1.0, 2.0, 0.0])}))
    model = core.compile()
    out = np.empty(model.ncon)
    with pytest.raises(EvalDomainError) as exc:
        eval_constraints(model, np.array([1.0, -1.0, -3.0]), out)
    # sqrt (instr 1) fails before div (instr 4) in tape order; first bad record 1
    assert exc.value.op == "sqrt" and exc.value.record == 1 and exc.value.kind == "constraint"
    assert exc.value.block_index == 1


@pytest.mark.parametrize("name", ["case14_polar", "case14_rect", "case5_strg_mp4_polar", "lv10"])
def test_host_buffer_c_abi_matches_oracle(name):
    """exa_eval_set_host (pinned host in/out, copies on the stream) returns the
    CR oracle's bits, across two workspaces on the legacy default stream and a
    side stream (D2H store kernel into the mapped arrays).  The host buffers
    start as NaN: the constant runs written on the host plus the copied
    ranges cover every slot."""
    import ctypes as C

    import torch

    from paper_2510_12897_b200 import _lib

    from paper_2510_12897_b200 import eval_callback_set

    g = load(name)
    model = build(name, lower_to_gpu=True, data=g)
    x, y, w = g["x0"], g["y0"], float(g["w0"])
    _, _, c0, J0, H0 = oracle_cr(model, x, y, w)
    exact = _exact_fixture(model)
    # the device path (torch CUDA buffers): the host path must return its exact bits
    dev = [torch.empty(n, dtype=torch.float64, device="cuda")
           for n in (model.ncon, model.plan.n_jac_slots, model.plan.n_hess_slots)]
    eval_callback_set(model, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), w, *dev)
    dev = [t.cpu().numpy() for t in dev]
    lib = _lib.load()
    dp = model.device_plan
    outs = []
    for k in range(2):
        wsp = C.c_void_p()
        _lib.check(lib.exa_workspace_create(dp.handle, C.byref(wsp)), "workspace")
        st = torch.cuda.Stream() if k else None
        hx = torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
        hy = torch.from_numpy(np.ascontiguousarray(y)).pin_memory()
        hc = torch.full((model.ncon,), float("nan"), dtype=torch.float64).pin_memory()
        hJ = torch.full((model.plan.n_jac_slots,), float("nan"), dtype=torch.float64).pin_memory()
        hH = torch.full((model.plan.n_hess_slots,), float("nan"), dtype=torch.float64).pin_memory()
        _lib.check(lib.exa_eval_set_host(dp.handle, wsp, hx.data_ptr(), hy.data_ptr(), w, hc.data_ptr(),
                                         hJ.data_ptr(), hH.data_ptr(), C.c_void_p(st.cuda_stream if k else 0)),
                   "set_host")
        torch.cuda.synchronize()
        lib.exa_workspace_destroy(wsp)
        outs.append((hc.numpy().copy(), hJ.numpy().copy(), hH.numpy().copy()))
    # the drop-in numpy call (pageable arrays: pinned staging, chunked D2H)
    npo = [np.full(n, np.nan) for n in (model.ncon, model.plan.n_jac_slots, model.plan.n_hess_slots)]
    eval_callback_set(model, np.array(x), np.array(y), w, *npo)
    outs.append(tuple(npo))
    for c, J, H in outs:
        for a, d in zip((c, J, H), dev):
            assert np.array_equal(a.view(np.int64), d.view(np.int64))
        if exact:
            assert ieee_equal(c, c0) and ieee_equal(J, J0) and ieee_equal(H, H0)
        else:
            # vs the reference's own outputs (as test_callbacks_match_reference)
            for a, r in ((c, g["cons0"]), (J, g["jac0"]), (H, g["hess0"])):
                assert strict_violations(a, r).size == 0


def test_strided_batch_equals_single_sets():
    """exa_eval_set_batch: k independent sets in one launch, each bitwise equal
    to its own exa_eval_set."""
    import ctypes as C

    import torch

    from paper_2510_12897_b200 import _lib
    from paper_2510_12897_b200.workloads import build_workload, eval_inputs

    model = build_workload("case1354")
    dp = model.device_plan
    lib = _lib.load()
    S = 3
    dev = torch.device("cuda", dp.device)
    X = torch.stack([torch.from_numpy(eval_inputs(model, k)[0]) for k in range(S)]).to(dev)
    Y = torch.stack([torch.from_numpy(eval_inputs(model, k)[1]) for k in range(S)]).to(dev)
    nj, nh = model.plan.n_jac_slots, model.plan.n_hess_slots
    Cb = torch.empty(S, model.ncon, dtype=torch.float64, device=dev)
    Jb = torch.empty(S, nj, dtype=torch.float64, device=dev)
    Hb = torch.empty(S, nh, dtype=torch.float64, device=dev)
    st = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    from paper_2510_12897_b200 import eval_callback_set_batch

    eval_callback_set_batch(model, X, Y, 0.5, Cb, Jb, Hb)
    for k in range(S):
        c = torch.empty(model.ncon, dtype=torch.float64, device=dev)
        J = torch.empty(nj, dtype=torch.float64, device=dev)
        H = torch.empty(nh, dtype=torch.float64, device=dev)
        _lib.check(lib.exa_eval_set(dp.handle, None, X[k].data_ptr(), Y[k].data_ptr(), 0.5, c.data_ptr(),
                                    J.data_ptr(), H.data_ptr(), st), "set")
        torch.cuda.synchronize()
        assert ieee_equal(Cb[k].cpu().numpy(), c.cpu().numpy())
        assert ieee_equal(Jb[k].cpu().numpy(), J.cpu().numpy())
        assert ieee_equal(Hb[k].cpu().numpy(), H.cpu().numpy())


@pytest.mark.parametrize("name", ["case14_polar", "case5_strg_mp4_polar"])
def test_back_to_back_sets_respect_dependencies(name):
    """Sets launched back to back on one stream with programmatic dependent
    launch (the next grid starts while this one drains): a set whose x is a
    slice of the previous set's Jacobian output (read-after-write) and a set
    that overwrites the previous set's outputs (write-after-write) both
    return exactly what isolated evaluations return."""
    import torch

    from paper_2510_12897_b200 import eval_callback_set

    model, g = gpu_model(name)
    n, m = model.nvar, model.ncon
    nj, nh = model.plan.n_jac_slots, model.plan.n_hess_slots
    x0 = torch.from_numpy(g["x0"]).cuda()
    y0 = torch.from_numpy(g["y0"]).cuda()
    w = float(g["w0"])

    def bufs():
        return [torch.empty(k, dtype=torch.float64, device="cuda") for k in (m, nj, nh)]

    if nj < n:
        pytest.skip("Jacobian shorter than x")
    # reference: isolated evaluations with a host round trip in between
    a = bufs()
    eval_callback_set(model, x0, y0, w, *a)
    torch.cuda.synchronize()
    x1 = (1.0 + 1e-3 * torch.tanh(a[1][:n])).clone()  # bounded, x-dependent
    ref = bufs()
    eval_callback_set(model, x1, y0, w, *ref)
    torch.cuda.synchronize()
    ref = [t.cpu().numpy() for t in ref]
    for _ in range(3):
        # back to back: set 1 writes J; a torch kernel maps it to x; set 2 reads it
        b, c, d = bufs(), bufs(), bufs()
        eval_callback_set(model, x0, y0, w, *b)
        eval_callback_set(model, b[1][:n], y0, w, *d)  # direct read-after-write (next launch)
        xb = 1.0 + 1e-3 * torch.tanh(b[1][:n])
        eval_callback_set(model, xb, y0, w, *c)
        # the direct read-after-write set against an isolated evaluation
        torch.cuda.synchronize()
        e = bufs()
        eval_callback_set(model, b[1][:n].clone(), y0, w, *e)
        torch.cuda.synchronize()
        for got, r in zip(d, e):
            assert np.array_equal(got.cpu().numpy().view(np.int64), r.cpu().numpy().view(np.int64))
        # write-after-write: overwrite c with a different point, then the same again
        eval_callback_set(model, x0, y0, w, *c)
        eval_callback_set(model, xb, y0, w, *c)
        torch.cuda.synchronize()
        for got, r in zip(c, ref):
            assert np.array_equal(got.cpu().numpy().view(np.int64), r.view(np.int64))


@pytest.mark.parametrize("name", ["case14_polar", "case5_strg_mp4_polar"])
def test_numpy_callbacks_with_pinned_arrays(name):
    """The separate numpy callbacks with page-locked arrays (``empty_pinned``:
    direct D2H of the x-dependent ranges, constant runs filled on the host)
    return the bits of the device path; outputs start as NaN."""
    import torch

    from paper_2510_12897_b200 import (empty_pinned, eval_callback_set, eval_constraints, eval_hessian,
                                       eval_jacobian)

    model, g = gpu_model(name)
    x, y, w = g["x0"], g["y0"], float(g["w0"])
    dev = [torch.empty(n, dtype=torch.float64, device="cuda")
           for n in (model.ncon, model.plan.n_jac_slots, model.plan.n_hess_slots)]
    eval_callback_set(model, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), w, *dev)
    ref = [t.cpu().numpy() for t in dev]
    xp, yp = empty_pinned(model.nvar), empty_pinned(model.ncon)
    xp[:], yp[:] = x, y
    out = [empty_pinned(n) for n in (model.ncon, model.plan.n_jac_slots, model.plan.n_hess_slots)]
    for o in out:
        o[:] = np.nan
    eval_constraints(model, xp, out[0])
    eval_jacobian(model, xp, out[1])
    eval_hessian(model, xp, yp, w, out[2])
    for a, r in zip(out, ref):
        assert np.array_equal(a.view(np.int64), r.view(np.int64))


@pytest.mark.parametrize("name", NAMES)
def test_compressed_set_matches_reference_sum_values(name):
    """eval_callback_set_compressed (set kernel + segmented sums on the GPU)
    against the reference's own sum_values of its raw slots (goldens
    jacc / hessc, reference solver.py:282-295) and, bit for bit, against
    compressing this package's raw slots in np.bincount order."""
    import torch

    from paper_2510_12897_b200 import eval_callback_set, eval_callback_set_compressed, model_patterns

    model, g = gpu_model(name)
    x, y, w = g["x0"], g["y0"], float(g["w0"])
    jp, hp = model_patterns(model)
    assert np.array_equal(jp.rows, g["jc_rows"]) and np.array_equal(hp.cols, g["hc_cols"])
    c, Jc, Hc = np.empty(model.ncon), np.empty(jp.nnz), np.empty(hp.nnz)
    eval_callback_set_compressed(model, x, y, w, c, Jc, Hc)
    raw = [np.empty(model.ncon), np.empty(model.plan.n_jac_slots), np.empty(model.plan.n_hess_slots)]
    eval_callback_set(model, x, y, w, *raw)
    assert bit_equal(c, raw[0])
    assert bit_equal(Jc, O.sum_values(jp.slot_map, jp.nnz, raw[1]))
    assert bit_equal(Hc, O.sum_values(hp.slot_map, hp.nnz, raw[2]))
    for got, ref in ((Jc, g["jacc0"]), (Hc, g["hessc0"])):
        bad = strict_violations(got, ref)
        if _exact_fixture(model):
            assert bad.size == 0
        else:
            assert np.allclose(got, ref, rtol=1e-12, atol=0)
    # device tensors: same bits
    d = torch.device("cuda", 0)
    td = [torch.empty(n, dtype=torch.float64, device=d) for n in (model.ncon, jp.nnz, hp.nnz)]
    eval_callback_set_compressed(model, torch.from_numpy(x).to(d), torch.from_numpy(y).to(d), w, *td)
    assert bit_equal(td[1].cpu().numpy(), Jc) and bit_equal(td[2].cpu().numpy(), Hc)
