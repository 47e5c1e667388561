"""The reference's OWN consumers driven by the GPU callbacks (SURVEY §8b
"Callers"; B200 only).

The unmodified reference package (``simdnlp``, installed read-only under the
git-ignored ``baseline/_ref`` -- DESIGN.md §9) is re-pointed at this
package's callbacks exactly the way its CLI re-points ``derivcheck``
(``cli.py:165-181``: module attributes replaced, restored afterwards), then:

* ``derivcheck.check_derivatives`` / ``pattern_covers_fd``
  (``derivcheck.py:158-215``) run on GPU-backed models at acceptance
  criterion 1 / 2's tolerances (``tests/test_acceptance.py:45-76``);
* ``solver.solve`` (``solver.py:298-``, its ``_Scratch`` callbacks
  ``solver.py:249-295``) solves case3 / case5 / case14 to optimality with
  the GPU callbacks, reaching the pure-reference solve's iteration count,
  status and iterates, and -- like ``test_solver.py:111-118`` -- two GPU solves
  give bitwise identical iterates.

Case data come from the committed ingest fixture (the reference's own
``pkg/data`` texts, tests/golden/ingest.npz).
"""

import contextlib
import sys
from pathlib import Path

import numpy as np
import pytest

from test_ingest_cpu import _text, golden

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
NAMES = ("eval_objective", "eval_gradient", "eval_constraints", "eval_jacobian", "eval_hessian",
         "jacobian_structure", "hessian_structure", "compress_coordinates")


def _ref():
    if not (REF / "simdnlp").is_dir():
        pytest.skip("reference package not installed under baseline/_ref (DESIGN.md §9)")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import simdnlp
    import simdnlp.autodiff  # noqa: F401  - submodules the consumers resolve names in
    import simdnlp.derivcheck  # noqa: F401
    import simdnlp.solver  # noqa: F401

    return simdnlp


@contextlib.contextmanager
def gpu_callbacks(ref):
    """cli.py:165-181 pattern: replace the callback names the reference's
    consumers resolve (module attributes), restore on exit."""
    import paper_2510_12897_b200.autodiff as gpu

    mods = [ref.autodiff, ref.solver, ref.derivcheck]
    saved = [(m, n, getattr(m, n)) for m in mods for n in NAMES if hasattr(m, n)]
    try:
        for m, n, _ in saved:
            setattr(m, n, getattr(gpu, n))
        yield
    finally:
        for m, n, f in saved:
            setattr(m, n, f)


def models(ref, case, form="polar"):
    import paper_2510_12897_b200 as ours

    text = _text(golden()[f"text_{case}"])
    rm = ref.opf_model(ref.parse_case(text, name=case), form=form)[0]
    om = ours.opf_model(ours.parse_case(text, name=case), form=form)[0]
    assert np.array_equal(rm.plan.hess_rows, om.plan.hess_rows)
    return rm, om


@pytest.mark.parametrize("case", ["case3", "case5", "case14"])
@pytest.mark.parametrize("form", ["polar", "rect"])
def test_reference_derivcheck_on_gpu_callbacks(case, form):
    ref = _ref()
    _, om = models(ref, case, form)
    with gpu_callbacks(ref):
        rep = ref.derivcheck.check_derivatives(om, points=5, seed=17)
    # acceptance criterion 1 tolerances (test_acceptance.py:57-59, cli.py:31-33)
    assert rep.grad_err <= 1e-6 and rep.jac_err <= 1e-6 and rep.hess_err <= 1e-5, rep


@pytest.mark.parametrize("case", ["case3", "case14"])
def test_reference_pattern_check_on_gpu_callbacks(case):
    ref = _ref()
    _, om = models(ref, case)
    x = ref.derivcheck.random_interior_point(om, np.random.default_rng(23))
    with gpu_callbacks(ref):
        assert ref.derivcheck.pattern_covers_fd(om, x) == (True, 0, True, 0)


@pytest.mark.parametrize("case", ["case3", "case5", "case14"])
def test_reference_solver_on_gpu_callbacks(case):
    ref = _ref()
    rm, om = models(ref, case)
    r_ref = ref.solver.solve(rm)  # the pure reference (numpy callbacks)
    with gpu_callbacks(ref):
        r1 = ref.solver.solve(om)
        r2 = ref.solver.solve(om)
        kkt = ref.solver.kkt_residuals(om, r1)
        cvio = ref.solver.constraint_violation(om, r1.x)
    assert r1.status == "optimal" == r_ref.status
    # test_solver.py:111-118: identical iterates run to run
    assert r1.iterations == r2.iterations
    assert np.array_equal(r1.x, r2.x) and np.array_equal(r1.y, r2.y)
    # the GPU callbacks reproduce the reference's solve: same path, same point
    assert r1.iterations == r_ref.iterations
    np.testing.assert_allclose(r1.x, r_ref.x, rtol=1e-9, atol=1e-12)
    assert abs(r1.objective - r_ref.objective) <= 1e-10 * abs(r_ref.objective)
    # acceptance criterion 3 (test_acceptance.py:79-90)
    assert max(kkt.values()) <= 1e-7 and cvio <= 1e-8
    if case == "case5":  # criterion 5: independent reference objective (pkg/data/case5_reference_objective.txt)
        assert abs(r1.objective - 1.7551890922e04) <= 1e-6 * 1.7551890922e04
