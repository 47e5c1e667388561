"""Per-call time of the drop-in numpy callbacks (pageable host arrays) at case13659."""
import time, numpy as np, torch
from paper_2510_12897_b200 import workloads, eval_constraints, eval_jacobian, eval_hessian, eval_callback_set
r = workloads.build_workload("case13659")
m = r[0] if isinstance(r, tuple) else r
x, y, w = workloads.eval_inputs(m, 0)[:3]
c, J, H = np.empty(m.ncon), np.empty(m.plan.n_jac_slots), np.empty(m.plan.n_hess_slots)
for name, f in (("cons", lambda: eval_constraints(m, x, c)), ("jac", lambda: eval_jacobian(m, x, J)),
                ("hess", lambda: eval_hessian(m, x, y, 1.0, H)), ("set", lambda: eval_callback_set(m, x, y, 1.0, c, J, H))):
    f(); f()
    t0 = time.perf_counter(); n = 50
    for _ in range(n): f()
    print(name, f"{(time.perf_counter() - t0) / n * 1e6:.0f} us/call (numpy)")

# page-locked arrays (paper_2510_12897_b200.empty_pinned): outputs only, then inputs too
from paper_2510_12897_b200 import empty_pinned

cp_, Jp_, Hp_ = (empty_pinned(n) for n in (m.ncon, m.plan.n_jac_slots, m.plan.n_hess_slots))
xp_, yp_ = empty_pinned(m.nvar), empty_pinned(m.ncon)
xp_[:], yp_[:] = x, y
for name, f in (("set, pinned outputs", lambda: eval_callback_set(m, x, y, 1.0, cp_, Jp_, Hp_)),
                ("set, pinned in+out", lambda: eval_callback_set(m, xp_, yp_, 1.0, cp_, Jp_, Hp_))):
    f(); f()
    t0 = time.perf_counter(); n = 50
    for _ in range(n): f()
    print(name, f"{(time.perf_counter() - t0) / n * 1e6:.0f} us/call")

# a solver's pattern: outputs reused (locked in place on their second use), x / y new every call
c2, J2, H2 = np.empty(m.ncon), np.empty(m.plan.n_jac_slots), np.empty(m.plan.n_hess_slots)
f = lambda: eval_callback_set(m, x.copy(), y.copy(), 1.0, c2, J2, H2)  # noqa: E731
f(); f()
t0 = time.perf_counter(); n = 50
for _ in range(n): f()
print("set, reused outputs, new x / y each call", f"{(time.perf_counter() - t0) / n * 1e6:.0f} us/call")
