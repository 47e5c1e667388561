"""Per-call time of the numpy drop-in set with reused pageable buffers, with
and without in-place page locking (autodiff._HostPins), vs page-locked arrays."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2510_12897_b200 import autodiff, empty_pinned, eval_callback_set  # noqa: E402
from paper_2510_12897_b200._lib import load  # noqa: E402
from paper_2510_12897_b200.workloads import build_workload, eval_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "case13659"
model = build_workload(name, lower_to_gpu=True)
x, y, w = eval_inputs(model, 0)
lib = load()


def run(label, xs, ys, c, J, H, n=200):
    t0 = time.perf_counter()
    eval_callback_set(model, xs, ys, w, c, J, H)
    t1 = time.perf_counter()
    eval_callback_set(model, xs, ys, w, c, J, H)
    t2 = time.perf_counter()
    t = time.perf_counter()
    for _ in range(n):
        eval_callback_set(model, xs, ys, w, c, J, H)
    dt = (time.perf_counter() - t) / n
    print(f"{label:28s} first {1e3*(t1-t0):7.2f} ms  second {1e3*(t2-t1):7.2f} ms  steady {1e6*dt:7.1f} us"
          f"  ({1/dt:7.0f} sets/s)  locked x/J/H {autodiff._PINS.locked(xs)}/{autodiff._PINS.locked(J)}/"
          f"{autodiff._PINS.locked(H)}  last_error {lib.exa_last_error().decode()[:80]!r}", flush=True)


nj, nh = model.plan.n_jac_slots, model.plan.n_hess_slots
autodiff._PINS.enabled = False
run("pageable, no locking", x.copy(), y.copy(), np.empty(model.ncon), np.empty(nj), np.empty(nh))
autodiff._PINS.enabled = True
run("pageable, locked in place", x.copy(), y.copy(), np.empty(model.ncon), np.empty(nj), np.empty(nh))
xp, yp = empty_pinned(model.nvar), empty_pinned(model.ncon)
xp[:], yp[:] = x, y
run("page-locked (empty_pinned)", xp, yp, empty_pinned(model.ncon), empty_pinned(nj), empty_pinned(nh))

# why an array stayed pageable: state of the registry, and a direct attempt
import ctypes as C  # noqa: E402

c, J, H = np.empty(model.ncon), np.empty(nj), np.empty(nh)
xs, ys = x.copy(), y.copy()
for _ in range(3):
    eval_callback_set(model, xs, ys, w, c, J, H)
P = autodiff._PINS
print("spans", len(P._spans), "seen", len(P._seen), "refused", len(P._refused), "bytes", P._bytes)
for lab, a in (("x", xs), ("y", ys), ("c", c), ("J", J), ("H", H)):
    print(lab, hex(a.ctypes.data), a.nbytes, "locked", P.locked(a), "refused", id(a) in P._refused,
          "seen", id(a) in P._seen)
rc = lib.exa_host_register(C.c_void_p(H.ctypes.data), H.nbytes)
print("direct H register rc", rc, lib.exa_last_error().decode())
