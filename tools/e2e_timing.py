"""End-to-end host-buffer throughput (exa_eval_set_host, pinned buffers) by
the number of workspaces / streams in flight, interleaved runs on one box so
that host noise hits every variant.

    python tools/e2e_timing.py [workload] [sets per run] [runs]
Prints one JSON line per run and a summary line (medians per stream count).
"""
import ctypes as C
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2510_12897_b200 import _lib
from paper_2510_12897_b200.device import DevicePlan
from paper_2510_12897_b200.workloads import build_workload, eval_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "case13659"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 600
RUNS = int(sys.argv[3]) if len(sys.argv) > 3 else 4
VARIANTS = (1, 2, 3, 4, 6)
model = build_workload(name, lower_to_gpu=False)
p = DevicePlan(model, 0)
lib = _lib.load()
x, y, w = eval_inputs(model, 0)
n = (model.ncon, model.plan.n_jac_slots, model.plan.n_hess_slots)
slots = []
for k in range(max(VARIANTS)):
    ws = C.c_void_p()
    _lib.check(lib.exa_workspace_create(p.handle, C.byref(ws)), "ws")
    slots.append({"st": torch.cuda.Stream(), "x": torch.from_numpy(x).pin_memory(), "y": torch.from_numpy(y).pin_memory(),
                  "o": [torch.empty(m, dtype=torch.float64).pin_memory() for m in n], "ws": ws})


def run(ns, count):
    t0 = time.perf_counter()
    for i in range(count):
        sl = slots[i % ns]
        _lib.check(lib.exa_eval_set_host(p.handle, sl["ws"], sl["x"].data_ptr(), sl["y"].data_ptr(), w,
                                         *(t.data_ptr() for t in sl["o"]), C.c_void_p(sl["st"].cuda_stream)), "set_host")
    for sl in slots[:ns]:
        sl["st"].synchronize()
    return count / (time.perf_counter() - t0)


for ns in VARIANTS:
    run(ns, 3 * ns)
res = {ns: [] for ns in VARIANTS}
for r in range(RUNS):
    for ns in (VARIANTS if r % 2 == 0 else VARIANTS[::-1]):
        v = run(ns, N)
        res[ns].append(v)
        print(json.dumps({"run": r, "streams": ns, "sets_per_s": v}), flush=True)
print(json.dumps({"workload": name, "sets_per_run": N, "median_by_streams": {ns: statistics.median(v) for ns, v in res.items()}}),
      flush=True)
