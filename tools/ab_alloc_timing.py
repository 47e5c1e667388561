"""A/B of the set's per-launch time under two buffer layouts in ONE process:
(a) x, y, c, J, H per replica (tools/set_timing.py), (b) the same plus the
bench's g, f buffers per replica; plans first in both."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_2510_12897_b200 import _lib
from paper_2510_12897_b200.device import DevicePlan
from paper_2510_12897_b200.workloads import build_workload, eval_inputs

model = build_workload("case13659", lower_to_gpu=False)
R = 11
dev = torch.device("cuda", 0)
lib = _lib.load()
st = torch.cuda.Stream(dev)


def make(extra):
    plans = [DevicePlan(model, 0) for _ in range(R)]
    bufs = []
    for r in range(R):
        x, y, w = eval_inputs(model, r)
        b = {"x": torch.from_numpy(x).to(dev), "y": torch.from_numpy(y).to(dev), "w": w,
             "c": torch.empty(model.ncon, dtype=torch.float64, device=dev),
             "J": torch.empty(model.plan.n_jac_slots, dtype=torch.float64, device=dev),
             "H": torch.empty(model.plan.n_hess_slots, dtype=torch.float64, device=dev)}
        if extra:
            b["g"] = torch.empty(model.nvar, dtype=torch.float64, device=dev)
            b["f"] = torch.empty(1, dtype=torch.float64, device=dev)
        bufs.append(b)
    return plans, bufs


A = make(False)
B = make(True)
out = {"a": [], "b": [], "addr_a": [hex(b["H"].data_ptr()) for b in A[1][:3]],
       "addr_b": [hex(b["H"].data_ptr()) for b in B[1][:3]]}
for _ in range(3):
    out["a"].append(bench.graph_us(bench.launcher(lib, *A, st), 704, st, dev))
    out["b"].append(bench.graph_us(bench.launcher(lib, *B, st), 704, st, dev))
print(json.dumps(out))
