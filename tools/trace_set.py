"""Per-warp timeline of one case13659 set (EXA_TRACE=1 module).

    EXA_TRACE=1 [EXA_PERSIST=0] python tools/trace_set.py case13659 OUT.npz
Runs 40 back-to-back sets on rotating replicas; the trace buffer keeps the
last launch's records (SM, virtual CTA, clock64 and globaltimer start/end).
"""
import ctypes as C
import os
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2510_12897_b200 import _lib, jit
from paper_2510_12897_b200.device import DevicePlan
from paper_2510_12897_b200.workloads import build_workload, eval_inputs

assert jit.TRACE, "set EXA_TRACE=1"
name = sys.argv[1]
out = sys.argv[2]
model = build_workload(name, lower_to_gpu=False)
R = int(os.environ.get("EXA_R", "11"))
dev = torch.device("cuda", 0)
plans = [DevicePlan(model, 0) for _ in range(R)]
lay = plans[0].layout
n_vb = lay.n_ctas[1]
th = lay.threads[1]
tr = torch.zeros(n_vb * (th // 32) * 12, dtype=torch.int64, device=dev)
lib = _lib.load()
bufs = []
for r in range(R):
    x, y, w = eval_inputs(model, r)
    bufs.append([torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev),
                 torch.empty(model.ncon, dtype=torch.float64, device=dev),
                 torch.empty(model.plan.n_jac_slots, dtype=torch.float64, device=dev),
                 torch.empty(model.plan.n_hess_slots, dtype=torch.float64, device=dev)])
st = torch.cuda.Stream(dev)
sh = C.c_void_p(st.cuda_stream)
lib.exa_debug_trace(C.c_void_p(tr.data_ptr()))
with torch.cuda.stream(st):
    for i in range(40):
        b = bufs[i % R]
        rc = lib.exa_eval_set(plans[i % R].handle, None, b[0].data_ptr(), b[1].data_ptr(), 1.0, b[2].data_ptr(),
                              b[3].data_ptr(), b[4].data_ptr(), sh)
        assert rc == 0
torch.cuda.synchronize()
lib.exa_debug_trace(None)
t = tr.cpu().numpy().reshape(-1, 12)
segs = np.array([(tt, kind, cta0, nrec) for (tt, kind, cta0, nrec, rpt) in lay.segs[1]])
np.savez(out, trace=t, segs=segs, persist=jit.PERSIST, threads=th)
print("saved", out, t.shape)
