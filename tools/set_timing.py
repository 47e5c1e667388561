"""Time the fused set kernel for one configuration (env knobs of jit.py).

    EXA_THREADS=128 EXA_MINB=6 python tools/set_timing.py case13659
Prints one JSON line: us per set (graph of rotating replicas), regs.
"""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2510_12897_b200 import _lib, jit
from paper_2510_12897_b200.device import DevicePlan
from paper_2510_12897_b200.workloads import algorithmic_bytes_mode, build_workload, eval_inputs, model_summary

name = sys.argv[1] if len(sys.argv) > 1 else "case13659"
mode = sys.argv[2] if len(sys.argv) > 2 else "set"
# EXA_SHARD=r/N: rank r's shard of an N-way split of a batched config
_shard = os.environ.get("EXA_SHARD")
_r, _n = (int(v) for v in _shard.split("/")) if _shard else (0, 1)
model = build_workload(name, lower_to_gpu=False, rank=_r, world=_n)
bps = model_summary(model)["bytes_per_set"]
mode_bytes = algorithmic_bytes_mode(model, mode)  # this callback's own compulsory bytes
R = int(os.environ.get("EXA_R", "0")) or max(3, int(np.ceil(2 * 126 * 2**20 / mode_bytes)))
dev = torch.device("cuda", 0)
t0 = time.time()
plans = [DevicePlan(model, 0) for _ in range(R)]
if os.environ.get("EXA_ATTACH_CMP") == "1":  # diagnostics: plans with the compressed-set module attached
    for _p in plans:
        _p.compressed_masks()
tjit = time.time() - t0
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


def launch(i):
    b = bufs[i % R]
    p = plans[i % R].handle
    if mode == "set":
        rc = lib.exa_eval_set(p, None, b[0].data_ptr(), b[1].data_ptr(), 1.0, b[2].data_ptr(), b[3].data_ptr(),
                              b[4].data_ptr(), sh)
    elif mode == "cons":
        rc = lib.exa_eval_cons(p, None, b[0].data_ptr(), b[2].data_ptr(), sh)
    elif mode == "jac":
        rc = lib.exa_eval_jac(p, None, b[0].data_ptr(), b[3].data_ptr(), sh)
    else:
        rc = lib.exa_eval_hess(p, None, b[0].data_ptr(), b[1].data_ptr(), 1.0, b[4].data_ptr(), sh)
    assert rc == 0, lib.exa_last_error()


S = 64
with torch.cuda.stream(st):
    for i in range(R):
        launch(i)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for i in range(S * R):
        launch(i)
with torch.cuda.stream(st):
    for _ in range(3):
        g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    e0.record(st)
    for _ in range(5):
        g.replay()
    e1.record(st)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / (5 * S * R)
info = plans[0].info()
print(json.dumps({"workload": name, "mode": mode, "bytes": mode_bytes, "set_bytes": bps, "R": R, "threads": plans[0].layout.threads[1], "minb": jit.MINB_ENV,
                  "sincos": jit.SINCOS_IMPL, "persist": jit.PERSIST, "pdl": jit.PDL, "env": {k: v for k, v in os.environ.items() if k.startswith("EXA_")}, "us_per_set": us, "GBps": mode_bytes / us / 1e3,
                  "regs": info["regs_set_kernel"], "ctas": info["ctas"], "jit_s": tjit}), flush=True)
