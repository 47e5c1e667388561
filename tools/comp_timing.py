"""Experiment: set-kernel timing with the OUTPUT buffers (c, J, H) allocated
as compressible memory (cuMemCreate, CU_MEM_ALLOCATION_COMP_GENERIC) vs plain.

    python tools/comp_timing.py [workload] [comp: 0|1]
"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from cuda.bindings import driver as drv

from paper_2510_12897_b200 import _lib
from paper_2510_12897_b200.device import DevicePlan
from paper_2510_12897_b200.workloads import build_workload, eval_inputs, model_summary

name = sys.argv[1] if len(sys.argv) > 1 else "case13659"
comp = int(sys.argv[2]) if len(sys.argv) > 2 else 1
model = build_workload(name, lower_to_gpu=False)
bps = model_summary(model)["bytes_per_set"]
R = max(2, int(np.ceil(2 * 126 * 2**20 / bps)))
dev = torch.device("cuda", 0)
torch.cuda.init()
plans = [DevicePlan(model, 0) for _ in range(R)]


def alloc(nbytes):
    if not comp:
        t = torch.empty(nbytes // 8 + 1, dtype=torch.float64, device=dev)
        keep.append(t)
        return t.data_ptr()
    prop = drv.CUmemAllocationProp()
    prop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = 0
    prop.allocFlags.compressionType = 1  # CU_MEM_ALLOCATION_COMP_GENERIC
    err, gran = drv.cuMemGetAllocationGranularity(prop, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED)
    sz = (nbytes + gran - 1) // gran * gran
    err, h = drv.cuMemCreate(sz, prop, 0)
    assert err == drv.CUresult.CUDA_SUCCESS, err
    err, d = drv.cuMemAddressReserve(sz, 0, 0, 0)
    err, = drv.cuMemMap(d, sz, 0, h, 0)
    acc = drv.CUmemAccessDesc()
    acc.location = prop.location
    acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    err, = drv.cuMemSetAccess(d, sz, [acc], 1)
    return int(d)


keep = []
lib = _lib.load()
bufs = []
for r in range(R):
    x, y, w = eval_inputs(model, r)
    xt, yt = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
    keep += [xt, yt]
    bufs.append((xt.data_ptr(), yt.data_ptr(), alloc(8 * model.ncon), alloc(8 * model.plan.n_jac_slots),
                 alloc(8 * model.plan.n_hess_slots)))
st = torch.cuda.Stream(dev)
sh = C.c_void_p(st.cuda_stream)


def launch(i):
    b = bufs[i % R]
    assert lib.exa_eval_set(plans[i % R].handle, None, b[0], b[1], 1.0, b[2], b[3], b[4], sh) == 0


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
print(json.dumps({"workload": name, "compressible_outputs": comp, "us_per_set": us, "GBps": bps / us / 1e3}))
