"""Eager (no CUDA graph) callback sets at case13659: host cost per call and
device time per set when the host issues calls back to back, through the C ABI
(ctypes) and through the Python API with torch tensors; vs the graph figure."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_12897_b200 import _lib, eval_callback_set  # noqa: E402
from paper_2510_12897_b200.workloads import build_workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "case13659"
model = build_workload(name, lower_to_gpu=False)
dev = torch.device("cuda", 0)
R = 11
plans, bufs = bench.replicas(model, R, 0, seed0=0)
lib = _lib.load()
st = torch.cuda.Stream(dev)
launch = bench.launcher(lib, plans, bufs, st)
print("graph us/set", round(bench.graph_us(launch, 8 * R, st, dev), 2))
for label, fn in (("C ABI (ctypes)", launch),):
    with torch.cuda.stream(st):
        for i in range(50):
            fn(i)
        torch.cuda.synchronize(dev)
        n = 2000
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        for i in range(n):
            fn(i)
        e1.record(st)
        th = time.perf_counter() - t0
        torch.cuda.synchronize(dev)
    print(f"{label:20s} host {1e6 * th / n:6.2f} us/call  device {1e3 * e0.elapsed_time(e1) / n:6.2f} us/set")
model.device_plan = plans[0]
b = bufs[0]
with torch.cuda.stream(st):
    for _ in range(50):
        eval_callback_set(model, b["x"], b["y"], b["w"], b["c"], b["J"], b["H"])
    torch.cuda.synchronize(dev)
    n = 2000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(n):
        eval_callback_set(model, b["x"], b["y"], b["w"], b["c"], b["J"], b["H"])
    e1.record(st)
    th = time.perf_counter() - t0
    torch.cuda.synchronize(dev)
print(f"{'Python API (torch)':20s} host {1e6 * th / n:6.2f} us/call  device {1e3 * e0.elapsed_time(e1) / n:6.2f} us/set"
      " (one replica: L2-warm)")

# where the Python API's host time goes (cProfile, tottime)
import cProfile  # noqa: E402
import pstats  # noqa: E402

with torch.cuda.stream(st):
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(2000):
        eval_callback_set(model, b["x"], b["y"], b["w"], b["c"], b["J"], b["H"])
    pr.disable()
    torch.cuda.synchronize(dev)
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
