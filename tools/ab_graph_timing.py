import sys, json, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch, ctypes as C
import bench
from paper_2510_12897_b200 import _lib
from paper_2510_12897_b200.workloads import build_workload
model = build_workload("case13659", lower_to_gpu=False)
R = 11
plans, bufs = bench.replicas(model, R, 0, seed0=0)
lib = _lib.load()
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
launch = bench.launcher(lib, plans, bufs, st)
out = {}
for n in (512, 704, 512, 704):
    out.setdefault(n, []).append(bench.graph_us(launch, n, st, dev))
# bench-style: 11 graphs of 512, replayed in sequence
S = 512
graphs = []
with torch.cuda.stream(st):
    for g0 in range(R):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(S):
                launch(g0 * S + i)
        graphs.append(g)
        if (g0 + 1) * S % R == 0:
            break
torch.cuda.synchronize()
for rep in range(2):
    with torch.cuda.stream(st):
        for k in range(10):
            graphs[k % len(graphs)].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for k in range(20):
            graphs[k % len(graphs)].replay()
        e1.record(st)
    torch.cuda.synchronize()
    out.setdefault("multi", []).append(e0.elapsed_time(e1) * 1e3 / (20 * S))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for k in range(20):
            graphs[0].replay()
        e1.record(st)
    torch.cuda.synchronize()
    out.setdefault("single", []).append(e0.elapsed_time(e1) * 1e3 / (20 * S))
print(json.dumps({"n_graphs": len(graphs), **{str(k): v for k, v in out.items()}}))
