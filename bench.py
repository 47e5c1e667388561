#!/usr/bin/env python
"""Benchmark: AC-OPF callback sets/s (cons + jac + hess) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload case13659]
    python bench.py --impl reference ...     # CPU reference arm (oracle port)

One *step* = ``--sets-per-step`` (default 64) callback sets, each a full
``eval_constraints + eval_jacobian + eval_hessian`` of the workload at its own
evaluation point, executed as ONE fused kernel launch per set.  Steps are
replayed from a CUDA graph.  L2 (126 MB) is defeated by rotating over R
replicas of the whole working set (plan parameters + x + y + outputs) whose
total exceeds 2x the L2 size.  N > 1 (torchrun): for the single-instance
configs (default case13659) every rank evaluates its own scenario stream (weak
scaling, no data-path collective); for the batched configs
(``--workload mp96_case1354`` / ``n1_case2000``) each rank evaluates its
period / instance shard of ONE instance (strong scaling; cons/jac/hess need
no collective).  Time = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

L2_BYTES = 126 * 2**20
METRIC = "AC-OPF callback sets/sec (cons+jac+hess) at 13659-bus; % of HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="case13659")
    ap.add_argument("--sets-per-step", type=int, default=64)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def profiled_traffic(workload):
    """dram bytes per launch of the set kernel from the committed ncu summary."""
    for p in sorted((ROOT / "profiles").glob("*ncu_summary*.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
        except Exception:
            continue
        if d.get("workload") == workload and d.get("dram_bytes_per_launch"):
            return float(d["dram_bytes_per_launch"]), p.name
    return None, None


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for _, _, flags in rows:
            for n, f in zip(names[1:], flags[1:]):
                if f.lower() in ("active", "1", "yes"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows)}


def dist_setup():
    import torch

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return ws, rank, local


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(model, x, y, w, seconds, workload):
    """Oracle port (numpy restatement of the reference) on 1 host core."""
    import numpy as np

    from oracle import tape_oracle as O

    os.environ.setdefault("OMP_NUM_THREADS", "1")
    O.eval_set(model.plan, x, y, w)  # warm
    n = 0
    t0 = time.perf_counter()
    while True:
        O.eval_set(model.plan, x, y, w)
        n += 1
        if time.perf_counter() - t0 >= seconds or n >= 400:
            break
    dt = time.perf_counter() - t0
    del np
    return {"value": n / dt, "unit": "sets/s", "cores": 1, "kind": "port", "cpu_model": _cpu_model(),
            "os_cpu_count": os.cpu_count(),
            "sample": f"{n} sets of {workload} cons+jac+hess (numpy oracle, single thread, {dt:.1f} s)"}


def run_reference(args):
    """--impl reference: the oracle port on all host cores (one process per core)."""
    import multiprocessing as mp

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2510_12897_b200.workloads import build_workload, eval_inputs

    model = build_workload(args.workload, lower_to_gpu=False)
    x, y, w = eval_inputs(model, 0)
    cores = os.cpu_count() or 1
    global _REF
    _REF = (model, x, y, w)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_ref_init) as pool:
        for _ in range(max(args.warmup, 1)):
            pool.map(_ref_one, range(cores))
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_ref_one, range(cores))
        dt = time.perf_counter() - t0
    sets = args.steps * cores
    value = sets / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "sets/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.workload.startswith(("mp", "n1", "scen")) else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.workload, "sets_per_step": cores},
        "cpu_baseline": {"value": value, "unit": "sets/s", "cores": cores, "kind": "port", "cpu_model": _cpu_model(),
                         "sample": f"{sets} sets ({cores} processes x {args.steps} steps) of "
                                   f"{args.workload} cons+jac+hess, numpy restatement of the reference"},
        "e2e": {"value": value, "unit": "sets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


_REF = None


def _ref_init():
    os.environ["OMP_NUM_THREADS"] = "1"


def _ref_one(_):
    from oracle import tape_oracle as O

    model, x, y, w = _REF
    O.eval_set(model.plan, x, y, w)
    return 0


def info_batchable(dp) -> bool:
    return bool(dp.layout.specialised) and not dp.has_checks


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import ctypes as C

    import numpy as np
    import torch

    from paper_2510_12897_b200 import _lib
    from paper_2510_12897_b200.device import DevicePlan
    from paper_2510_12897_b200.workloads import build_workload, eval_inputs, model_summary

    ws, rank, local = dist_setup()
    dev = torch.device("cuda", local)
    sharded = args.workload.startswith(("mp", "n1", "scen"))
    # batched configs: this rank's shard of ONE instance (strong scaling);
    # single-instance configs: every rank evaluates its own sets (weak scaling)
    model = build_workload(args.workload, lower_to_gpu=False, rank=rank, world=ws if sharded else 1)
    summ = model_summary(model)
    bps = summ["bytes_per_set"]
    R = max(2, int(np.ceil(2 * L2_BYTES / bps)))
    R = min(R, 64)
    lib = _lib.load()
    plans, bufs = [], []
    for r in range(R):
        dp = DevicePlan(model, local)
        x, y, w = eval_inputs(model, seed=1000 * rank + r)
        bufs.append({
            "x": torch.from_numpy(x).to(dev), "y": torch.from_numpy(y).to(dev), "w": w,
            "c": torch.empty(model.ncon, dtype=torch.float64, device=dev),
            "J": torch.empty(model.plan.n_jac_slots, dtype=torch.float64, device=dev),
            "H": torch.empty(model.plan.n_hess_slots, dtype=torch.float64, device=dev),
        })
        plans.append(dp)
    stream = torch.cuda.Stream(dev)
    sh = C.c_void_p(stream.cuda_stream)

    def launch(i):
        b = bufs[i % R]
        rc = lib.exa_eval_set(plans[i % R].handle, None, b["x"].data_ptr(), b["y"].data_ptr(), b["w"],
                              b["c"].data_ptr(), b["J"].data_ptr(), b["H"].data_ptr(), sh)
        if rc:
            raise RuntimeError(lib.exa_last_error().decode())

    S = args.sets_per_step
    # one CUDA graph = one step of S sets (rotating replicas); rotation phase kept across steps
    graphs = []
    with torch.cuda.stream(stream):
        for ph in range(R):
            launch(ph)  # eager warm
        torch.cuda.synchronize(dev)
        for g0 in range(R):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for i in range(S):
                    launch(g0 * S + i)
            graphs.append(g)
            if (g0 + 1) * S % R == 0:
                break
    n_graphs = len(graphs)

    def step(k):
        graphs[k % n_graphs].replay()

    with torch.cuda.stream(stream):
        for k in range(args.warmup):
            step(k)
    torch.cuda.synchronize(dev)

    # parity spot check of replica 0 against the bitwise-equal numpy API path
    ref_c = np.empty(model.ncon)
    b0 = bufs[0]
    with torch.cuda.stream(stream):
        launch(0)
    torch.cuda.synchronize(dev)
    ref_c[:] = b0["c"].cpu().numpy()
    assert np.isfinite(ref_c).all()

    sampler = ClockSampler(local)
    with sampler:
        # keep the device busy around the timed region so clocks are sampled under load
        t_soak = time.perf_counter()
        with torch.cuda.stream(stream):
            k = 0
            while time.perf_counter() - t_soak < 0.4:
                step(k)
                k += 1
                if k % 8 == 0:
                    torch.cuda.synchronize(dev)
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for k in range(args.steps):
                step(k)
            e1.record(stream)
        torch.cuda.synchronize(dev)
        if ws > 1:
            torch.distributed.barrier()
        with torch.cuda.stream(stream):
            t_soak = time.perf_counter()
            k = 0
            while time.perf_counter() - t_soak < 0.3:
                step(k)
                k += 1
                if k % 8 == 0:
                    torch.cuda.synchronize(dev)
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    n_sets = args.steps * S * (1 if sharded else ws)
    value = n_sets / (ms / 1e3)
    per_launch_s = (ms / 1e3) / (args.steps * S)
    achieved = bps / per_launch_s / 1e9
    peak, peak_src = peaks()
    traffic, traffic_src = profiled_traffic(args.workload)

    # ---- extra (not the headline): NB independent sets per launch
    # (exa_eval_set_batch), for throughput on independent evaluation points
    batched = None
    if not sharded and ws == 1 and info_batchable(plans[0]):
        NB = 8
        RB = max(2, int(np.ceil(2 * L2_BYTES / (NB * bps))))
        bb = []
        for r in range(RB):
            X = torch.stack([torch.from_numpy(eval_inputs(model, 100 + r * NB + k)[0]) for k in range(NB)]).to(dev)
            Y = torch.stack([torch.from_numpy(eval_inputs(model, 100 + r * NB + k)[1]) for k in range(NB)]).to(dev)
            bb.append((DevicePlan(model, local, group_max=2), X, Y,
                       torch.empty(NB, model.ncon, dtype=torch.float64, device=dev),
                       torch.empty(NB, model.plan.n_jac_slots, dtype=torch.float64, device=dev),
                       torch.empty(NB, model.plan.n_hess_slots, dtype=torch.float64, device=dev)))

        def launch_b(i):
            dp_, X, Y, Cb, Jb, Hb = bb[i % RB]
            rc = lib.exa_eval_set_batch(dp_.handle, None, NB, X.data_ptr(), Y.data_ptr(), 1.0, Cb.data_ptr(),
                                        Jb.data_ptr(), Hb.data_ptr(), sh)
            if rc:
                raise RuntimeError(lib.exa_last_error().decode())

        with torch.cuda.stream(stream):
            for i in range(RB):
                launch_b(i)
            gb = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gb, stream=stream):
                for i in range(4 * RB):
                    launch_b(i)
            gb.replay()
        torch.cuda.synchronize(dev)
        eb0, eb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            eb0.record(stream)
            for _ in range(5):
                gb.replay()
            eb1.record(stream)
        torch.cuda.synchronize(dev)
        sb = 5 * 4 * RB * NB / (eb0.elapsed_time(eb1) / 1e3)
        batched = {"sets_per_launch": NB, "value": sb, "unit": "sets/s",
                   "roofline_frac": sb * bps / 1e9 / peaks()[0],
                   "note": "extra, not the headline: independent evaluation points per launch"}
        del bb

    # ---- end to end: host buffers through the C ABI, copies inside the timed region.
    # exa_eval_set_host = H2D(x, y) + set kernel + D2H(c, J, H) on one stream;
    # NS slots (workspace + stream + pinned host buffers) in round robin, so set
    # i+1's copies overlap set i's (PCIe is full duplex).  Every step copies its
    # inputs in and its full result out inside the timed region.
    NS = 3
    xh, yh = eval_inputs(model, 7)[:2]
    slots = []
    for k in range(NS):
        wsp = C.c_void_p()
        _lib.check(lib.exa_workspace_create(plans[0].handle, C.byref(wsp)), "workspace")
        slots.append({
            "ws": wsp, "st": torch.cuda.Stream(dev),
            "x": torch.from_numpy(xh).pin_memory(), "y": torch.from_numpy(yh).pin_memory(),
            "c": torch.empty(model.ncon, dtype=torch.float64).pin_memory(),
            "J": torch.empty(model.plan.n_jac_slots, dtype=torch.float64).pin_memory(),
            "H": torch.empty(model.plan.n_hess_slots, dtype=torch.float64).pin_memory(),
        })

    def e2e_issue(i):
        sl = slots[i % NS]
        rc = lib.exa_eval_set_host(plans[0].handle, sl["ws"], sl["x"].data_ptr(), sl["y"].data_ptr(), 1.0,
                                   sl["c"].data_ptr(), sl["J"].data_ptr(), sl["H"].data_ptr(),
                                   C.c_void_p(sl["st"].cuda_stream))
        if rc:
            raise RuntimeError(lib.exa_last_error().decode())

    def e2e_sync():
        for sl in slots:
            sl["st"].synchronize()

    for i in range(2 * NS):
        e2e_issue(i)
    e2e_sync()
    # the pipelined host path returns the same bits as the device path
    assert np.array_equal(slots[0]["c"].numpy(), slots[1]["c"].numpy())
    n_e2e = max(1, args.e2e_steps) * 8 * NS
    if ws > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for i in range(n_e2e):
        e2e_issue(i)
    e2e_sync()
    e2e_dt = time.perf_counter() - t0
    # the drop-in Python call with numpy arrays (pageable host memory)
    from paper_2510_12897_b200 import eval_callback_set

    model.device_plan = plans[0]
    xn, yn = xh.copy(), yh.copy()
    cn, Jn, Hn = np.empty(model.ncon), np.empty(model.plan.n_jac_slots), np.empty(model.plan.n_hess_slots)
    eval_callback_set(model, xn, yn, 1.0, cn, Jn, Hn)
    t0 = time.perf_counter()
    n_np = max(4, n_e2e // (2 * NS))
    for _ in range(n_np):
        eval_callback_set(model, xn, yn, 1.0, cn, Jn, Hn)
    e2e_numpy = n_np / (time.perf_counter() - t0)
    # ... with the outputs in page-locked arrays (paper_2510_12897_b200.empty_pinned)
    from paper_2510_12897_b200 import empty_pinned

    cp_, Jp_, Hp_ = (empty_pinned(n) for n in (model.ncon, model.plan.n_jac_slots, model.plan.n_hess_slots))
    xp_, yp_ = empty_pinned(model.nvar), empty_pinned(model.ncon)
    xp_[:], yp_[:] = xn, yn
    eval_callback_set(model, xp_, yp_, 1.0, cp_, Jp_, Hp_)
    t0 = time.perf_counter()
    for _ in range(n_np):
        eval_callback_set(model, xp_, yp_, 1.0, cp_, Jp_, Hp_)
    e2e_numpy_pinned = n_np / (time.perf_counter() - t0)
    assert np.array_equal(Hp_, Hn) and np.array_equal(Jp_, Jn)
    # latency view: one set at a time, synchronised per set
    t0 = time.perf_counter()
    for i in range(n_e2e // NS):
        e2e_issue(0)
        slots[0]["st"].synchronize()
    e2e_seq = (n_e2e // NS) / (time.perf_counter() - t0)
    if ws > 1:
        t = torch.tensor([e2e_dt], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_dt = float(t.item())
    for sl in slots:
        lib.exa_workspace_destroy(sl["ws"])
    e2e_value = n_e2e * (1 if sharded else ws) / e2e_dt
    h2d = 8 * (model.nvar + model.ncon)
    # D2H: c plus the x-dependent J/H ranges; the constant runs (constant J
    # slots, structural-zero H pairs) are written into the host arrays by host
    # threads inside the same call (plans[0].layout.fill_*)
    lay0 = plans[0].layout
    filled = 8 * int(lay0.fill_jac[:, 1].sum() + lay0.fill_hess[:, 1].sum())
    d2h = 8 * (model.ncon + model.plan.n_jac_slots + model.plan.n_hess_slots) - filled

    if rank != 0:
        if ws > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline and bps < 2e9 and ws == 1:  # rank 0 at N=1 only
        xb, yb, wb = eval_inputs(model, 0)
        cpu = cpu_baseline(model, xb, yb, wb, args.cpu_seconds, args.workload)
    info = plans[0].info()
    line = {
        "metric": METRIC, "value": value, "unit": "sets/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {
            "workload": args.workload, "sets_per_step": S, "form": "polar",
            "nvar": summ["nvar"], "ncon": summ["ncon"], "jac_slots": summ["jac_slots"],
            "hess_slots": summ["hess_slots"], "bytes_per_set": bps,
            "l2": f"rotating {R} full replicas ({R * bps / 2**20:.0f} MiB > 2x126 MiB L2)",
            "launch": "CUDA graph of single-set fused kernel launches (exa_k_set)",
            "parallelism": (f"{'period' if args.workload.startswith('mp') else 'instance'} shards x{ws}"
                            if sharded and ws > 1 else (f"replicas x{ws}" if ws > 1 else "single GPU")),
            "shard_bytes_per_set": bps,
        },
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "exa_k_set", "traffic_source": traffic_src,
                     "achieved_basis": "algorithmic bytes per set (SURVEY 8d) / mean per-launch time"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "sets/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": (f"exa_eval_set_host (C ABI): pinned host x,y -> HBM -> set kernel -> pinned host c,J,H; "
                         f"one set per step, {NS} streams in round robin; constant J/H runs "
                         f"({filled / 1e6:.1f} MB) written by host threads, not copied"),
                "host_filled_bytes_per_step": filled,
                "d2h_GBps": d2h * e2e_value / (1 if sharded else ws) / 1e9,
                "sequential_value": e2e_seq, "numpy_api_value": e2e_numpy,
                "numpy_api_pinned_value": e2e_numpy_pinned},
        "clocks": sampler.summary(),
        "batched": batched,
        "gpu_launches": args.steps * S,
        "kernel_regs": info["regs_set_kernel"],
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
