"""Period sharding of multi-period OPF: host logic and 2-rank gloo assembly (CPU).

The CUDA kernels are checked elsewhere; here the oracle evaluates each shard
so that the sharding plan itself (windows, overlap variables, maps) is shown
to reproduce the global callbacks bit-for-bit, with the objective combined by
an all-reduce as on the multi-GPU path.
"""

import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tape_oracle as O
from paper_2510_12897_b200 import mpopf_model, synthetic_case
from paper_2510_12897_b200.sharding import attach_maps, mpopf_shard, period_windows
from paper_2510_12897_b200.synth import demand_curve, evaluation_point


def _case(storage=False):
    case = synthetic_case(40, 8, 60, seed=5)
    if storage:
        from paper_2510_12897_b200.matpower import Storage

        case.storage = [Storage(3, 2.0, 0.5, 0.5, 0.9, 0.95), Storage(7, 1.0, 0.3, 0.4, 0.92, 0.9)]
    return case


def test_period_windows_partition():
    for T, n in ((96, 8), (96, 3), (7, 7), (5, 2)):
        w = period_windows(T, n)
        assert w[0][0] == 0 and w[-1][1] == T
        assert all(a[1] == b[0] for a, b in zip(w, w[1:]))
        assert max(b - a for a, b in w) - min(b - a for a, b in w) <= 1


def _set(model, x, y, w):
    return O.eval_set(model.plan, x, y, w)


@pytest.mark.parametrize("storage", [False, True])
@pytest.mark.parametrize("n", [2, 3])
def test_shards_reassemble_global_bitwise(storage, n):
    case = _case(storage)
    curve = demand_curve(7)
    gm = mpopf_model(case, curve, 0.25, lower_to_gpu=False)[0]
    x, y, w = evaluation_point(gm, 3)
    gc, gJ, gH = _set(gm, x, y, w)
    gg = np.empty(gm.nvar)
    O.eval_gradient(gm.plan, x, gg)
    c = np.full(gm.ncon, np.nan)
    J = np.full(gm.plan.n_jac_slots, np.nan)
    H = np.full(gm.plan.n_hess_slots, np.nan)
    g = np.zeros(gm.nvar)
    f = 0.0
    for r in range(n):
        sh = attach_maps(mpopf_shard(case, curve, r, n, lower_to_gpu=False), gm)
        xs, ys = x[sh.var_map], y[sh.row_map]
        sc, sJ, sH = _set(sh.model, xs, ys, w)
        assert np.all(np.isnan(c[sh.row_map])), "rows owned twice"
        c[sh.row_map], J[sh.jac_map], H[sh.hess_map] = sc, sJ, sH
        sg = np.empty(sh.model.nvar)
        O.eval_gradient(sh.model.plan, xs, sg)
        np.add.at(g, sh.var_map, sg)
        f += O.eval_objective(sh.model.plan, xs)
    for a, b in ((c, gc), (J, gJ), (H, gH), (g, gg)):
        assert not np.isnan(a).any()
        assert np.all(a == b)
    assert f == pytest.approx(O.eval_objective(gm.plan, x), rel=1e-13)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    case = _case(False)
    curve = demand_curve(6)
    gm = mpopf_model(case, curve, 0.25, lower_to_gpu=False)[0]
    x, y, w = evaluation_point(gm, 1)
    sh = attach_maps(mpopf_shard(case, curve, rank, world, lower_to_gpu=False), gm)
    sc, sJ, sH = _set(sh.model, x[sh.var_map], y[sh.row_map], w)
    f = torch.tensor([O.eval_objective(sh.model.plan, x[sh.var_map])], dtype=torch.float64)
    dist.all_reduce(f)  # the only collective of the sharded callback set (objective)
    parts = [None] * world
    dist.all_gather_object(parts, (sh.row_map, sc, sh.jac_map, sJ, sh.hess_map, sH))
    if rank == 0:
        gc, gJ, gH = _set(gm, x, y, w)
        c = np.empty(gm.ncon)
        J = np.empty(gm.plan.n_jac_slots)
        H = np.empty(gm.plan.n_hess_slots)
        for rm, a, jm, b, hm, d in parts:
            c[rm], J[jm], H[hm] = a, b, d
        ok = bool(np.all(c == gc) and np.all(J == gJ) and np.all(H == gH))
        rel = abs(float(f.item()) - O.eval_objective(gm.plan, x)) / abs(O.eval_objective(gm.plan, x))
        q.put((ok, rel))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_set():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, rel = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert ok and rel < 1e-13
