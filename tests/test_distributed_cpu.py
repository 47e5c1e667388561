"""Product-level shard communication (distributed.ShardComm) on CPU with gloo:
halo / linking-variable exchange refreshes exactly the variables each shard's
terms read from other shards, the objective reduction is rank-ordered and
deterministic, and with the exchanged x every shard's cons/jac/hess reassemble
the global callbacks bit for bit (oracle as the evaluator; the CUDA kernels
are checked in the -m gpu suites)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tape_oracle as O
from paper_2510_12897_b200 import mpopf_model, synthetic_case
from paper_2510_12897_b200.distributed import ShardComm, mpopf_comm, scopf_comm
from paper_2510_12897_b200.scopf import attach_instance_maps, scopf_model, scopf_shard
from paper_2510_12897_b200.sharding import attach_maps, mpopf_shard
from paper_2510_12897_b200.synth import demand_curve, evaluation_point


def _mp_case():
    from paper_2510_12897_b200.matpower import Storage

    case = synthetic_case(40, 8, 60, seed=5)
    case.storage = [Storage(3, 2.0, 0.5, 0.5, 0.9, 0.95), Storage(7, 1.0, 0.3, 0.4, 0.92, 0.9)]
    return case


def _shard(kind, rank, world):
    if kind == "mp":
        case, curve = _mp_case(), demand_curve(7)
        gm = mpopf_model(case, curve, 0.25, lower_to_gpu=False)[0]
        sh = attach_maps(mpopf_shard(case, curve, rank, world, lower_to_gpu=False), gm)
        comm = mpopf_comm(sh, curve.size, True, rank, world)
        return gm, sh.model, sh.var_map, sh.row_map, sh.jac_map, sh.hess_map, comm
    case, cont = synthetic_case(30, 6, 45, seed=11), [2, 5, 7, 11, 20, 23, 30]
    gm = scopf_model(case, cont, lower_to_gpu=False)[0]
    sm, owned = scopf_shard(case, cont, rank, world, lower_to_gpu=False)
    var_map, _, row_map, jac_map, hess_map = attach_instance_maps(sm, gm, owned)
    comm = scopf_comm(sm, len(cont) + 1, rank, world)
    return gm, sm, var_map, row_map, jac_map, hess_map, comm


def _worker(kind, rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gm, sm, var_map, row_map, jac_map, hess_map, comm = _shard(kind, rank, world)
        comm.setup()
        x, y, w = evaluation_point(gm, 3)
        # the caller fills only what this rank owns; borrowed entries start as NaN
        xl = torch.full((sm.nvar,), float("nan"), dtype=torch.float64)
        owned = np.ones(sm.nvar, dtype=bool)
        for ids in comm.recv.values():
            owned[ids] = False
        xl[torch.as_tensor(np.flatnonzero(owned))] = torch.as_tensor(x[var_map[owned]])
        comm.exchange(xl)
        xs = xl.numpy()
        used = np.zeros(sm.nvar, dtype=bool)
        for tp in sm.plan.obj_terms + sm.plan.con_terms:
            for cols in tp.cols:
                used[np.asarray(cols)] = True
        ok_x = bool(np.array_equal(xs[used], x[var_map][used]))
        xs = np.where(np.isnan(xs), 0.0, xs)  # unread borrowed entries never enter a term
        c, J, H = O.eval_set(sm.plan, xs, y[row_map], w)
        f = comm.reduce_objective(O.eval_objective(sm.plan, xs))
        f2 = comm.reduce_objective(O.eval_objective(sm.plan, xs))
        parts = [None] * world
        dist.all_gather_object(parts, (row_map, c, jac_map, J, hess_map, H, ok_x, comm.halo_doubles()))
        if rank == 0:
            gc, gJ, gH = O.eval_set(gm.plan, x, y, w)
            cc, JJ, HH = np.full(gm.ncon, np.nan), np.full(gm.plan.n_jac_slots, np.nan), np.full(gm.plan.n_hess_slots, np.nan)
            for rm, a, jm, b, hm, d, _, _ in parts:
                cc[rm], JJ[jm], HH[hm] = a, b, d
            ok = bool(np.all(cc == gc) and np.all(JJ == gJ) and np.all(HH == gH))
            fg = O.eval_objective(gm.plan, x)
            q.put((ok, all(p[6] for p in parts), abs(f - fg) / abs(fg), f == f2, [p[7] for p in parts]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(kind, world):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(kind, r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("kind,world", [("mp", 2), ("mp", 3), ("n1", 2)])
def test_sharded_exchange_and_objective(kind, world):
    ok, ok_x, rel, det, halos = _run(kind, world)
    assert ok_x, "borrowed variables not refreshed from their owners"
    assert ok, "sharded cons/jac/hess do not reassemble the global callbacks"
    assert rel < 1e-13 and det
    assert all(h > 0 for h in halos[1:]) or kind == "n1"


def test_plan_borrows_only_linking_variables():
    """Period shards borrow only the variables their linking rows read: the
    next period's generator outputs (ramp) and, with storage, the previous
    period's stored energy (SoC chain) -- never voltages or flows."""
    case, curve = _mp_case(), demand_curve(7)
    sh = mpopf_shard(case, curve, 1, 3, lower_to_gpu=False)
    comm = mpopf_comm(sh, curve.size, True, 1, 3)
    v = sh.model.variables
    names = {id(b): n for n, b in zip(("va", "vm", "pg", "qg", "p", "q"), v)}
    borrowed = np.concatenate(list(comm.recv.values()))
    for i in borrowed:
        blk = next(b for b in v if b.offset <= i < b.offset + b.size)
        assert names.get(id(blk)) not in ("va", "vm", "p", "q", "qg")
    assert set(comm.recv) == {0, 2}
    assert isinstance(comm, ShardComm)
