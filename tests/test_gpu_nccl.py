"""ShardComm over NCCL on >= 2 B200s (skipped with fewer GPUs): the same
contract as tests/test_distributed_cpu.py (gloo), with the halo exchange and
the objective reduction on the GPUs and every shard's cons/jac/hess evaluated
by the CUDA kernels -- the sharded callbacks reassemble the global set
(IEEE-equal to the CR-trig oracle), and the rank-ordered objective is deterministic."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(kind, rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parent))
        from test_distributed_cpu import _shard

        from oracle import crtrig
        from oracle import tape_oracle as O
        from paper_2510_12897_b200 import eval_callback_set
        from paper_2510_12897_b200.synth import evaluation_point

        dev = torch.device("cuda", rank)
        gm, sm, var_map, row_map, jac_map, hess_map, comm = _shard(kind, rank, world)
        sm.to_device(rank)
        comm.setup()
        x, y, w = evaluation_point(gm, 3)
        xl = torch.full((sm.nvar,), float("nan"), dtype=torch.float64, device=dev)
        owned = np.ones(sm.nvar, dtype=bool)
        for ids in comm.recv.values():
            owned[ids] = False
        xl[torch.as_tensor(np.flatnonzero(owned), device=dev)] = torch.as_tensor(x[var_map[owned]], device=dev)
        comm.exchange(xl)
        xl = torch.nan_to_num(xl, nan=0.0)  # unread borrowed entries never enter a term
        out = [torch.empty(n, dtype=torch.float64, device=dev)
               for n in (sm.ncon, sm.plan.n_jac_slots, sm.plan.n_hess_slots)]
        with torch.cuda.device(rank):
            eval_callback_set(sm, xl, torch.as_tensor(y[row_map], device=dev), w, *out)
        c, J, H = (t.cpu().numpy() for t in out)
        f = comm.objective(xl)
        f2 = comm.objective(xl)
        parts = [None] * world
        dist.all_gather_object(parts, (row_map, c, jac_map, J, hess_map, H))
        if rank == 0:
            O.use_trig(crtrig.TRIG)
            gc, gJ, gH = O.eval_set(gm.plan, x, y, w)
            cc, JJ, HH = (np.full(n, np.nan) for n in (gm.ncon, gm.plan.n_jac_slots, gm.plan.n_hess_slots))
            for rm, a, jm, b, hm, d in parts:
                cc[rm], JJ[jm], HH[hm] = a, b, d
            ok = bool(np.all(cc == gc) and np.all(JJ == gJ) and np.all(HH == gH))
            q.put((ok, f == f2, np.isfinite(f)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("kind", ["mp", "n1"])
def test_nccl_sharded_callbacks(kind):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(kind, r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, det, fin = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
    assert ok, "NCCL-sharded GPU callbacks do not reassemble the global set"
    assert det and fin
