"""The sharded multi-GPU path (bench.py --gpus N) end to end on one GPU: two
processes each run libpbe on their round-robin shard of a C5-shaped ensemble, pack the per-
simulation records and all-gather them (gloo), and the gathered table must equal the records
of one process running the whole ensemble BITWISE (a simulation's result never depends on
the batch it runs in).  The ranks' kernels are independent (no data-path collective), so two
processes on one GPU exercise exactly the code the N-GPU run executes."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import workloads as W

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload(kind):
    if kind == "c5":
        return W.c5_ensemble(n_sims=21, N=400, t_max=12.0, M=12)
    return W.c4_sweep(3000, batch=7, n_steps=60)


def _worker(rank, world, port, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_2411_00742_b200 as pb
    from paper_2411_00742_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = _workload(kind)
    mine = D.shard(w.n_sims, rank, world)
    r = pb.run_workload(w.subset(mine), want_n=False)
    loc = torch.from_numpy(D.pack_records(r["status"], r["steps"], r["samples"], r["loss"], r.get("grad")))
    full = D.allgather_records(loc, w.n_sims)
    if rank == 0:
        q.put(full.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["c5", "c4"])
def test_two_rank_shards_equal_one_rank_run(kind):
    import paper_2411_00742_b200 as pb
    from paper_2411_00742_b200 import dist as D
    w = _workload(kind)
    r = pb.run_workload(w, want_n=False)
    ref = D.pack_records(r["status"], r["steps"], r["samples"], r["loss"], r.get("grad"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, 2, port, kind, q)) for k in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert full.shape == ref.shape
    assert np.array_equal(full, ref, equal_nan=True)
