"""Multi-process (world_size 2, gloo, CPU) tests of the sharding + record all-gather used by
bench.py --gpus N: every simulation is owned by exactly one rank, and the
gathered table equals the single-process table in global order, bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_00742_b200 import dist as D


def test_shard_partition():
    for n, w in [(4096, 8), (10, 3), (7, 2), (5, 8)]:
        parts = [D.shard(n, r, w) for r in range(w)]
        allv = np.sort(np.concatenate(parts))
        assert np.array_equal(allv, np.arange(n))
        assert [len(p) for p in parts] == D.shard_sizes(n, w)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_sims, P, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    M = 7
    samples = rng.standard_normal((n_sims, M, 6))
    samples[3, 5:] = np.nan                      # a failed sim with fewer valid samples
    status = np.zeros(n_sims, np.int32); status[3] = 4
    steps = rng.integers(1, 1000, n_sims)
    loss = rng.standard_normal(n_sims)
    grad = rng.standard_normal((n_sims, P))
    mine = D.shard(n_sims, rank, world)
    loc = torch.from_numpy(D.pack_records(status[mine], steps[mine], samples[mine], loss[mine], grad[mine]))
    full = D.allgather_records(loc, n_sims)
    ref = D.pack_records(status, steps, samples, loss, grad)
    q.put((rank, bool(np.array_equal(full.numpy(), ref))))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_sims", [9, 16])
def test_allgather_two_ranks(n_sims):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_sims, 3, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_pack_records_torch_matches_numpy():
    rng = np.random.default_rng(1)
    samples = rng.standard_normal((5, 4, 6)); samples[2, 1:] = np.nan
    st = np.arange(5, dtype=np.int32); steps = np.arange(5, dtype=np.int64) * 10
    loss = rng.standard_normal(5); grad = rng.standard_normal((5, 2))
    a = D.pack_records(st, steps, samples, loss, grad)
    b = D.pack_records(torch.from_numpy(st), torch.from_numpy(steps), torch.from_numpy(samples),
                       torch.from_numpy(loss), torch.from_numpy(grad)).numpy()
    assert np.array_equal(a, b)
