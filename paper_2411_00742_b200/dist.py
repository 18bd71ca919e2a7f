"""Multi-GPU sharding of independent simulations.

Simulations are independent, so the ensemble shards with no data-path collective:
rank r of W runs sims {s : s mod W = r} (round-robin spreads the App. B experiments and the
parameter draws evenly).  The only exchange is ONE all-gather of fixed-size per-simulation
records (status, steps, final state, loss, gradient) at the end — NCCL over NVLink on the
GPU box, gloo in the CPU tests.  No simulation ever spans GPUs.
"""
from __future__ import annotations

import numpy as np

REC_FIXED = 10   # status, steps, t_end, c_end, mu0, mu1, mu2, mu3, loss, n_valid_samples


def shard(n_sims: int, rank: int, world: int) -> np.ndarray:
    """Simulation indices owned by `rank` (round-robin)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return np.arange(rank, n_sims, world, dtype=np.int64)


def shard_sizes(n_sims: int, world: int):
    return [len(range(r, n_sims, world)) for r in range(world)]


def record_width(n_tangents: int) -> int:
    return REC_FIXED + n_tangents


def pack_records(status, steps, samples, loss, grad=None):
    """Per-simulation fixed-size records [S][REC_FIXED + P] (float64) from one rank's
    outputs: the last valid sample (t, c, mu0..mu3), loss and gradient.  Accepts numpy
    arrays or torch tensors (torch stays on its device)."""
    try:
        import torch
        is_t = isinstance(samples, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_t = False
    if is_t:
        import torch
        S, M, _ = samples.shape
        valid = ~torch.isnan(samples[:, :, 0])
        nvalid = valid.sum(dim=1)
        idx = torch.clamp(nvalid - 1, min=0)
        last = samples[torch.arange(S, device=samples.device), idx]
        P = 0 if grad is None else grad.shape[1]
        out = torch.empty((S, REC_FIXED + P), dtype=torch.float64, device=samples.device)
        out[:, 0] = status.to(torch.float64)
        out[:, 1] = steps.to(torch.float64)
        out[:, 2:8] = last
        out[:, 8] = loss
        out[:, 9] = nvalid.to(torch.float64)
        if P:
            out[:, REC_FIXED:] = grad
        return out
    samples = np.asarray(samples)
    S = samples.shape[0]
    valid = ~np.isnan(samples[:, :, 0])
    nvalid = valid.sum(axis=1)
    last = samples[np.arange(S), np.maximum(nvalid - 1, 0)]
    P = 0 if grad is None else np.asarray(grad).shape[1]
    out = np.empty((S, REC_FIXED + P))
    out[:, 0] = status; out[:, 1] = steps; out[:, 2:8] = last; out[:, 8] = loss; out[:, 9] = nvalid
    if P:
        out[:, REC_FIXED:] = grad
    return out


def allgather_records(local, n_sims: int, group=None):
    """All-gathers every rank's records (torch tensor [S_r][R]) and returns the full
    [n_sims][R] table in global simulation order.  Uses one all_gather_into_tensor on a
    padded [W][S_max][R] buffer (equal-size chunks, as NCCL requires)."""
    import torch
    import torch.distributed as dist
    W = dist.get_world_size(group)
    sizes = shard_sizes(n_sims, W)
    smax = max(sizes)
    R = local.shape[1]
    pad = torch.full((smax, R), float("nan"), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    full = torch.empty((W * smax, R), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(full, pad, group=group)
    full = full.view(W, smax, R)
    out = torch.empty((n_sims, R), dtype=local.dtype, device=local.device)
    for r in range(W):
        out[r::W] = full[r, : sizes[r]]
    return out
