"""NEXT-3 timing: one gradient of the RSS loss over all n_params POLY coefficients for the 9
App-B experiments, three ways on the GPU:
  adjoint   pbe_run_adjoint (reverse mode, cost independent of n_params)
  tangents  forward mode, ceil(n_params / 10) passes of 10 tangent lanes (pbe_run_batch)
  fd        batched forward differences (the paper's jax-ND analogue): one pbe_run_batch of
            9 x (n_params + 1) primal simulations
usage: next3_time.py [n_params=1000] [N=2000] [t_max=600] [M=600] [tangent_passes_timed=3]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402


def main():
    a = sys.argv[1:]
    P = int(a[0]) if len(a) > 0 else 1000
    N = int(a[1]) if len(a) > 1 else 2000
    t_max = float(a[2]) if len(a) > 2 else 600.0
    M = int(a[3]) if len(a) > 3 else 600
    n_tp = int(a[4]) if len(a) > 4 else 3
    w = W.next3_estimation(n_params=P, N=N, t_max=t_max, M=M)
    S = w.n_sims
    dev = torch.device("cuda", 0)
    n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).to(dev)
    res = dict(n_params=P, N=N, sims=S, M=M)

    # ---- adjoint -----------------------------------------------------------------------------
    ctx = pb.context_for(w)
    times = []
    for it in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ctx.run_adjoint(n0, w.c0, w.t_samples, w.target)
        g = ctx.adjoint_gradient(P)
        torch.cuda.synchronize(); times.append(time.perf_counter() - t0)
    rec = ctx.moments()
    res.update(adjoint_ms=1e3 * min(times), adjoint_kernel_ms=ctx.last_run_info()["main_ms"],
               steps=int(rec["steps"].max()), loss=float(g["loss"].sum()))
    ctx.close()
    # the O(sqrt K)-checkpoint mode (re-march each segment) for comparison
    os.environ["PBE_ADJ_RECOMPUTE"] = "1"
    ctx = pb.context_for(w)
    times = []
    for it in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ctx.run_adjoint(n0, w.c0, w.t_samples, w.target)
        g2 = ctx.adjoint_gradient(P)
        torch.cuda.synchronize(); times.append(time.perf_counter() - t0)
    res.update(adjoint_recompute_ms=1e3 * min(times),
               traj_vs_recompute_maxabs=float(np.abs(g2["grad"] - g["grad"]).max()))
    ctx.close()
    del os.environ["PBE_ADJ_RECOMPUTE"]

    # ---- forward-mode tangents: 10 lanes per pass --------------------------------------------
    passes = (P + 9) // 10
    Q = w.sol.shape[0]
    ptimes = []
    gt = np.zeros((S, P))
    for j0 in range(0, min(P, 10 * n_tp), 10):
        nl = min(10, P - j0)
        seed = np.zeros((nl, P + Q)); seed[np.arange(nl), j0 + np.arange(nl)] = 1.0
        wk = W.replace(w, n_tangents=nl, tangent_seed=seed)
        c = pb.context_for(wk)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        c.run_batch(n0, w.c0, w.t_samples, w.target)
        tg = c.tangents()
        torch.cuda.synchronize(); ptimes.append(time.perf_counter() - t0)
        gt[:, j0:j0 + nl] = tg["grad"]
        c.close()
    res.update(tangent_pass_ms=1e3 * float(np.median(ptimes)), tangent_passes=passes,
               tangent_ms_total=1e3 * float(np.median(ptimes)) * passes)
    k = min(P, 10 * n_tp)
    scale = np.max(np.abs(g["grad"][:, :k]), axis=1, keepdims=True)
    res["adjoint_vs_tangent_maxrel"] = float((np.abs(g["grad"][:, :k] - gt[:, :k]) / scale).max())

    # ---- batched forward differences (jax-ND analogue) ---------------------------------------
    h = 1e-6
    th = np.repeat(w.theta, P + 1, axis=0)                     # [S (P+1)][P]
    for s in range(S):
        blk = th[s * (P + 1):(s + 1) * (P + 1)]
        blk[1 + np.arange(P), np.arange(P)] += h * np.maximum(np.abs(w.theta[s]), 1e-3)
    wf = W.replace(w, theta=th, c0=np.repeat(w.c0, P + 1), knot_T=np.repeat(w.knot_T, P + 1, axis=0),
                   target=np.repeat(w.target, P + 1, axis=0))
    c = pb.context_for(wf)
    ftimes = []
    for it in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        c.run_batch(n0, wf.c0, wf.t_samples, wf.target)
        r = c.moments()
        torch.cuda.synchronize(); ftimes.append(time.perf_counter() - t0)
    c.close()
    res.update(fd_ms=1e3 * min(ftimes), fd_sims=int(wf.n_sims))
    res["speedup_vs_tangents"] = res["tangent_ms_total"] / res["adjoint_ms"]
    res["speedup_vs_fd"] = res["fd_ms"] / res["adjoint_ms"]
    print("NEXT3", res, flush=True)


if __name__ == "__main__":
    main()
