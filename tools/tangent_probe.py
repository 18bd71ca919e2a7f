"""Tangent-pass timing for the NEXT-3 experiment at several parameter/lane counts (diagnostics)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2411_00742_b200 as pb, workloads as W
for P, nl in [(8, 8), (10, 8), (10, 10), (1000, 10), (1000, 8)]:
    w = W.next3_estimation(n_params=P)
    Q = w.sol.shape[0]
    seed = np.zeros((nl, P + Q)); seed[np.arange(nl), np.arange(nl)] = 1.0
    wk = W.replace(w, n_tangents=nl, tangent_seed=seed)
    ctx = pb.context_for(wk)
    n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).cuda()
    ctx.run_batch(n0, w.c0, w.t_samples, w.target); ctx.moments()
    ctx.run_batch(n0, w.c0, w.t_samples, w.target); r = ctx.moments()
    print("params", P, "lanes", nl, "ms %.1f" % ctx.last_run_info()["main_ms"], ctx.last_run_info(), flush=True)
    ctx.close()
