"""Adjoint-vs-forward discrepancy of fuzz seed 5 as a function of the mesh (diagnostics)."""
import os, sys
sys.path[:0] = [os.getcwd()]
import numpy as np
import workloads as W
import paper_2411_00742_b200 as pb
from tests.test_gpu_adjoint import gpu_adjoint, oracle_grad
from tests.test_gpu_fuzz import random_case
seed = 5
rng = np.random.Generator(np.random.PCG64(9000 + seed))
w, _ = random_case(seed)
w = W.replace(w, n_tangents=0, tangent_seed=None)
mean = float(sys.argv[1]) if len(sys.argv) > 1 else 500.0
lim = int(sys.argv[2]) if len(sys.argv) > 2 else w.limiter
w = W.replace(w, limiter=lim)
for N in (60, 61, 120, 240, 480):
    wN = W.replace(w, N=N, dL=1200.0 / N, n0=W.gaussian_seed(N, 1200.0 / N, mean=mean, sigma=70.0)[None, :],
                   t_samples=np.array([2.0, 4.0]))
    wN = W.replace(wN, target=W._target(wN.c0, wN.t_samples))
    lo, go = oracle_grad(W.replace(wN, max_steps=4000), allow_fail=True)
    g, rec, _ = gpu_adjoint(wN)
    P = wN.n_params; Q = wN.sol.shape[0]
    seedm = np.zeros((P, P + Q)); seedm[np.arange(P), np.arange(P)] = 1.0
    r = pb.run_workload(W.replace(wN, n_tangents=P, tangent_seed=seedm), want_n=False)
    sc = np.max(np.abs(go))
    print(N, "steps", rec["steps"], "adj-ora %.2e" % (np.abs(g["grad"] - go).max() / sc), "tan-ora %.2e" % (np.abs(r["grad"] - go).max() / sc),
          "adj-tan %.2e" % (np.abs(g["grad"] - r["grad"]).max() / sc), flush=True)
