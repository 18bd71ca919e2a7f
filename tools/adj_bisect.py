"""Bisect an adjoint-vs-oracle gradient mismatch from the fuzz sweep: vary one factor at a time."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from tests.test_gpu_adjoint import gpu_adjoint, oracle_grad  # noqa: E402
from tests.test_gpu_fuzz import random_case  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 5
rng = np.random.Generator(np.random.PCG64(9000 + seed))
w, _ = random_case(seed)
if w.n_steps:
    w = W.replace(w, n_steps=0, t_samples=np.linspace(2.0, 2.0 * int(rng.integers(1, 6)), int(rng.integers(1, 6))))
w = W.replace(w, n_tangents=0, tangent_seed=None, target=W._target(w.c0, w.t_samples))
print("case: N", w.N, "lim", w.limiter, "law", w.law, "params", w.n_params, "sol", w.sol_kind, "knots", w.knot_t.shape[0],
      "dt_fixed", w.dt_fixed, "dt_max", w.dt_max, "M", w.M, "sims", w.n_sims)


def err(wv, tag):
    lo, go = oracle_grad(W.replace(wv, max_steps=4000), allow_fail=True)
    g, rec, _ = gpu_adjoint(wv)
    ok = np.isfinite(lo)
    if not ok.any():
        print(tag, "all failed", rec["status"]); return
    scale = np.max(np.abs(go[ok]), axis=1, keepdims=True)
    e = (np.abs(g["grad"][ok] - go[ok]) / np.maximum(scale, 1e-300))
    print(f"{tag:28s} max rel {e.max():.2e}  per-param {np.round(e.max(axis=0), 12)}  status {rec['status']}")


err(w, "as drawn")
err(W.replace(w, limiter=W.LIM_VANLEER), "limiter -> van Leer")
err(W.replace(w, limiter=W.LIM_UPWIND), "limiter -> upwind")
err(W.replace(w, sol_kind=W.SOL_EXP, sol=np.array(W.SOL_EXP_DEFAULT)), "sol -> exp")
err(W.replace(w, knot_t=np.array([0.0]), knot_T=w.knot_T[:, :1].copy()), "T -> constant")
err(W.replace(w, dt_max=np.inf), "dt -> uncapped")
err(W.replace(w, t_samples=w.t_samples[:1]), "one sample")

# three-way comparison on the one-sample variant
import paper_2411_00742_b200 as pb  # noqa: E402
w1 = W.replace(w, t_samples=w.t_samples[:1], target=w.target[:, :1].copy())
lo, go = oracle_grad(W.replace(w1, max_steps=4000), allow_fail=True)
P = w1.n_params
Q = w1.sol.shape[0]
seed = np.zeros((P, P + Q)); seed[np.arange(P), np.arange(P)] = 1.0
r = pb.run_workload(W.replace(w1, n_tangents=P, tangent_seed=seed), want_n=False)
g, rec, _ = gpu_adjoint(w1)
print("oracle  ", go[0], lo[0])
print("tangents", r["grad"][0], r["loss"][0])
print("adjoint ", g["grad"][0], g["loss"][0], "steps", rec["steps"][0])
