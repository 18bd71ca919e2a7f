"""Print the adjoint-vs-oracle gradient errors of the NEXT-3 parity cases (diagnostics)."""
import os, sys; sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'tests']
import numpy as np, math
from test_gpu_adjoint import *
cases = dict(poly=lambda: small_ensemble(), long=lambda: small_ensemble(n_params=40, n_sims=3),
             upwind=lambda: small_ensemble(n_sims=3, limiter=W.LIM_UPWIND),
             cfl=lambda: small_ensemble(n_sims=3, dt_max=math.inf, t_max=120.0, M=12))
for name, f in cases.items():
    w = f(); lo, go = oracle_grad(w); g, rec, info = gpu_adjoint(w)
    scale = np.max(np.abs(go), axis=1, keepdims=True)
    print(name, "grad err %.2e" % (np.abs(g["grad"] - go) / scale).max(), "loss err %.2e" % (np.abs(g["loss"] - lo) / np.abs(lo)).max(),
          "scale", scale.ravel()[:3], "g0", g["grad"][0, :3], "go", go[0, :3], "steps", rec["steps"][:3], "ms", info["main_ms"])
