"""Quick oracle check of the resident tangent kernel (default variant or PBE_WS_VARIANT):
C5-shaped cases at N = 200 and 2000, and a dissolution case (C < 0) with tangents."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

cases = [W.c5_ensemble(n_sims=4, N=200, t_max=5.0, M=5), W.c5_ensemble(n_sims=3, N=2000, t_max=3.0, M=3)]
w = W.c2_dissolution()
cases.append(W.replace(w, n_tangents=6, t_samples=w.t_samples[:30]))
worst = 0.0
for w in cases:
    g = pb.run_workload(w)
    o = oracle.run(w, mode=oracle.MODE_DUAL, threads=8)
    e = dict(status=bool(np.array_equal(g["status"], o["status"])), steps=bool(np.array_equal(g["steps"], o["steps"])),
             mom=float(np.nanmax(np.abs(g["samples"] - o["samples"]) / np.abs(o["samples"]))),
             tan=float(np.nanmax(np.abs(g["tsamples"] - o["tsamples"])) / np.nanmax(np.abs(o["tsamples"]))),
             n=float(np.max(np.abs(g["n_final"] - o["n_final"])) / np.max(o["n_final"])),
             ndot=float(np.max(np.abs(g["ndot_final"] - o["ndot_final"])) / np.max(np.abs(o["ndot_final"]))))
    if w.target is not None:
        lo, go = oracle.loss_and_grad(o["samples"], o["tsamples"], w.target)
        e["loss"] = float(np.max(np.abs(g["loss"] - lo) / np.abs(lo)))
        e["grad"] = float(np.max(np.abs(g["grad"] - go)) / np.max(np.abs(go)))
    print(w.name, g["info"]["warp_specialized"], e)
    worst = max(worst, e["mom"], e["tan"], e["n"], e["ndot"])
print("WORST", worst, "OK" if worst < 1e-9 else "FAIL")
