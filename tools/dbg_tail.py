import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, workloads as W, paper_2411_00742_b200 as pb
w = W.c5_ensemble(n_sims=148, N=300, t_max=15.0, M=15)
gf = pb.run_workload(w)
g = pb.run_workload(w.subset([17]))
for k in ("samples", "tsamples", "n_final", "ndot_final", "loss", "grad", "steps"):
    a, b = g[k], gf[k][[17]]
    d = np.abs(a - b)
    print(k, "equal" if np.array_equal(a, b, equal_nan=True) else f"maxdiff {np.nanmax(d):.3e} rel {np.nanmax(d/np.maximum(np.abs(b),1e-300)):.3e} first idx {np.argwhere(d>0)[:3].tolist()}")
