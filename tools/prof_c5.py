"""Small C5-shaped run for ncu captures: 296 sims (2 waves on 148 SMs), 2000 bins,
8 tangent lanes, 60 min of the march (~1200 steps).  Exits 0 on success."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

sims = int(sys.argv[1]) if len(sys.argv) > 1 else 296
tmax = float(sys.argv[2]) if len(sys.argv) > 2 else 60.0
w = W.c5_ensemble(n_sims=sims, t_max=tmax, M=int(tmax))
r = pb.run_workload(w, want_n=False)
assert np.all(r["status"] == 0)
print("ok", r["info"], "steps/sim", r["steps"].mean())
