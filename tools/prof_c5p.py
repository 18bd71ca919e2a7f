"""C5-shaped run with a chosen number of tangent lanes (for ncu): sims, t_max, lanes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

sims, tmax, P = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
w = W.c5_ensemble(n_sims=sims, t_max=tmax, M=int(tmax), n_tangents=P)
r = pb.run_workload(w, want_n=False)
assert np.all(r["status"] == 0)
print("ok", r["info"])
