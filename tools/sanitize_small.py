"""Tiny runs of every kernel variant for compute-sanitizer (memcheck / racecheck / synccheck):
resident (primal + 8 lanes, landing, dissolution), cluster (2 lanes), stream (primal, 2 lanes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

cases = [
    ("resident P0 landing", W.c3_cycling(N=300, t_max=2.0, M=4, dt_max=0.1), pb.KERNEL_RESIDENT),
    ("resident P8", W.c5_ensemble(n_sims=3, N=500, t_max=2.0, M=2), pb.KERNEL_RESIDENT),
    ("resident dissolution", W.c2_dissolution(N=400, t_max=2.0, M=2, dt_max=0.2), pb.KERNEL_RESIDENT),
    ("cluster P2", W.c5_ensemble(n_sims=2, N=3000, t_max=1.0, M=1, n_tangents=2), pb.KERNEL_CLUSTER),
    ("cluster P0 steps", W.c4_sweep(9000, batch=2, n_steps=5), pb.KERNEL_CLUSTER),
    ("stream P0 steps", W.c4_sweep(5000, batch=3, n_steps=4), pb.KERNEL_STREAM),
    ("stream P2 landing", W.c5_ensemble(n_sims=2, N=3001, t_max=0.5, M=1, n_tangents=2), pb.KERNEL_STREAM),
]
for name, w, k in cases:
    r = pb.run_workload(w, kernel=k)
    assert np.all(r["status"] == 0), (name, r["status"])
    print("ok", name, r["info"]["kernel"], r["steps"])
