"""C4-shaped run for ncu captures: batch of 64 x 10^6 bins, van Leer, uncapped CFL,
`steps` time steps (default 50) through the streaming kernel.  Exits 0 on success."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
w = W.c4_sweep(N, batch=batch, n_steps=steps)
r = pb.run_workload(w, want_n=False)
assert np.all(r["status"] == 0)
print("ok", r["info"])
