"""Time the 2D march (c2d_base N1 x N2, uncapped CFL steps) for batches: ab_2d.py N1 N2 steps b1,b2,..
Prints main_ms and cells*steps/s per batch (kernel from the loaded library, PBE_LIB to switch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

N1, N2, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
for b in [int(x) for x in sys.argv[4].split(",")]:
    w = W.c2d_base(N1, N2, n_sims=b)
    w.n_steps = steps
    w.t_samples = np.array([1.0])
    ctx = pb.context_for(w)
    n0 = torch.from_numpy(w.n0).cuda()
    ms = []
    for it in range(4):
        ctx.run_batch(n0, w.c0, None, None)
        r = ctx.moments()
        if it:
            ms.append(ctx.last_run_info()["main_ms"])
    cu = float(N1) * N2 * float(r["steps"].sum())
    print("RESULT", os.path.basename(os.environ.get("PBE_LIB", "default")), N1, N2, b, "%.3f ms" % min(ms),
          "%.3e cells/s" % (cu / (min(ms) * 1e-3)), "ctas", ctx.last_run_info()["ctas"], flush=True)
    ctx.close()
