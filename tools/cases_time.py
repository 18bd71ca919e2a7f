"""GPU time of C1-C3 and small C4 cases (AUTO kernels): us/step, for A/B of kernel changes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

for name, w in (("c1", W.c1_growth(W.LIM_VANLEER, M=1000)), ("c2", W.c2_dissolution()), ("c3", W.c3_cycling()),
                ("c4_1e4x64", W.c4_sweep(10000, batch=64, n_steps=1000)), ("c4_1e3x1184", W.c4_sweep(1000, batch=1184, n_steps=1000))):
    ctx = pb.context_for(w)
    n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).cuda()
    ts = w.t_samples if w.n_steps == 0 else None
    ms = []
    for it in range(5):
        ctx.run_batch(n0, w.c0, ts, w.target)
        r = ctx.moments()
        if it >= 2:
            ms.append(ctx.last_run_info()["main_ms"])
    steps = float(np.mean(r["steps"]))
    print(name, "kernel", ctx.last_run_info()["kernel"], "us/step %.3f" % (1e3 * min(ms) / steps),
          "rate %.3e" % (w.N * np.sum(r["steps"]) / (min(ms) * 1e-3)))
    ctx.close()
