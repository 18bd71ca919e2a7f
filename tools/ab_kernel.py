"""Forced-kernel timing of C4-shaped batches: N batch steps kernels(comma: 1=resident,2=cluster,3=stream)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

N, B, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
for kern in [int(k) for k in sys.argv[4].split(",")]:
    w = W.c4_sweep(N, batch=B, n_steps=steps)
    try:
        ctx = pb.context_for(w, kernel=kern)
        n0 = torch.from_numpy(w.n0).cuda()
        for _ in range(2):
            ctx.run_batch(n0, w.c0, None, None); r = ctx.moments()
        ms = []
        for _ in range(3):
            ctx.run_batch(n0, w.c0, None, None); r = ctx.moments(); ms.append(ctx.last_run_info()["main_ms"])
        bu = float(N) * float(r["steps"].sum())
        print("RESULT", N, B, kern, "%.3e" % (bu / (min(ms) * 1e-3)), ctx.last_run_info())
        ctx.close()
    except Exception as e:
        print("RESULT", N, B, kern, "error", str(e)[:120])
