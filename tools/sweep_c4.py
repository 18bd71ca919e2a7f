"""C4 bin-count sweep: bin-updates/s for N in 1e3..1e6, single simulation and batches, AUTO
kernel choice.  Writes profiles/r01_c4_sweep.json (and prints one line per point)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

out = []
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
for N in (1000, 10_000, 100_000, 1_000_000):
    for B in (1, 64, 1184):
        if N * B > 64_000_000:
            continue
        w = W.c4_sweep(N, batch=B, n_steps=steps)
        ctx = pb.context_for(w)
        n0 = torch.from_numpy(w.n0).cuda()
        for _ in range(2):
            ctx.run_batch(n0, w.c0, None, None)
            r = ctx.moments()
        ms = []
        for _ in range(3):
            ctx.run_batch(n0, w.c0, None, None)
            r = ctx.moments()
            ms.append(ctx.last_run_info()["main_ms"])
        info = ctx.last_run_info()
        bu = float(N) * float(r["steps"].sum())
        rec = dict(N=N, batch=B, steps=steps, ms=min(ms), rate=bu / (min(ms) * 1e-3),
                   us_per_step=1e3 * min(ms) / steps, kernel={1: "resident", 2: "cluster", 3: "stream"}[info["kernel"]],
                   info=info, ok=bool(np.all(r["status"] == 0)))
        if info["kernel"] == 3:
            rec["hbm_gbs_algorithmic"] = 16.0 * bu / (min(ms) * 1e-3) / 1e9
        out.append(rec)
        print(json.dumps(rec), flush=True)
        ctx.close()
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "c4_sweep.json"), "w"), indent=1)
