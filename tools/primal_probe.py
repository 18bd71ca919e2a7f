"""Per-step latency of small primal batches (NEXT-3 shape, 9 sims x 2000 bins, 600 samples):
primal_probe.py -> ms and us/step for several parameter counts; PBE_RESIDENT_K to vary K."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

for P in (8, 1000):
    for tgt in (True, False):
        w = W.next3_estimation(n_params=P)
        n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).cuda()
        ctx = pb.context_for(w)
        for _ in range(2):
            ctx.run_batch(n0, w.c0, w.t_samples, w.target if tgt else None); r = ctx.moments()
        i = ctx.last_run_info()
        print(f"params {P} target {tgt}: {i['main_ms']:.1f} ms, {1e3 * i['main_ms'] / r['steps'].max():.2f} us/step, "
              f"K {i['bins_per_thread']} threads {i['threads_per_cta']}", flush=True)
        ctx.close()
