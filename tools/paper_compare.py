"""Wall-clock of the paper's reported workloads on this GPU (context for BASELINE.md §1; the
paper's numbers are on an RTX 4090 and are not targets):
  2d      Table 1 base case on the 6000 x 3000 grid, uncapped CFL to 1000 min (the paper's
          "1339 time steps"), one simulation: seconds per march
  est4    one Adam iteration of the App. B estimation with 4 coefficients (9 experiments,
          5 um bins, 600 min): loss + exact gradient (tangent lanes)
  est4x   the same, 64 independent fits per launch (multi-start), seconds per fit-iteration
Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2411_00742_b200.estimate import Estimator, make_experiments  # noqa: E402


def wall(f, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        f()
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best


out = {}
w = W.c2d_base(6000, 3000, t_max=1000.0, M=1)
ctx = pb.context_for(w)
n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).cuda()


def march():
    ctx.run_batch(n0, w.c0, w.t_samples, None)
    return ctx.moments()


s2d = wall(march, reps=2)
r = march()
out["2d_6000x3000"] = dict(seconds=s2d, steps=int(r["steps"][0]), paper_rtx4090_seconds_derived=0.4,
                           cell_steps_per_s=6000 * 3000 * float(r["steps"][0]) / s2d)
ctx.close()

N = 240                                          # 5 um bins on [0, 1200] um
exps = make_experiments(N, W.gaussian_seed(N, 1200.0 / N), t_max=600.0, M=600)
th = np.array([[0.5, 5.0, 20.0, 50.0]])
est = Estimator(exps, th)
t1 = wall(lambda: est.loss_and_grad(th))
est.close()
est = Estimator(exps, np.repeat(th, 64, axis=0))
t64 = wall(lambda: est.loss_and_grad(np.repeat(th, 64, axis=0)))
est.close()
out["est4"] = dict(seconds_per_iteration=t1, paper_jax_ad_seconds=0.10, paper_jax_nd_seconds=0.02)
out["est4x64"] = dict(seconds_per_launch=t64, seconds_per_fit_iteration=t64 / 64)
print("PAPERCMP", json.dumps(out), flush=True)
