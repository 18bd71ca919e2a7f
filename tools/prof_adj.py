"""One NEXT-3 adjoint gradient (9 App-B experiments, N = 2000, n_params coefficients) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
w = W.next3_estimation(n_params=P)
ctx = pb.context_for(w)
n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).cuda()
ctx.run_adjoint(n0, w.c0, w.t_samples, w.target)
g = ctx.adjoint_gradient(P)
torch.cuda.synchronize()
print("adjoint ms", ctx.last_run_info()["main_ms"], "loss", float(g["loss"].sum()))
