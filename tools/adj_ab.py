"""A/B of adjoint variants in one process (env toggles read per run):
python tools/adj_ab.py [n_params] VAR=VAL[,VAR=VAL] ...   ('-' = defaults)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

P = int(sys.argv[1])
w = W.next3_estimation(n_params=P)
n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).cuda()
ref = None
for rnd in range(2):
    for spec in sys.argv[2:]:
        env = dict(kv.split("=") for kv in spec.split(",")) if spec != "-" else {}
        for k, v in env.items():
            os.environ[k] = v
        ctx = pb.context_for(w)
        ts = []
        for it in range(3):
            ctx.run_adjoint(n0, w.c0, w.t_samples, w.target)
            g = ctx.adjoint_gradient(P)
            ts.append(ctx.last_run_info()["main_ms"])
        info = ctx.last_run_info()
        ctx.close()
        for k in env:
            del os.environ[k]
        d = 0.0 if ref is None else float(np.abs(g["grad"] - ref).max() / np.abs(ref).max())
        ref = g["grad"] if ref is None else ref
        print(f"{spec:30s} K={info['bins_per_thread']} NT={info['threads_per_cta']} {min(ts):8.2f} ms  "
              f"rel diff {d:.1e}", flush=True)
