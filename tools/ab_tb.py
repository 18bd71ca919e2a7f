"""C4 with and without temporal blocking (NEXT-4): ab_tb.py N batch steps."""
import os
import subprocess
import sys

code = """
import sys, numpy as np, torch, paper_2411_00742_b200 as pb, workloads as W
N, B, steps = %d, %d, %d
w = W.c4_sweep(N, batch=B, n_steps=steps)
ctx = pb.context_for(w)
n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).cuda()
ms = []
for it in range(4):
    ctx.run_batch(n0, w.c0, None, None); r = ctx.moments()
    if it: ms.append(ctx.last_run_info()['main_ms'])
print('RESULT', 'tb' if ctx.last_run_info()['steps_per_pass'] > 1 else 'plain', N, B, steps,
      '%%.3e' %% (float(N) * r['steps'].sum() / (min(ms) * 1e-3)), 'ok' if (r['status'] == 0).all() else r['status'])
"""
N, B, steps = (int(a) for a in sys.argv[1:4])
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for tb in ("0", "1"):
    env = dict(os.environ, PBE_TEMPORAL_BLOCK=tb)
    out = subprocess.run([sys.executable, "-c", code % (N, B, steps)], env=env, capture_output=True, text=True, cwd=root)
    print([l for l in out.stdout.splitlines() if l.startswith("RESULT")] or out.stderr[-1500:])
