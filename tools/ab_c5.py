"""A/B timing of C5-shaped ensembles under different env settings (run in subprocesses).
usage: python tools/ab_c5.py <n_sims> <t_max> <tangents>"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sims, tmax, P = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
code = f"""
import time, numpy as np, torch, paper_2411_00742_b200 as pb, workloads as W
w = W.c5_ensemble(n_sims={sims}, t_max={tmax}, M=int({tmax}), n_tangents={P})
ctx = pb.context_for(w)
n0 = torch.from_numpy(w.n0).cuda()
for _ in range(2):
    ctx.run_batch(n0, w.c0, w.t_samples, w.target); r = ctx.moments()
ms = []
for _ in range(3):
    ctx.run_batch(n0, w.c0, w.t_samples, w.target); r = ctx.moments(); ms.append(ctx.last_run_info()['main_ms'])
bu = w.N * r['steps'].sum()
print('RESULT', dict(ms=min(ms), rate=bu / (min(ms) * 1e-3), info=ctx.last_run_info(), ok=bool((r['status'] == 0).all())))
"""
envs = [{}] if len(sys.argv) < 5 else [{}, dict(kv.split("=") for kv in sys.argv[4].split(","))]
for env in envs:
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
    print(env, line[0] if line else out.stderr[-2000:])
