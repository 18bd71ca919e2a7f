"""A/B timing of C4-shaped batches under env settings: N batch steps 'ENV=..;ENV2=..|...'"""
import os
import subprocess
import sys

N, B, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
envs = [dict(kv.split("=") for kv in e.split(",") if kv) for e in (sys.argv[4] if len(sys.argv) > 4 else "").split("|")]
code = f"""
import numpy as np, torch, paper_2411_00742_b200 as pb, workloads as W
w = W.c4_sweep({N}, batch={B}, n_steps={steps})
ctx = pb.context_for(w)
n0 = torch.from_numpy(w.n0).cuda()
for _ in range(2):
    ctx.run_batch(n0, w.c0, None, None); r = ctx.moments()
ms = []
for _ in range(3):
    ctx.run_batch(n0, w.c0, None, None); r = ctx.moments(); ms.append(ctx.last_run_info()['main_ms'])
bu = w.N * r['steps'].sum()
print('RESULT', dict(ms=round(min(ms), 3), rate='%.3e' % (bu / (min(ms) * 1e-3)), info=ctx.last_run_info(), ok=bool((r['status'] == 0).all())))
"""
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for env in envs:
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True, cwd=root)
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
    print(N, B, env, line[0] if line else out.stderr[-1500:])
