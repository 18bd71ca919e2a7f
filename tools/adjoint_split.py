"""Adjoint cost split (NEXT-3): primal march vs adjoint at several checkpoint intervals and parameter counts."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2411_00742_b200 as pb, workloads as W
w = W.next3_estimation(n_params=1000)
n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).cuda()
ctx = pb.context_for(w)
for _ in range(2):
    ctx.run_batch(n0, w.c0, w.t_samples, w.target); ctx.moments()
print("primal 9 sims (resident, P=0): %.1f ms" % ctx.last_run_info()["main_ms"], ctx.last_run_info())
for ck in (0, 16, 64, 256):
    ctx.run_adjoint(n0, w.c0, w.t_samples, w.target, checkpoint_every=ck); ctx.adjoint_gradient(1000)
    ctx.run_adjoint(n0, w.c0, w.t_samples, w.target, checkpoint_every=ck); ctx.adjoint_gradient(1000)
    print("adjoint ck=%d: %.1f ms" % (ck, ctx.last_run_info()["main_ms"]))
w8 = W.next3_estimation(n_params=8)
c8 = pb.context_for(w8)
c8.run_adjoint(n0, w8.c0, w8.t_samples, w8.target); c8.adjoint_gradient(8)
c8.run_adjoint(n0, w8.c0, w8.t_samples, w8.target); c8.adjoint_gradient(8)
print("adjoint 8 params: %.1f ms" % c8.last_run_info()["main_ms"])
