"""Bitwise A/B of two libpbe builds on streaming-kernel cases (steps and sample mode): run once per
build (PBE_LIB=...) writing an .npz, then compare with numpy.array_equal.
usage: [PBE_LIB=...] PBE_TEMPORAL_BLOCK=0 python tools/bitwise_ab.py out.npz"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys, numpy as np, paper_2411_00742_b200 as pb, workloads as W
out = {}
for name, w in [("plain", W.c4_sweep(300000, batch=8, n_steps=40)),
                ("sample", W.replace(W.c4_sweep(300000, batch=4, n_steps=0), t_samples=__import__('numpy').linspace(0.5, 3.0, 5), dt_max=0.02, n_steps=0))]:
    r = pb.run_workload(w, want_n=True)
    out[name + "_s"] = r["samples"]; out[name + "_n"] = r["n_final"]
    print(name, r["info"])
np.savez(sys.argv[1], **out)
