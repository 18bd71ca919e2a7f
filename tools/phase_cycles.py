"""Per-phase cycle split of the resident kernel (needs a -DPBE_TIMING=1 build via PBE_LIB):
usage: PBE_LIB=variants/libpbe_timing.so python tools/phase_cycles.py [sims] [t_max] [tangents]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

sims = int(sys.argv[1]) if len(sys.argv) > 1 else 148
tmax = float(sys.argv[2]) if len(sys.argv) > 2 else 30.0
P = int(sys.argv[3]) if len(sys.argv) > 3 else 8
w = W.c5_ensemble(n_sims=sims, t_max=tmax, M=int(tmax), n_tangents=P)
lib = pb.load_library()
r = pb.run_workload(w, want_n=False)
buf = (C.c_ulonglong * 12)()
assert lib.pbe_debug_phase_cycles(buf) == 0
c = np.array(buf[:5], dtype=np.float64)
steps = c[4]
names = ["sweep", "moments+publish", "barrier wait", "scalar phase"]
tot = c[:4].sum()
print(f"steps {steps:.0f}  cycles/step {tot / steps:.0f}  (main_ms {r['info']['main_ms']:.3f})")
for n, v in zip(names, c[:4]):
    print(f"  {n:18s} {v / steps:8.0f} cycles/step  {100 * v / tot:5.1f}%")
c2 = np.array(buf[5:8], dtype=np.float64)
for n, v in zip(["  scalar: load+sums", "  scalar: mass bal.", "  scalar: kinetics"], c2):
    print(f"  {n:18s} {v / steps:8.0f} cycles/step")
c3 = np.array(buf[8:10], dtype=np.float64)
for n, v in zip(["    S + growth law", "    time step"], c3):
    print(f"  {n:18s} {v / steps:8.0f} cycles/step")
