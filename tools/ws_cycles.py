"""Per-phase cycle split of k_resident_ws (needs a -DPBE_TIMING=1 build via PBE_LIB):
usage: PBE_LIB=variants/libpbe_timing.so python tools/ws_cycles.py [sims] [t_max] [tangents]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

sims = int(sys.argv[1]) if len(sys.argv) > 1 else 148
tmax = float(sys.argv[2]) if len(sys.argv) > 2 else 30.0
P = int(sys.argv[3]) if len(sys.argv) > 3 else 8
w = W.c5_ensemble(n_sims=sims, t_max=tmax, M=int(tmax), n_tangents=P)
lib = pb.load_library()
r = pb.run_workload(w, want_n=False)
buf = (C.c_ulonglong * 8)()
assert lib.pbe_debug_ws_cycles(buf) == 0
c = np.array(buf[:], dtype=np.float64)
steps = max(c[7], 1)
print(f"steps {steps:.0f}  main_ms {r['info']['main_ms']:.3f}  info {r['info']}")
for name, v in zip(["A primal sweep (warp 1)", "barrier 1 wait", "B tangent sweep (warp 1)", "barrier 2 wait",
                    "D tangent scalars + halo", "chain (warp 0)", "B of warp 0 after chain"], c[:7]):
    print(f"  {name:28s} {v / steps:8.0f} cycles/step")
print(f"  step total (warp 1)          {c[:5].sum() / steps:8.0f} cycles/step")
