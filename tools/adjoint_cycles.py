"""Phase split of the adjoint kernel (needs a -DPBE_TIMING=1 build via PBE_LIB):
PBE_LIB=variants/libpbe_timing.so python tools/adjoint_cycles.py [n_params]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
w = W.next3_estimation(n_params=P)
ctx = pb.context_for(w)
n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).cuda()
ctx.run_adjoint(n0, w.c0, w.t_samples, w.target)
ctx.adjoint_gradient(P)
lib = pb.load_library()
buf = (C.c_ulonglong * 16)()
assert lib.pbe_debug_adjoint_cycles(buf) == 0
c = np.array(buf[:16], dtype=np.float64)
steps = c[4]
print(f"params {P}: {ctx.last_run_info()['main_ms']:.1f} ms, {steps:.0f} steps")
for n, v in zip(["forward", "fwd exchange wait (traj: no recompute)", "backward vector", "backward scalar"], c[:4]):
    print(f"  {n:16s} {v / steps:8.0f} cycles/step")
for n, v in zip(["fwd update+moments", "fwd barrier+poly", "fwd warp-0 chain"], c[5:8]):
    print(f"    {n:18s} {v / steps:8.0f} cycles/step")
for n, v in zip(["bwd theta", "bwd loads", "bwd faces", "bwd out+shfl"], c[8:12]):
    print(f"    {n:18s} {v / steps:8.0f} cycles/step")
for n, v in zip(["chain pre-kinetics", "chain kinetics"], c[12:14]):
    print(f"    {n:18s} {v / steps:8.0f} cycles/step")
for n, v in zip(["poly: reduction", "poly: partials"], c[14:16]):
    print(f"    {n:18s} {v / steps:8.0f} cycles/step")
