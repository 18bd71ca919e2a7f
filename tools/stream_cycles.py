"""Per-CTA step split of the plain streaming kernel (needs a -DPBE_TIMING=1 build via PBE_LIB):
own tile work, grid-barrier wait, scalar phase — mean / min / max over CTAs, cycles per step.
usage: PBE_LIB=variants/libpbe_timing.so PBE_TEMPORAL_BLOCK=0 python tools/stream_cycles.py [N] [batch] [steps]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2411_00742_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
w = W.c4_sweep(N, batch=B, n_steps=steps)
lib = pb.load_library()
r = pb.run_workload(w, want_n=False)
info = r["info"]
assert info["kernel"] == 3 and info["steps_per_pass"] == 1, info
G = info["ctas"]
tile = 256
while tile < 4096 and tile * 256 < N:      # stream_tile(N, 1), k_stream.cuh
    tile *= 2
buf = (C.c_ulonglong * (1024 * 5))()
assert lib.pbe_debug_stream_cycles(buf) == 0
a = np.array(buf, dtype=np.float64).reshape(1024, 5)[:G]
st = a[:, 3]
per = a[:, :3] / st[:, None]
tot = per.sum(axis=1)
print(f"N {N} batch {B} steps {int(st.max())} CTAs {G}  main_ms {info['main_ms']:.3f}  "
      f"cycles/step (CTA mean) {tot.mean():.0f}")
for k, name in enumerate(["own tile work", "grid-barrier wait", "scalar phase"]):
    v = per[:, k]
    print(f"  {name:18s} mean {v.mean():8.0f}  min {v.min():8.0f}  max {v.max():8.0f}  ({100 * v.mean() / tot.mean():5.1f}%)")
print(f"  clip-path warp-tiles per step (all CTAs) {a[:, 4].sum() / st.max():.1f} "
      f"of {8 * np.ceil(N / tile) * B:.0f}")
