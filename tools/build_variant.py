"""Build libpbe variants with extra -D flags for A/B timing: build_variant.py TAG -DX=1 ...
Output: variants/libpbe_TAG.so (git-ignored; travels with gpurun).  Load with PBE_LIB=..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_00742_b200 import build as B  # noqa: E402

tag, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(B.ROOT, "variants"), exist_ok=True)
out = os.path.join(B.ROOT, "variants", f"libpbe_{tag}.so")
cmd = [B.NVCC, *B.FLAGS, *defs, "-o", out, os.path.join(B.CSRC, "pbe_api.cu")]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-3000:])
lines = r.stdout.splitlines() + r.stderr.splitlines()
for k, l in enumerate(lines):
    if "Compiling entry function" in l and "k_2d_fused" in l:
        print(tag, lines[k + 2].strip(), "|", lines[k + 3].strip())
print(out)
