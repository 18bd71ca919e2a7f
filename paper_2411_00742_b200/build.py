"""Builds libpbe.so (the C-ABI shared library, include/pbe.h) with nvcc for sm_100a, in-tree."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpbe.so")
SOURCES = ["pbe_api.cu"]
MB_LIB = os.path.join(HERE, "libpbe_mb.so")      # roofline microbenchmarks (bench.py only)
MB_SOURCES = ["microbench.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def _deps():
    out = [os.path.join(ROOT, "include", "pbe.h")]
    for f in os.listdir(CSRC):
        if f.endswith((".cu", ".cuh", ".h")) and f != "microbench.cu":
            out.append(os.path.join(CSRC, f))
    return out


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in _deps())


def _nvcc(out, sources, tag, verbose):
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, "-o", tmp, *[os.path.join(CSRC, s) for s in sources]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, f"build_{tag}.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed (see {log}):\n{r.stderr[-4000:]}")
    if verbose:
        print(r.stderr[-2000:], file=sys.stderr)
    os.replace(tmp, out)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        _nvcc(LIB, SOURCES, "pbe", verbose)
    mb_src = os.path.join(CSRC, MB_SOURCES[0])
    if force or not os.path.exists(MB_LIB) or os.path.getmtime(MB_LIB) < os.path.getmtime(mb_src):
        _nvcc(MB_LIB, MB_SOURCES, "mb", verbose)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
