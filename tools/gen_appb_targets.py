"""Writes workloads/data/appb_targets.npy: the App. B in-silico "measurements" (PAPER.md
L734-744: 9 experiments, T in {10, 15, 20} C x S0 in {1.15, 1.25, 1.5}, 600 uniform samples,
targets from the method of moments with the Arrhenius truth, L741-743) that C5 and NEXT-3 use
as the RSS target (row a7, R-23).

Method of moments: tests/mom.py (SI eq-mom2D reduced to one length, fixed-step RK4, kinetics
re-typed from Eq. A.1/A.2; it routes through neither oracle/ nor the CUDA path), started from the
discrete moments of the C5 seed (N = 2000 bins, Gaussian 400/30 um, m0 = 1 g/kg), h = 0.005 min
(step halving changes the stored values by < 1e-9 relative; checked below).
Output: float64 [9][600][2] = (c, mean length mu1/mu0) at t = 1, 2, ..., 600 min.
usage: python tools/gen_appb_targets.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from tests import mom  # noqa: E402

OUT = os.path.join(ROOT, "workloads", "data", "appb_targets.npy")
N, M, T_MAX = 2000, 600, 600.0
TRUTH = W.ARRHENIUS_DEFAULT[:3]             # Table A.1 dimension 1 (growth only: S0 > 1 throughout)


def traces(h: float) -> np.ndarray:
    dL = 1200.0 / N
    n0 = W.gaussian_seed(N, dL, m0=1.0)
    L = W.bin_centers(N, dL)
    mu0 = np.array([np.sum(dL * L ** k * n0) for k in range(4)])
    out = np.empty((9, M, 2))
    for e in range(9):
        T = W.APPB_T[e // 3]
        c0 = W.APPB_S0[e % 3] * W.APPB_CSAT[e // 3]
        w = W.Workload(name="appb", N=N, dL=dL, law=W.LAW_ARRHENIUS, theta=np.array([TRUTH]),
                       sol_kind=W.SOL_EXP, sol=np.array(W.SOL_EXP_DEFAULT), knot_t=np.array([0.0]),
                       knot_T=np.array([[T]]), n0=n0[None, :], c0=np.array([c0]))
        y = np.concatenate([[c0], mu0])
        per = int(round((T_MAX / M) / h))
        for m in range(M):
            w.c0 = np.array([y[0]])
            y = mom.solve(w, y[1:], T_MAX / M, per)
            out[e, m] = (y[0], y[2] / y[1])
    return out


if __name__ == "__main__":
    a = traces(0.005)
    if "--check" in sys.argv:
        b = traces(0.01)
        print("step-halving max rel diff", np.max(np.abs(a - b) / np.abs(a)))
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.save(OUT, a)
    print(OUT, a.shape, a[:, -1])
