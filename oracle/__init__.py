"""CPU oracle for the batched 1D PBE finite-volume march — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product path (paper_2411_00742_b200/) must never import it:
it shares no code with the CUDA path.

The arithmetic lives in oracle/pbe_oracle.cpp (serial C++17, templated on the scalar:
double, Dual tangents, complex step).  This file only marshals a workloads.Workload into
the oracle's own C struct and calls it through ctypes.  It also builds the .so with g++
(-O2, no -ffast-math, no -march=native; denormals enabled) when it is missing or stale.

Parity status: every function is pinned in tests/test_oracle_pins.py (see DESIGN.md
"Pins").  The dissolution law (R-12), the polynomial solubility (R-13) and the temperature
profile (R-14) are our readings of the paper; their *values* are "parity unpinned" by any
paper passage (they are pinned only by self-consistency identities: mirror symmetry,
conservation, positivity, exact-rational brute force and the method of moments).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pbe_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
GXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-shared", "-Wall"]
_lock = threading.Lock()
_lib = None

MODE_DOUBLE, MODE_DUAL, MODE_CSTEP = 0, 1, 2


class _Problem(C.Structure):
    _fields_ = [
        ("N", C.c_int32), ("L_lo", C.c_double), ("dL", C.c_double), ("limiter", C.c_int32),
        ("courant", C.c_double), ("dt_fixed", C.c_double), ("dt_max", C.c_double),
        ("max_steps", C.c_int64), ("n_steps", C.c_int64), ("rho_c", C.c_double), ("k_v", C.c_double),
        ("law", C.c_int32), ("n_params", C.c_int32), ("sol_kind", C.c_int32), ("n_sol", C.c_int32),
        ("sol", C.POINTER(C.c_double)), ("n_knots", C.c_int32), ("knot_t", C.POINTER(C.c_double)),
        ("knot_T", C.POINTER(C.c_double)), ("knot_T_stride", C.c_int64),
        ("M", C.c_int32), ("t_samples", C.POINTER(C.c_double)),
        ("n_tan", C.c_int32), ("tangent_seed", C.POINTER(C.c_double)),
        ("N2", C.c_int32), ("L2_lo", C.c_double), ("dL2", C.c_double),
    ]


def build(force: bool = False) -> str:
    """Compile oracle/liboracle.so with g++ (building the checker is not using it)."""
    with _lock:
        stale = (not os.path.exists(_LIB)) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC)
        if force or stale:
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["g++", *GXX_FLAGS, "-o", tmp, _SRC, "-lpthread"])
            os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB)
        dp, ip, lp = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int64)
        lib.oracle_run_batch.argtypes = [C.POINTER(_Problem), C.c_int32, dp, dp, C.c_int64, dp, dp, dp, ip,
                                         lp, dp, dp, C.c_int32, C.c_int32]
        lib.oracle_run_batch.restype = C.c_int
        lib.oracle_kinetics.argtypes = [C.POINTER(_Problem), dp, C.c_double, C.c_double, dp]
        lib.oracle_sweep.argtypes = [C.c_int32, dp, C.c_double, C.c_int32, dp]
        lib.oracle_moments.argtypes = [C.POINTER(_Problem), dp, dp]
        lib.oracle_dual_si_example.argtypes = [C.c_double] * 4 + [dp]
        lib.oracle_run_batch_2d.argtypes = [C.POINTER(_Problem), C.c_int32, dp, dp, C.c_int64, dp, dp, ip, lp, dp,
                                            C.c_int32]
        lib.oracle_run_batch_2d.restype = C.c_int
        lib.oracle_split_step_2d.argtypes = [C.c_int32, C.c_int32, dp, C.c_double, C.c_double, C.c_int32, dp]
        _lib = lib
    return _lib


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _problem(w, keep):
    sol = _f64(w.sol); kt = _f64(w.knot_t); kT = _f64(w.knot_T); ts = _f64(w.t_samples)
    seed = _f64(w.tangent_seed)
    keep.extend([sol, kt, kT, ts, seed])
    return _Problem(
        N=w.N, L_lo=w.L_lo, dL=w.dL, limiter=w.limiter, courant=w.courant, dt_fixed=w.dt_fixed,
        dt_max=w.dt_max, max_steps=w.max_steps, n_steps=w.n_steps, rho_c=w.rho_c, k_v=w.k_v,
        law=w.law, n_params=w.n_params, sol_kind=w.sol_kind, n_sol=int(sol.shape[0]), sol=_dp(sol),
        n_knots=int(kt.shape[0]), knot_t=_dp(kt), knot_T=_dp(kT),
        knot_T_stride=int(kt.shape[0]) if kT.shape[0] > 1 else 0,
        M=int(ts.shape[0]), t_samples=_dp(ts), n_tan=w.n_tangents, tangent_seed=_dp(seed),
        N2=getattr(w, "N2", 0), L2_lo=getattr(w, "L2_lo", 0.0), dL2=getattr(w, "dL2", 0.0))


def run(w, mode: int = MODE_DOUBLE, threads: int = 1, want_n: bool = True) -> dict:
    """March every simulation of workload `w` (rows a1-a8).  Returns numpy arrays:
    samples [S][M][6] = (t, c, mu0, mu1, mu2, mu3); status [S]; steps [S];
    n_final [S][N]; and for mode DUAL/CSTEP tsamples [S][M][P][5] = d(c, mu0..mu3) and
    ndot_final [S][P][N]."""
    lib = _load()
    keep = []
    pb = _problem(w, keep)
    S, N, M, P = w.n_sims, w.N, w.M, w.n_tangents
    theta = _f64(w.theta); n0 = _f64(w.n0); c0 = _f64(w.c0)
    samples = np.full((S, M, 6), np.nan)
    tsamples = np.full((S, M, P, 5), np.nan) if mode != MODE_DOUBLE else None
    status = np.zeros(S, np.int32); steps = np.zeros(S, np.int64)
    n_final = np.zeros((S, N)) if want_n else None
    ndot = np.zeros((S, P, N)) if (want_n and mode != MODE_DOUBLE) else None
    rc = lib.oracle_run_batch(C.byref(pb), S, _dp(theta), _dp(n0), N if n0.shape[0] > 1 else 0, _dp(c0),
                              _dp(samples), _dp(tsamples), status.ctypes.data_as(C.POINTER(C.c_int32)),
                              steps.ctypes.data_as(C.POINTER(C.c_int64)), _dp(n_final), _dp(ndot),
                              mode, threads)
    if rc != 0:
        raise RuntimeError(f"oracle_run_batch failed ({rc})")
    out = dict(samples=samples, status=status, steps=steps, n_final=n_final)
    if mode != MODE_DOUBLE:
        out.update(tsamples=tsamples, ndot_final=ndot)
    return out


def kinetics(w, theta, t: float, c: float, sim: int = 0):
    """(T, c*, S, G) at time t and concentration c for simulation `sim`'s T-profile (row a1)."""
    lib = _load()
    keep = []
    ws = w.subset([sim]) if w.knot_T.shape[0] > 1 else w
    pb = _problem(ws, keep)
    th = _f64(np.asarray(theta))
    out = np.zeros(4)
    lib.oracle_kinetics(C.byref(pb), _dp(th), float(t), float(c), _dp(out))
    return tuple(out)


def sweep(f, C_: float, limiter: int) -> np.ndarray:
    """One eq-highRes_growth update (rows a3-a4, no clip) of f with Courant number C_."""
    lib = _load()
    f = _f64(f); out = np.zeros_like(f)
    lib.oracle_sweep(int(f.shape[0]), _dp(f), float(C_), int(limiter), _dp(out))
    return out


def moments(w, n) -> np.ndarray:
    """(mu0, mu1, mu2, mu3) of n on w's grid (row a5)."""
    lib = _load()
    keep = []
    pb = _problem(w, keep)
    n = _f64(n); out = np.zeros(4)
    lib.oracle_moments(C.byref(pb), _dp(n), _dp(out))
    return out


def loss_and_grad(samples, tsamples, target):
    """Row a7 epilogue (R-23): RSS over concentration and mean length
    Lbar = mu1/mu0, each residual normalised by the RMS of its target trace.
      loss = sum_m ((c_m - c^_m)/rms_c)^2 + ((Lbar_m - L^_m)/rms_L)^2
      grad_p = sum_m 2 (c_m - c^_m)/rms_c^2 dc_m/dp + 2 (Lbar_m - L^_m)/rms_L^2 dLbar_m/dp
    samples [S][M][6], tsamples [S][M][P][5] or None, target [S][M][2]."""
    c = samples[:, :, 1]; mu0 = samples[:, :, 2]; mu1 = samples[:, :, 3]
    Lbar = mu1 / mu0
    rms_c = np.sqrt(np.mean(target[:, :, 0] ** 2, axis=1))[:, None]
    rms_L = np.sqrt(np.mean(target[:, :, 1] ** 2, axis=1))[:, None]
    rc = (c - target[:, :, 0]) / rms_c
    rL = (Lbar - target[:, :, 1]) / rms_L
    loss = np.sum(rc ** 2 + rL ** 2, axis=1)
    grad = None
    if tsamples is not None:
        dc = tsamples[:, :, :, 0]; dmu0 = tsamples[:, :, :, 1]; dmu1 = tsamples[:, :, :, 2]
        dL = (dmu1 * mu0[:, :, None] - mu1[:, :, None] * dmu0) / (mu0[:, :, None] ** 2)
        grad = np.sum(2.0 * (rc / rms_c)[:, :, None] * dc + 2.0 * (rL / rms_L)[:, :, None] * dL, axis=1)
    return loss, grad


def dual_si_example(x1: float, x2: float, v1: float, v2: float):
    """SI Table S1 function y1 = sin x1/(x1+x2), y2 = (x1+x2) e^{x2} in the oracle's Dual."""
    lib = _load()
    out = np.zeros(4)
    lib.oracle_dual_si_example(x1, x2, v1, v2, _dp(out))
    return tuple(out)


def run2d(w, threads: int = 1, want_f: bool = True) -> dict:
    """NEXT-1 2D march (Godunov splitting) of every simulation of 2D workload `w`:
    samples [S][M][8] = (t, c, mu00, mu10, mu01, mu11, mu02, mu12), status, steps,
    f_final [S][N2][N1] (L1 fastest)."""
    lib = _load()
    keep = []
    pb = _problem(w, keep)
    S, M, NN = w.n_sims, w.M, w.N * w.N2
    theta = _f64(w.theta); f0 = _f64(w.n0); c0 = _f64(w.c0)
    samples = np.full((S, M, 8), np.nan)
    status = np.zeros(S, np.int32); steps = np.zeros(S, np.int64)
    f_final = np.zeros((S, w.N2, w.N)) if want_f else None
    rc = lib.oracle_run_batch_2d(C.byref(pb), S, _dp(theta), _dp(f0), NN if f0.shape[0] > 1 else 0, _dp(c0),
                                 _dp(samples), status.ctypes.data_as(C.POINTER(C.c_int32)),
                                 steps.ctypes.data_as(C.POINTER(C.c_int64)), _dp(f_final), threads)
    if rc != 0:
        raise RuntimeError(f"oracle_run_batch_2d failed ({rc})")
    return dict(samples=samples, status=status, steps=steps, f_final=f_final)


def split_step_2d(f, C1: float, C2: float, limiter: int) -> np.ndarray:
    """One Godunov-split step (rows along L1 with C1, then columns along L2 with C2) of f[N2][N1]."""
    lib = _load()
    f = _f64(f); out = np.zeros_like(f)
    lib.oracle_split_step_2d(int(f.shape[1]), int(f.shape[0]), _dp(f), float(C1), float(C2), int(limiter), _dp(out))
    return out
