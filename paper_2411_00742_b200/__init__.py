"""paper_2411_00742_b200 — B200-native batched PBE finite-volume time-march.

Thin ctypes binding over libpbe.so (C ABI: include/pbe.h).  Argument marshalling only:
every step of the march (kinetics, time step, flux-limited update, moments, mass balance,
sampling, loss, tangent lanes) runs in the sm_100a CUDA kernels of csrc/.  PyTorch is
used for device memory and streams.  There is no CPU fallback: if libpbe.so is missing or
no CUDA device is visible, the calls raise.

Names follow include/pbe.h: Context.create / set_kinetics / run_batch / moments / tangents.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from typing import Optional

import numpy as np

__all__ = ["PBEError", "Context", "run_workload", "lib_path", "load_library", "EXPORTS",
           "LIM_UPWIND", "LIM_VANLEER", "LAW_CONST", "LAW_ARRHENIUS_GD", "LAW_POLY",
           "SOL_EXP", "SOL_POLY", "KERNEL_AUTO", "KERNEL_RESIDENT", "KERNEL_CLUSTER", "KERNEL_STREAM"]

_HERE = os.path.dirname(os.path.abspath(__file__))

LIM_UPWIND, LIM_VANLEER, LIM_MINMOD, LIM_SUPERBEE, LIM_MC = 0, 1, 2, 3, 4
LAW_CONST, LAW_ARRHENIUS_GD, LAW_POLY = 0, 1, 2
SOL_EXP, SOL_POLY = 0, 1
KERNEL_AUTO, KERNEL_RESIDENT, KERNEL_CLUSTER, KERNEL_STREAM, KERNEL_2D, KERNEL_ADJOINT = 0, 1, 2, 3, 4, 5
STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_CFL", 3: "ERR_NEGATIVE", 4: "ERR_INFEASIBLE",
          5: "ERR_MAXSTEPS", 6: "ERR_CUDA", 7: "ERR_NOMEM", 8: "ERR_STATE"}

# every symbol include/pbe.h declares
EXPORTS = ("pbe_create", "pbe_destroy", "pbe_last_error", "pbe_set_kinetics", "pbe_run_batch", "pbe_run_adjoint",
           "pbe_adjoint_gradient",
           "pbe_moments", "pbe_tangents", "pbe_last_run_info", "pbe_version")


class PBEError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Config(C.Structure):
    _fields_ = [("n_bins", C.c_int32), ("L_lo", C.c_double), ("dL", C.c_double), ("limiter", C.c_int32),
                ("courant", C.c_double), ("dt_fixed", C.c_double), ("dt_max", C.c_double),
                ("max_steps", C.c_int64), ("n_steps", C.c_int64), ("rho_c", C.c_double), ("k_v", C.c_double),
                ("n_samples", C.c_int32), ("n_tangents", C.c_int32), ("max_sims", C.c_int32),
                ("kernel", C.c_int32), ("n_bins2", C.c_int32), ("L2_lo", C.c_double), ("dL2", C.c_double)]


class RunInfo(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("launches", C.c_int32), ("threads_per_cta", C.c_int32),
                ("ctas", C.c_int32), ("cluster", C.c_int32), ("bins_per_thread", C.c_int32),
                ("main_ms", C.c_double), ("steps_per_pass", C.c_int32), ("warp_specialized", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib_path() -> str:
    # PBE_LIB: an alternative build of the same library (tools/build_variant.py A/B runs)
    return os.environ.get("PBE_LIB") or os.path.join(_HERE, "libpbe.so")


def load_library():
    """Loads libpbe.so (raises if it has not been built: run __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    vp, dp, ip, lp = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int64)
    lib.pbe_create.argtypes = [C.POINTER(_Config), C.c_int, C.POINTER(vp)]
    lib.pbe_create.restype = C.c_int
    lib.pbe_destroy.argtypes = [vp]
    lib.pbe_destroy.restype = None
    lib.pbe_last_error.argtypes = [vp]
    lib.pbe_last_error.restype = C.c_char_p
    lib.pbe_set_kinetics.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, vp, C.c_int32, C.c_int32, vp,
                                     C.c_int32, vp, vp, C.c_int32, vp]
    lib.pbe_set_kinetics.restype = C.c_int
    lib.pbe_run_batch.argtypes = [vp, C.c_int32, vp, C.c_int64, C.c_int32, vp, vp, vp, vp, vp, vp]
    lib.pbe_run_batch.restype = C.c_int
    lib.pbe_moments.argtypes = [vp, vp, vp, vp, vp, C.c_int32]
    lib.pbe_moments.restype = C.c_int
    lib.pbe_tangents.argtypes = [vp, vp, vp, C.c_int32]
    lib.pbe_tangents.restype = C.c_int
    lib.pbe_run_adjoint.argtypes = [vp, C.c_int32, vp, C.c_int64, C.c_int32, vp, vp, vp, C.c_int32, vp]
    lib.pbe_run_adjoint.restype = C.c_int
    lib.pbe_adjoint_gradient.argtypes = [vp, vp, vp, C.c_int32]
    lib.pbe_adjoint_gradient.restype = C.c_int
    lib.pbe_last_run_info.argtypes = [vp, C.POINTER(RunInfo)]
    lib.pbe_last_run_info.restype = C.c_int
    lib.pbe_version.argtypes = []
    lib.pbe_version.restype = C.c_char_p
    _lib = lib
    return lib


def _ptr(a) -> Optional[int]:
    """Address of a numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()   # torch.Tensor


def _host(a, dtype=np.float64):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


def _check_dev(name: str, t, device: int, shapes) -> None:
    """libpbe cannot check device buffers: a device tensor must be float64, contiguous, on the
    context's device and of one of the allowed shapes (else out-of-bounds device accesses)."""
    if t is None:
        return
    if isinstance(t, np.ndarray):
        raise TypeError(f"{name}: expected a CUDA tensor, got a numpy array")
    import torch
    if t.dtype != torch.float64:
        raise TypeError(f"{name}: dtype must be float64, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if t.device.type != "cuda" or t.device.index != device:
        raise ValueError(f"{name}: must live on cuda:{device}, got {t.device}")
    if tuple(t.shape) not in [tuple(s) for s in shapes]:
        raise ValueError(f"{name}: shape {tuple(t.shape)} not in {[tuple(s) for s in shapes]}")


class Context:
    """One libpbe context (pbe_create): a problem shape bound to one CUDA device."""

    def __init__(self, n_bins: int, dL: float, *, L_lo: float = 0.0, limiter: int = LIM_VANLEER,
                 courant: float = 0.9, dt_fixed: float = 0.0, dt_max: float = math.inf,
                 max_steps: int = 10_000_000, n_steps: int = 0, rho_c: float = 1.11e-12,
                 k_v: float = math.pi / 4, n_samples: int = 1, n_tangents: int = 0, max_sims: int = 1,
                 kernel: int = KERNEL_AUTO, device: int = 0, n_bins2: int = 0, L2_lo: float = 0.0,
                 dL2: float = 0.0):
        self._lib = load_library()
        self.cfg = _Config(n_bins, L_lo, dL, limiter, courant, dt_fixed, dt_max, max_steps, n_steps, rho_c,
                           k_v, n_samples, n_tangents, max_sims, kernel, n_bins2, L2_lo, dL2)
        h = C.c_void_p()
        st = self._lib.pbe_create(C.byref(self.cfg), device, C.byref(h))
        if st != 0:
            raise PBEError(st, self._lib.pbe_last_error(None).decode())
        self._h = h
        self.device = device
        self.n_sims = 0
        self._keep = []

    # ----------------------------------------------------------------------------------
    def _check(self, st: int):
        if st != 0:
            raise PBEError(st, self._lib.pbe_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.pbe_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ----------------------------------------------------------------------------------
    def set_kinetics(self, law: int, theta, sol_kind: int, sol, knot_t, knot_T, tangent_seed=None):
        theta = _host(np.atleast_2d(theta))
        sol = _host(sol); knot_t = _host(np.atleast_1d(knot_t)); knot_T = _host(np.atleast_2d(knot_T))
        seed = _host(tangent_seed)
        per_sim = 1 if knot_T.shape[0] > 1 else 0
        if knot_T.shape[0] not in (1, theta.shape[0]) or knot_T.shape[1] != knot_t.shape[0]:
            raise ValueError(f"knot_T shape {knot_T.shape}: expected [1 or {theta.shape[0]}][{knot_t.shape[0]}]")
        if seed is not None:
            P, nsd = self.cfg.n_tangents, theta.shape[1] + sol.shape[0]
            if seed.size != P * nsd:
                raise ValueError(f"tangent_seed has {seed.size} values: expected [{P}][{nsd}]")
        self._check(self._lib.pbe_set_kinetics(
            self._h, law, theta.shape[1], theta.shape[0], _ptr(theta), sol_kind, sol.shape[0], _ptr(sol),
            knot_t.shape[0], _ptr(knot_t), _ptr(knot_T), per_sim, _ptr(seed)))
        self.n_sims = theta.shape[0]

    def run_batch(self, n0, c0, t_samples=None, target=None, n_final=None, ndot_final=None, stream=None):
        """n0: torch CUDA tensor [S or 1][N] (device path) or numpy array (host path, H2D inside).
        n_final / ndot_final: optional torch CUDA tensors.  stream: torch.cuda.Stream or None
        (= torch's current stream)."""
        on_dev = not isinstance(n0, np.ndarray)
        if not on_dev:
            n0 = _host(n0)
        rows = n0.shape[0] if n0.ndim == 2 else 1
        cells = self.cfg.n_bins * max(self.cfg.n_bins2, 1)
        stride = 0 if rows == 1 else cells
        S, P = self.n_sims, self.cfg.n_tangents
        if on_dev:
            _check_dev("n0", n0, self.device, [(cells,), (1, cells), (S, cells)])
        elif n0.size not in (cells, S * cells):
            raise ValueError(f"n0 has {n0.size} values: expected [1 or {S}][{cells}]")
        _check_dev("n_final", n_final, self.device, [(S, cells)])
        _check_dev("ndot_final", ndot_final, self.device, [(S, P, self.cfg.n_bins)])
        c0 = _host(np.atleast_1d(c0))
        ts = _host(t_samples) if t_samples is not None else np.zeros(1)
        tg = _host(target)
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(self.device) if torch.cuda.is_available() else None
        sp = None if stream is None else C.c_void_p(stream.cuda_stream)
        self._keep = [n0, c0, ts, tg]
        self._check(self._lib.pbe_run_batch(self._h, self.n_sims, _ptr(n0), stride, 1 if on_dev else 0, _ptr(c0),
                                            _ptr(ts), _ptr(tg), _ptr(n_final), _ptr(ndot_final), sp))

    def run_adjoint(self, n0, c0, t_samples, target, checkpoint_every: int = 0, stream=None):
        """NEXT-3: forward march + discrete adjoint (pbe_run_adjoint); read the result with
        adjoint_gradient() and the forward records with moments()."""
        on_dev = not isinstance(n0, np.ndarray)
        if not on_dev:
            n0 = _host(n0)
        rows = n0.shape[0] if n0.ndim == 2 else 1
        stride = 0 if rows == 1 else self.cfg.n_bins
        if on_dev:
            _check_dev("n0", n0, self.device, [(self.cfg.n_bins,), (1, self.cfg.n_bins), (self.n_sims, self.cfg.n_bins)])
        c0 = _host(np.atleast_1d(c0)); ts = _host(t_samples); tg = _host(target)
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(self.device) if torch.cuda.is_available() else None
        sp = None if stream is None else C.c_void_p(stream.cuda_stream)
        self._keep = [n0, c0, ts, tg]
        self._check(self._lib.pbe_run_adjoint(self._h, self.n_sims, _ptr(n0), stride, 1 if on_dev else 0, _ptr(c0),
                                              _ptr(ts), _ptr(tg), int(checkpoint_every), sp))

    def adjoint_gradient(self, n_params: int, on_device: bool = False):
        """d loss / d theta [S][n_params] and loss [S] of the last run_adjoint."""
        S = self.n_sims
        if on_device:
            import torch
            dev = torch.device("cuda", self.device)
            out = dict(grad=torch.empty((S, n_params), dtype=torch.float64, device=dev),
                       loss=torch.empty(S, dtype=torch.float64, device=dev))
        else:
            out = dict(grad=np.empty((S, n_params)), loss=np.empty(S))
        self._check(self._lib.pbe_adjoint_gradient(self._h, _ptr(out["grad"]), _ptr(out["loss"]), 1 if on_device else 0))
        return out

    def moments(self, on_device: bool = False, out: Optional[dict] = None):
        """Records of the last run.  `out` may supply preallocated destinations (e.g. pinned
        host tensors' numpy views) with keys moments/status/steps/loss."""
        S, M = self.n_sims, self.cfg.n_samples
        RW = 8 if self.cfg.n_bins2 > 0 else 6
        if out is not None:
            pass
        elif on_device:
            import torch
            dev = torch.device("cuda", self.device)
            out = dict(moments=torch.empty((S, M, RW), dtype=torch.float64, device=dev),
                       status=torch.empty(S, dtype=torch.int32, device=dev),
                       steps=torch.empty(S, dtype=torch.int64, device=dev),
                       loss=torch.empty(S, dtype=torch.float64, device=dev))
        else:
            out = dict(moments=np.empty((S, M, RW)), status=np.empty(S, np.int32), steps=np.empty(S, np.int64),
                       loss=np.empty(S))
        self._check(self._lib.pbe_moments(self._h, _ptr(out.get("moments")), _ptr(out.get("status")),
                                          _ptr(out.get("steps")), _ptr(out.get("loss")), 1 if on_device else 0))
        return out

    def tangents(self, on_device: bool = False, out: Optional[dict] = None):
        S, M, P = self.n_sims, self.cfg.n_samples, self.cfg.n_tangents
        if out is not None:
            out = dict(out)
            out.setdefault("tangents", None)
        elif on_device:
            import torch
            dev = torch.device("cuda", self.device)
            out = dict(tangents=torch.empty((S, M, P, 5), dtype=torch.float64, device=dev),
                       grad=torch.empty((S, P), dtype=torch.float64, device=dev))
        else:
            out = dict(tangents=np.empty((S, M, P, 5)), grad=np.empty((S, P)))
        self._check(self._lib.pbe_tangents(self._h, _ptr(out.get("tangents")), _ptr(out.get("grad")),
                                           1 if on_device else 0))
        return out

    def last_run_info(self) -> dict:
        info = RunInfo()
        self._check(self._lib.pbe_last_run_info(self._h, C.byref(info)))
        return info.as_dict()


def context_for(w, kernel: int = KERNEL_AUTO, device: int = 0, max_sims: Optional[int] = None) -> Context:
    """A Context shaped for workloads.Workload `w` (kinetics set)."""
    ctx = Context(w.N, w.dL, L_lo=w.L_lo, limiter=w.limiter, courant=w.courant, dt_fixed=w.dt_fixed,
                  dt_max=w.dt_max, max_steps=w.max_steps, n_steps=w.n_steps, rho_c=w.rho_c, k_v=w.k_v,
                  n_samples=w.M, n_tangents=w.n_tangents, max_sims=max_sims or w.n_sims, kernel=kernel,
                  device=device, n_bins2=getattr(w, "N2", 0), L2_lo=getattr(w, "L2_lo", 0.0),
                  dL2=getattr(w, "dL2", 0.0))
    ctx.set_kinetics(w.law, w.theta, w.sol_kind, w.sol, w.knot_t, w.knot_T, w.tangent_seed)
    return ctx


def run_workload(w, kernel: int = KERNEL_AUTO, device: int = 0, want_n: bool = True, host_n0: bool = False):
    """Runs workload `w` end to end on the GPU and returns host numpy arrays shaped like
    oracle.run(): samples, status, steps, loss, n_final (+ tsamples, grad, ndot_final)."""
    import torch
    dev = torch.device("cuda", device)
    ctx = context_for(w, kernel=kernel, device=device)
    n0 = w.n0 if host_n0 else torch.from_numpy(np.ascontiguousarray(w.n0)).to(dev)
    cells = w.N * max(getattr(w, "N2", 0), 1)
    nf = torch.empty((w.n_sims, cells), dtype=torch.float64, device=dev) if want_n else None
    ndf = (torch.empty((w.n_sims, w.n_tangents, w.N), dtype=torch.float64, device=dev)
           if (want_n and w.n_tangents) else None)
    ctx.run_batch(n0, w.c0, w.t_samples if w.n_steps == 0 else None, w.target, nf, ndf)
    out = ctx.moments()
    res = dict(samples=out["moments"], status=out["status"], steps=out["steps"], loss=out["loss"],
               info=ctx.last_run_info())
    if w.n_tangents:
        tg = ctx.tangents()
        res.update(tsamples=tg["tangents"], grad=tg["grad"])
    if want_n:
        res["n_final"] = nf.cpu().numpy()
        if ndf is not None:
            res["ndot_final"] = ndf.cpu().numpy()
    ctx.close()
    return res
