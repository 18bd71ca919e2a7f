"""Seeded synthetic inputs for the batched 1D PBE march (shared by tests, bench and smoke).

This module is the ONE place both the CUDA path and the CPU oracle take inputs from.
It holds no arithmetic of the method itself: no kinetics, no flux, no moments, no
mass balance.  It only builds arrays (seed distributions, parameter draws, sample
times, temperature knots) with the shapes of the paper's workloads (DESIGN.md
"Input recipe"), and hard-coded constants where an input value would otherwise need
the method's arithmetic (each such constant is re-derived by a test through the
oracle, tests/test_oracle_pins.py::test_workload_constants_rederived_through_oracle).

Paper sources for the shapes: Table 1 (Gaussian seed, mean 400 um,
sigma 30 um, m0 = 1 g/kg, c0 = 8 g/kg, T = 15 C, L_max = 1200 um, rho_c, k_v);
Table A.1 (L711-729: solubility and Arrhenius constants); App. B (L734-744: 9 in-silico
experiments, T in {10,15,20} C x S0 in {1.15,1.25,1.5}, 600 samples); eq-poly_growth_rate
(L565-571).  Configs C1-C5 are BASELINE.json "configs" in order.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

# enums (values mirror include/pbe.h; the oracle has its own copy of these small ints)
LIM_UPWIND, LIM_VANLEER, LIM_MINMOD, LIM_SUPERBEE, LIM_MC = 0, 1, 2, 3, 4
LAW_CONST, LAW_ARRHENIUS, LAW_POLY = 0, 1, 2
SOL_EXP, SOL_POLY = 0, 1

RHO_C = 1.11e-12          # g/um^3, Table 1 (L451)
K_V = math.pi / 4.0       # cylinder, Table 1 (L452)
NU = 0.9                  # Courant number (L301)

# Table A.1 (L717-727), dimension 1, with the dissolution branch mirrored (R-12)
ARRHENIUS_DEFAULT = (8.86e6, 2.45e3, 3.7, 8.86e6, 2.45e3, 3.7)
SOL_EXP_DEFAULT = (3.37, 0.036)
# R-13: 2nd-order Taylor expansion of 3.37 exp(0.036 T): (a, a b, a b^2 / 2)
SOL_POLY_DEFAULT = (3.37, 3.37 * 0.036, 3.37 * 0.036 * 0.036 / 2.0)

# c*(T) values needed as INPUTS (initial concentrations).  Hard-coded so this module
# holds no kinetics; tests/test_oracle_pins.py::test_workload_constants_rederived_through_oracle
# re-derives each through the oracle.
#   C2: c0 = c*_poly(15) = 3.37 + 0.12132*15 + 0.00218376*225
C2_C0 = 5.681146
#   C5 / App. B: c0 = S0 * 3.37 exp(0.036 T) for T in (10, 15, 20), S0 in (1.15, 1.25, 1.5)
APPB_T = (10.0, 15.0, 20.0)
APPB_S0 = (1.15, 1.25, 1.5)
APPB_CSAT = (4.8303201270683465, 5.782943125562973, 6.923439919869901)  # 3.37 exp(0.036 T)


@dataclass
class Workload:
    """Everything one pbe_run_batch call consumes (host numpy arrays)."""
    name: str
    N: int
    dL: float
    L_lo: float = 0.0
    limiter: int = LIM_VANLEER
    courant: float = NU
    dt_fixed: float = 0.0
    dt_max: float = math.inf
    max_steps: int = 10_000_000
    n_steps: int = 0                 # > 0: steps mode (exactly n_steps steps, one final sample)
    rho_c: float = RHO_C
    k_v: float = K_V
    law: int = LAW_ARRHENIUS
    theta: np.ndarray = None         # [S][P]
    sol_kind: int = SOL_EXP
    sol: np.ndarray = None           # [n_sol]
    knot_t: np.ndarray = None        # [K]
    knot_T: np.ndarray = None        # [S or 1][K]
    n0: np.ndarray = None            # [S or 1][N]
    c0: np.ndarray = None            # [S]
    t_samples: np.ndarray = None     # [M]
    target: Optional[np.ndarray] = None   # [S][M][2] (c, mean length)
    n_tangents: int = 0
    tangent_seed: Optional[np.ndarray] = None  # [n_tangents][P + n_sol]
    meta: dict = field(default_factory=dict)
    # 2D model (NEXT-1): N2 > 0 -> n0 rows hold N2 * N1 values (L1 fastest); theta = [dim 1 | dim 2]
    N2: int = 0
    dL2: float = 0.0
    L2_lo: float = 0.0

    @property
    def n_sims(self) -> int:
        return int(self.theta.shape[0])

    @property
    def n_params(self) -> int:
        return int(self.theta.shape[1])

    @property
    def M(self) -> int:
        return 1 if self.n_steps > 0 else int(self.t_samples.shape[0])

    def n0_for(self, s: int) -> np.ndarray:
        return self.n0[s if self.n0.shape[0] > 1 else 0]

    def subset(self, sims) -> "Workload":
        """The same workload restricted to the given simulation indices."""
        sims = np.asarray(sims, dtype=np.int64)
        pick = lambda a: None if a is None else (a[sims] if a.shape[0] > 1 else a)
        return replace(self, theta=self.theta[sims], n0=pick(self.n0), c0=self.c0[sims],
                       knot_T=pick(self.knot_T),
                       target=None if self.target is None else self.target[sims])


def bin_centers(N: int, dL: float, L_lo: float = 0.0) -> np.ndarray:
    return L_lo + (np.arange(N, dtype=np.float64) + 0.5) * dL


def gaussian_seed(N: int, dL: float, mean: float = 400.0, sigma: float = 30.0, m0: float = 1.0,
                  L_lo: float = 0.0, rho_c: float = RHO_C, k_v: float = K_V) -> np.ndarray:
    """Gaussian number density at bin centers (SI S1.3, L877-889), scaled ANALYTICALLY so
    that the continuous distribution has crystal mass rho_c k_v E[L^3] N_c = m0
    (E[L^3] = mean^3 + 3 mean sigma^2 for a normal).  The discrete midpoint mass matches
    m0 to ~1e-16 when sigma/dL >= 2.5 (pinned in tests)."""
    L = bin_centers(N, dL, L_lo)
    Nc = m0 / (rho_c * k_v * (mean ** 3 + 3.0 * mean * sigma ** 2))
    return Nc * np.exp(-0.5 * ((L - mean) / sigma) ** 2) / (sigma * math.sqrt(2.0 * math.pi))


def lognormal_seed(N: int, dL: float, mean: float = 400.0, sigma: float = 30.0, m0: float = 1.0,
                   L_lo: float = 0.0, rho_c: float = RHO_C, k_v: float = K_V) -> np.ndarray:
    """Log-normal number density at bin centers with the given mean and standard deviation of
    L ("Our framework supports normal and log-normal distributions for the
    seed PSSD"): ln L ~ N(mu_l, s_l^2), s_l^2 = ln(1 + sigma^2/mean^2), mu_l = ln(mean) - s_l^2/2,
    raw moments E[L^k] = exp(k mu_l + k^2 s_l^2 / 2); scaled analytically to crystal mass
    rho_c k_v E[L^3] N_c = m0 like gaussian_seed."""
    L = bin_centers(N, dL, L_lo)
    s2 = math.log1p((sigma / mean) ** 2)
    mu = math.log(mean) - 0.5 * s2
    EL3 = math.exp(3.0 * mu + 4.5 * s2)
    Nc = m0 / (rho_c * k_v * EL3)
    out = np.zeros(N)
    pos = L > 0.0
    Lp = L[pos]
    out[pos] = Nc * np.exp(-0.5 * (np.log(Lp) - mu) ** 2 / s2) / (Lp * math.sqrt(2.0 * math.pi * s2))
    return out


def _target(c0: np.ndarray, t: np.ndarray, L0: float = 400.0) -> np.ndarray:
    """Synthetic measured trace shaped like App. B's (L743): concentration relaxing
    toward saturation and mean crystal length increasing.  Closed-form shapes, not a
    model solution; only the loss epilogue (row a7) consumes it."""
    S, M = c0.shape[0], t.shape[0]
    out = np.empty((S, M, 2))
    decay = np.exp(-t / 100.0)
    out[:, :, 0] = c0[:, None] * (0.75 + 0.25 * decay[None, :])
    out[:, :, 1] = L0 + 150.0 * (1.0 - decay[None, :])
    return out


_APPB = None


def appb_target(e: np.ndarray, t: np.ndarray, c0: np.ndarray) -> np.ndarray:
    """App. B "measurements" for experiments e (0..8) at sample times t: (c, mu1/mu0) of the
    1D method of moments with the Arrhenius truth, precomputed at
    t = 1, 2, ..., 600 min by tools/gen_appb_targets.py (workloads/data/appb_targets.npy).
    Sample grids that are not a subset of that grid fall back to the closed-form _target."""
    global _APPB
    if _APPB is None:
        _APPB = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "appb_targets.npy"))
    idx = np.rint(t).astype(np.int64) - 1
    if not (np.all(np.abs(t - (idx + 1)) == 0.0) and idx.min() >= 0 and idx.max() < _APPB.shape[1]):
        return _target(c0, t)
    return _APPB[np.asarray(e)][:, idx, :].copy()


# ------------------------------------------------------------------------------------
# BASELINE.json configs
# ------------------------------------------------------------------------------------
def c1_growth(limiter: int = LIM_VANLEER, N: int = 100, M: int = 100) -> Workload:
    """C1: 100 bins, constant size-independent G = 0.5 um/min, fixed dt = 1 min,
    1000 steps (t_max = 1000 min), Gaussian seed (m0 = 0.5), c0 = 8."""
    dL = 1200.0 / N
    return Workload(
        name=f"c1_growth_{'vanleer' if limiter else 'upwind'}_N{N}", N=N, dL=dL, limiter=limiter,
        dt_fixed=1.0, law=LAW_CONST, theta=np.array([[0.5]]),
        sol_kind=SOL_EXP, sol=np.array(SOL_EXP_DEFAULT),
        knot_t=np.array([0.0]), knot_T=np.array([[15.0]]),
        n0=gaussian_seed(N, dL, m0=0.5)[None, :], c0=np.array([8.0]),
        t_samples=np.linspace(1000.0 / M, 1000.0, M))


def c2_dissolution(N: int = 1000, t_max: float = 600.0, M: int = 600, dt_max: float = 0.1) -> Workload:
    """C2: 1000 bins, dissolution (S < 1 after heating), polynomial c*(T) (R-13),
    T ramps 15 -> 25 C over 120 min then holds, c0 = c*(15), m0 = 3, dt_max = 0.1."""
    dL = 1200.0 / N
    return Workload(
        name=f"c2_dissolution_N{N}", N=N, dL=dL, dt_max=dt_max,
        law=LAW_ARRHENIUS, theta=np.array([ARRHENIUS_DEFAULT]),
        sol_kind=SOL_POLY, sol=np.array(SOL_POLY_DEFAULT),
        knot_t=np.array([0.0, 120.0, 600.0]), knot_T=np.array([[15.0, 25.0, 25.0]]),
        n0=gaussian_seed(N, dL, m0=3.0)[None, :], c0=np.array([C2_C0]),
        t_samples=np.linspace(t_max / M, t_max, M))


def c3_cycling(N: int = 1000, t_max: float = 1000.0, M: int = 1000, dt_max: float = 0.01) -> Workload:
    """C3: 1000 bins, van Leer, triangle T(t) 15 <-> 25 C with period 200 min,
    c0 = 8, m0 = 1, dt_max = 0.01 -> exactly 10^5 capped steps over 1000 min."""
    dL = 1200.0 / N
    kt = np.arange(0.0, t_max + 1e-9, 100.0)
    kT = np.where((np.arange(kt.shape[0]) % 2) == 0, 15.0, 25.0)
    return Workload(
        name=f"c3_cycling_N{N}", N=N, dL=dL, dt_max=dt_max,
        law=LAW_ARRHENIUS, theta=np.array([ARRHENIUS_DEFAULT]),
        sol_kind=SOL_EXP, sol=np.array(SOL_EXP_DEFAULT),
        knot_t=kt, knot_T=kT[None, :],
        n0=gaussian_seed(N, dL, m0=1.0)[None, :], c0=np.array([8.0]),
        t_samples=np.linspace(t_max / M, t_max, M))


def c4_sweep(N: int, batch: int = 1, n_steps: int = 1000, seed: int = 2411) -> Workload:
    """C4: bin-count sweep, dL = 1200/N, van Leer, base-case Arrhenius growth at 15 C,
    c0 = 8, m0 = 1, exactly n_steps uncapped CFL steps (C = 0.9).  batch > 1 perturbs
    k_g by U(0.8, 1.2) (numpy PCG64 seed 2411); all sims share one n0 row."""
    dL = 1200.0 / N
    rng = np.random.Generator(np.random.PCG64(seed))
    th = np.tile(np.array(ARRHENIUS_DEFAULT), (batch, 1))
    if batch > 1:
        th[:, 0] *= rng.uniform(0.8, 1.2, size=batch)
    return Workload(
        name=f"c4_sweep_N{N}_b{batch}", N=N, dL=dL, n_steps=n_steps,
        law=LAW_ARRHENIUS, theta=th, sol_kind=SOL_EXP, sol=np.array(SOL_EXP_DEFAULT),
        knot_t=np.array([0.0]), knot_T=np.array([[15.0]]),
        n0=gaussian_seed(N, dL, m0=1.0)[None, :], c0=np.full(batch, 8.0),
        t_samples=np.array([1.0]))


POLY_A = (0.5, 5.0, 20.0, 50.0, 50.0, 20.0, 5.0, 0.5)   # um/min, k = 8


def c5_ensemble(n_sims: int = 4096, N: int = 2000, t_max: float = 600.0, M: int = 600,
                dt_max: float = 0.05, n_tangents: int = 8, seed: int = 241100742) -> Workload:
    """C5: ensemble of kinetic parameter sets with forward-mode tangents.
    Polynomial growth (k = 8) theta_{s,j} = A_j exp(0.25 z_{s,j}), z ~ N(0,1) (PCG64);
    sim s runs App. B experiment e = s mod 9: T = (10,15,20)[e // 3], S0 = (1.15,1.25,1.5)[e % 3],
    c0 = S0 c*(T); m0 = 1; 600 samples over 600 min; dt_max = 0.05; tangents e_1..e_8."""
    dL = 1200.0 / N
    rng = np.random.Generator(np.random.PCG64(seed))
    z = rng.standard_normal((n_sims, len(POLY_A)))
    theta = np.array(POLY_A)[None, :] * np.exp(0.25 * z)
    e = np.arange(n_sims) % 9
    T = np.array(APPB_T)[e // 3]
    c0 = np.array(APPB_S0)[e % 3] * np.array(APPB_CSAT)[e // 3]
    t = np.linspace(t_max / M, t_max, M)
    return Workload(
        name=f"c5_ensemble_S{n_sims}_N{N}", N=N, dL=dL, dt_max=dt_max,
        law=LAW_POLY, theta=theta, sol_kind=SOL_EXP, sol=np.array(SOL_EXP_DEFAULT),
        knot_t=np.array([0.0]), knot_T=T[:, None].copy(),
        n0=gaussian_seed(N, dL, m0=1.0)[None, :], c0=c0, t_samples=t,
        target=appb_target(e, t, c0), n_tangents=n_tangents)


def next3_estimation(n_params: int = 1000, N: int = 2000, t_max: float = 600.0, M: int = 600,
                     dt_max: float = 0.05, seed: int = 599) -> Workload:
    """NEXT-3: the paper's parameter-estimation regime with many parameters (L565-572: the
    polynomial is lengthened to raise the parameter count; L599: 1000 parameters).  The 9 App-B
    experiments (L734-744), one simulation each, POLY growth with a_1..a_8 = POLY_A and
    a_9..a_n drawn U(0, 0.05) (PCG64 `seed`), C5's grid and clock, target as C5."""
    dL = 1200.0 / N
    rng = np.random.Generator(np.random.PCG64(seed))
    theta = np.zeros((9, n_params))
    k = min(n_params, len(POLY_A))
    theta[:, :k] = np.array(POLY_A)[:k]
    if n_params > k:
        theta[:, k:] = 0.05 * rng.random((9, n_params - k))
    e = np.arange(9)
    T = np.array(APPB_T)[e // 3]
    c0 = np.array(APPB_S0)[e % 3] * np.array(APPB_CSAT)[e // 3]
    t = np.linspace(t_max / M, t_max, M)
    return Workload(
        name=f"next3_estimation_P{n_params}_N{N}", N=N, dL=dL, dt_max=dt_max, max_steps=int(1.2 * t_max / dt_max) + 1000,
        law=LAW_POLY, theta=theta, sol_kind=SOL_EXP, sol=np.array(SOL_EXP_DEFAULT),
        knot_t=np.array([0.0]), knot_T=T[:, None].copy(),
        n0=gaussian_seed(N, dL, m0=1.0)[None, :], c0=c0, t_samples=t, target=appb_target(e, t, c0))


CONFIGS = {
    "c1": c1_growth,
    "c2": c2_dissolution,
    "c3": c3_cycling,
    "c4": c4_sweep,
    "c5": c5_ensemble,
}


# Table A.1 (L722-727): growth-rate constants for the two crystal dimensions (growth only)
ARRHENIUS_2D = (8.86e6, 2.45e3, 3.7, 4.088e5, 2.4e3, 2.5)


def gaussian_seed_2d(N1: int, dL1: float, N2: int, dL2: float, mean=(400.0, 250.0), sigma=(30.0, 30.0),
                     m0: float = 1.0, rho_c: float = RHO_C, k_v: float = K_V) -> np.ndarray:
    """Bivariate normal seed with independent marginals (Table 1) at cell centers,
    scaled analytically to crystal mass rho_c k_v E[L1 L2^2] N_c = m0 (SI S1.3, L887);
    returns [N2][N1] flattened (L1 fastest)."""
    L1 = bin_centers(N1, dL1)
    L2 = bin_centers(N2, dL2)
    Nc = m0 / (rho_c * k_v * mean[0] * (mean[1] ** 2 + sigma[1] ** 2))
    g1 = np.exp(-0.5 * ((L1 - mean[0]) / sigma[0]) ** 2) / (sigma[0] * math.sqrt(2 * math.pi))
    g2 = np.exp(-0.5 * ((L2 - mean[1]) / sigma[1]) ** 2) / (sigma[1] * math.sqrt(2 * math.pi))
    return (Nc * np.outer(g2, g1)).reshape(-1)


def c2d_base(N1: int = 1200, N2: int = 600, t_max: float = 10.0, M: int = 10, n_sims: int = 1,
             dt_max: float = math.inf, limiter: int = LIM_VANLEER) -> Workload:
    """NEXT-1 / Table 1 base case: 2D PSSD on L1 in [0, 1200] x L2 in [0, 600] um, Gaussian seed
    (400, 250) um, sigma 30 um, m0 = 1 g/kg, c0 = 8 g/kg, T = 15 C, Arrhenius growth for both
    dimensions (Table A.1), CFL nu = 0.9 over both dimensions (SI L859)."""
    dL1, dL2 = 1200.0 / N1, 600.0 / N2
    return Workload(
        name=f"c2d_base_{N1}x{N2}", N=N1, dL=dL1, N2=N2, dL2=dL2, limiter=limiter, dt_max=dt_max,
        law=LAW_ARRHENIUS, theta=np.tile(np.array(ARRHENIUS_2D), (n_sims, 1)),
        sol_kind=SOL_EXP, sol=np.array(SOL_EXP_DEFAULT),
        knot_t=np.array([0.0]), knot_T=np.array([[15.0]]),
        n0=gaussian_seed_2d(N1, dL1, N2, dL2)[None, :], c0=np.full(n_sims, 8.0),
        t_samples=np.linspace(t_max / M, t_max, M))
