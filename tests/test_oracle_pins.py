"""Pins for the CPU oracle: every check compares oracle/ against
something other than itself — paper-printed values, closed forms, high-precision
independent evaluation, exact-rational brute force, conservation/positivity theorems,
the method of moments and the complex-step derivative.  CPU only."""
import json
import math
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import oracle
import workloads as W
from tests import exact_march as X

HERE = os.path.dirname(os.path.abspath(__file__))


def _small(**kw):
    """A small single-simulation workload (defaults: 10 bins, van Leer, const G)."""
    base = dict(name="small", N=10, dL=1.0, law=W.LAW_CONST, theta=np.array([[0.5]]),
                sol_kind=W.SOL_POLY, sol=np.array([3.0, 0.0, 0.0]), knot_t=np.array([0.0]),
                knot_T=np.array([[15.0]]), n0=None, c0=np.array([8.0]), t_samples=np.array([1.0]))
    base.update(kw)
    return W.Workload(**base)


# ------------------------------------------------------------------------------------
# PIN-15: SI Tables S1-S2 (paper-printed worked example) pin the Dual arithmetic
# ------------------------------------------------------------------------------------
def test_pin15_si_table_dual_arithmetic():
    g = json.load(open(os.path.join(HERE, "golden", "si_tables_s1_s2.json")))
    x1, x2 = g["x"]
    y1, y2, dy1_dx1, dy2_dx1 = oracle.dual_si_example(x1, x2, 1.0, 0.0)
    _, _, dy1_dx2, dy2_dx2 = oracle.dual_si_example(x1, x2, 0.0, 1.0)
    d = g["decimals"]
    assert round(y1, d) == g["primal_printed"]["y1"] and round(y2, d) == g["primal_printed"]["y2"]
    J = [[dy1_dx1, dy1_dx2], [dy2_dx1, dy2_dx2]]
    for r in range(2):
        for c in range(2):
            assert round(J[r][c], d) == pytest.approx(g["jacobian_printed"][r][c], abs=1e-12)
    # the symbolic Jacobian printed at L970-979
    s = x1 + x2
    Jsym = [[(s * math.cos(x1) - math.sin(x1)) / s ** 2, -math.sin(x1) / s ** 2],
            [math.exp(x2), (s + 1) * math.exp(x2)]]
    assert np.allclose(J, Jsym, rtol=1e-15, atol=0)


# ------------------------------------------------------------------------------------
# PIN-1: kinetics scalars vs closed forms and 50-digit evaluation
# ------------------------------------------------------------------------------------
mp = mpmath.mp.clone()
mp.dps = 50


def _w_exp(T=15.0, law=W.LAW_ARRHENIUS, theta=W.ARRHENIUS_DEFAULT):
    return _small(law=law, theta=np.array([theta]), sol_kind=W.SOL_EXP, sol=np.array(W.SOL_EXP_DEFAULT),
                  knot_T=np.array([[T]]))


def test_pin1_solubility_special_case_T0():
    w = _w_exp(T=0.0)
    T, cs, S, G = oracle.kinetics(w, W.ARRHENIUS_DEFAULT, 0.0, 8.0)
    assert T == 0.0 and cs == 3.37            # exp(0) = 1: c*(0) = a (Table A.1)


@pytest.mark.parametrize("T", [10.0, 15.0, 20.0, 25.0])
def test_pin1_kinetics_vs_50_digits(T):
    w = _w_exp(T=T)
    c = 8.0
    Tk, cs, S, G = oracle.kinetics(w, W.ARRHENIUS_DEFAULT, 3.0, c)
    cs_ref = mp.mpf("3.37") * mp.exp(mp.mpf("0.036") * T)
    S_ref = c / cs_ref
    k1, k2, k3 = (mp.mpf(repr(x)) for x in W.ARRHENIUS_DEFAULT[:3])
    G_ref = (k1 * mp.exp(-k2 / (T + mp.mpf("273.15"))) * (S_ref - 1) ** k3) if S_ref > 1 else (
        -(k1 * mp.exp(-k2 / (T + mp.mpf("273.15"))) * (1 - S_ref) ** k3))
    assert Tk == T
    assert cs == pytest.approx(float(cs_ref), rel=2e-16)
    assert S == pytest.approx(float(S_ref), rel=4e-16)
    assert G == pytest.approx(float(G_ref), rel=2e-14)


# R-12 dissolution constants deliberately different from the growth constants, so a branch that
# reads theta[0..2] instead of theta[3..5] (or mixes them) is caught
ARRH_DISTINCT = (8.86e6, 2.45e3, 3.7, 2.0e5, 2.0e3, 1.5)


@pytest.mark.parametrize("T", [10.0, 25.0])
@pytest.mark.parametrize("c", [8.0, 4.0, 5.5])
def test_pin1_dissolution_branch_own_parameters_vs_50_digits(T, c):
    # Eq. A.2 for S > 1 with (kg, Eg, g) = theta[0..2]; R-12 for S < 1 with (kd, Ed, d) = theta[3..5]
    w = _w_exp(T=T, theta=ARRH_DISTINCT)
    Tk, cs, S, G = oracle.kinetics(w, ARRH_DISTINCT, 0.0, c)
    cs_ref = mp.mpf("3.37") * mp.exp(mp.mpf("0.036") * T)
    S_ref = c / cs_ref
    k = [mp.mpf(repr(x)) for x in ARRH_DISTINCT]
    if S_ref > 1:
        G_ref = k[0] * mp.exp(-k[1] / (T + mp.mpf("273.15"))) * (S_ref - 1) ** k[2]
    else:
        G_ref = -(k[3] * mp.exp(-k[4] / (T + mp.mpf("273.15"))) * (1 - S_ref) ** k[5])
    assert (S > 1) == (S_ref > 1)
    assert G == pytest.approx(float(G_ref), rel=2e-14)


def test_pin1_base_case_growth_value():
    # Table 1 base case: T = 15 C, c0 = 8 -> S0 = 1.38338, G(S0) = 51.79 um/min
    T, cs, S, G = oracle.kinetics(_w_exp(), W.ARRHENIUS_DEFAULT, 0.0, 8.0)
    assert S == pytest.approx(1.383379, abs=1e-6)
    assert G == pytest.approx(51.79182, abs=1e-4)


def test_pin1_growth_zero_at_saturation_and_branches():
    w = _w_exp()
    cs = oracle.kinetics(w, W.ARRHENIUS_DEFAULT, 0.0, 1.0)[1]
    assert oracle.kinetics(w, W.ARRHENIUS_DEFAULT, 0.0, cs)[3] == 0.0          # S = 1
    # growth-only Arrhenius (3 params): S < 1 -> 0 (Eq. A.2 "only applies when S exceeds one")
    w3 = _w_exp(theta=W.ARRHENIUS_DEFAULT[:3])
    assert oracle.kinetics(w3, W.ARRHENIUS_DEFAULT[:3], 0.0, 0.9 * cs)[3] == 0.0
    # dissolution branch (R-12) is the odd extension for the default parameters
    Gp = oracle.kinetics(w, W.ARRHENIUS_DEFAULT, 0.0, 1.1 * cs)[3]
    Gm = oracle.kinetics(w, W.ARRHENIUS_DEFAULT, 0.0, 0.9 * cs)[3]
    assert Gp > 0 and Gm == pytest.approx(-Gp, rel=1e-12)


def test_pin1_polynomial_growth_and_solubility():
    # eq-poly_growth_rate with a = [2, 3] at S = 1.2: 2*0.2 + 3*0.04 = 0.52 (closed form)
    w = _small(law=W.LAW_POLY, theta=np.array([[2.0, 3.0]]), sol=np.array([1.0, 0.0, 0.0]))
    assert oracle.kinetics(w, [2.0, 3.0], 0.0, 1.2)[3] == pytest.approx(0.52, rel=1e-15)
    assert oracle.kinetics(w, [2.0, 3.0], 0.0, 0.8)[3] == 0.0
    # R-13 polynomial solubility with the Taylor coefficients: c*(15) = 5.681146
    w2 = _small(sol=np.array(W.SOL_POLY_DEFAULT))
    assert oracle.kinetics(w2, [0.5], 0.0, 1.0)[1] == pytest.approx(5.681146, rel=1e-15)


def test_pin1_temperature_profile_piecewise_linear():
    w = _small(knot_t=np.array([0.0, 120.0, 600.0]), knot_T=np.array([[15.0, 25.0, 25.0]]))
    Ts = [oracle.kinetics(w, [0.5], t, 8.0)[0] for t in (-1.0, 0.0, 60.0, 90.0, 120.0, 300.0, 700.0)]
    assert Ts == [15.0, 15.0, 20.0, 22.5, 25.0, 25.0, 25.0]


def test_workload_constants_rederived_through_oracle():
    # workloads/ hard-codes c* values so it holds no kinetics; re-derive them here
    for T, cs in zip(W.APPB_T, W.APPB_CSAT):
        assert oracle.kinetics(_w_exp(T=T), W.ARRHENIUS_DEFAULT, 0.0, 1.0)[1] == pytest.approx(cs, rel=1e-15)
    w2 = _small(sol=np.array(W.SOL_POLY_DEFAULT))
    assert oracle.kinetics(w2, [0.5], 0.0, 1.0)[1] == pytest.approx(W.C2_C0, rel=1e-15)
    # the estimation driver's copy of the same table (product code evaluates no kinetics)
    from paper_2411_00742_b200 import estimate as E
    assert E.APPB_CSAT == W.APPB_CSAT and E.APPB_T == W.APPB_T and E.SOL_DEFAULT == W.SOL_EXP_DEFAULT


# ------------------------------------------------------------------------------------
# PIN-2/3/4/6/8: the sweep in isolation
# ------------------------------------------------------------------------------------
def _rand_profile(rng, N):
    f = rng.random(N) * (rng.random(N) < 0.8)
    f[:2] = 0.0
    return f


ALL_LIMS = [W.LIM_UPWIND, W.LIM_VANLEER, W.LIM_MINMOD, W.LIM_SUPERBEE, W.LIM_MC]


@pytest.mark.parametrize("lim", ALL_LIMS)
def test_pin3_zero_courant_is_identity(lim):
    f = _rand_profile(np.random.default_rng(1), 40)
    assert np.array_equal(oracle.sweep(f, 0.0, lim), f)


@pytest.mark.parametrize("lim", ALL_LIMS)
def test_pin4_courant_one_is_exact_shift(lim):
    f = _rand_profile(np.random.default_rng(2), 50)
    out = oracle.sweep(f, 1.0, lim)
    assert np.array_equal(out[1:], f[:-1]) and out[0] == 0.0
    out = oracle.sweep(f, -1.0, lim)
    assert np.array_equal(out[:-1], f[1:]) and out[-1] == 0.0


@pytest.mark.parametrize("lim", [W.LIM_MINMOD, W.LIM_SUPERBEE, W.LIM_MC])
def test_pin2_extra_limiters_phi_values(lim):
    """phi(theta) of the NEXT-4 limiters at closed-form points, read off one face: with
    f = (0, 0, p, p + 1, 0...) the face between bins 2 and 3 has d_2 = p, d_3 = 1, i.e.
    theta = p, and the flux difference isolates phi(p) (C = 1/2, kappa = 1/8)."""
    table = {W.LIM_MINMOD: {0.25: 0.25, 0.5: 0.5, 1.0: 1.0, 2.0: 1.0, 3.0: 1.0},
             W.LIM_SUPERBEE: {0.25: 0.5, 0.5: 1.0, 1.0: 1.0, 1.5: 1.5, 2.0: 2.0, 3.0: 2.0},
             W.LIM_MC: {0.25: 0.5, 0.5: 0.75, 1.0: 1.0, 2.0: 1.5, 3.0: 2.0}}[lim]
    for p, phi in table.items():
        f = np.array([0.0, 0.0, p, p + 1.0, 0.0, 0.0, 0.0])
        up = oracle.sweep(f, 0.5, W.LIM_UPWIND)
        out = oracle.sweep(f, 0.5, lim)
        # bin 3 gains F_{3-1/2} - F_{3+1/2}; the limited part of F_{3-1/2} is kappa phi(p) * 1
        # and F_{3+1/2} has theta = 1/(-(p+1)) < 0 -> no limited part
        assert (out[3] - up[3]) == pytest.approx(0.125 * phi, rel=1e-14, abs=1e-15), (p, phi)


def test_pin2_vanleer_values_through_sweep():
    # f = (0, 1, 2, 3, ...): theta = 1 in the interior -> phi = 1 -> Lax-Wendroff, which is
    # exact for linear data: f_i - C * slope.  Check interior bins (away from ghosts).
    f = np.arange(12, dtype=np.float64)
    C = 0.25
    out = oracle.sweep(f, C, W.LIM_VANLEER)
    assert np.allclose(out[2:-2], f[2:-2] - C, rtol=0, atol=1e-15)
    # f with theta = 3 at face 3-1/2: phi(3) = 1.5; theta = -1 -> phi = 0 (SPEC examples)
    # pinned in exact arithmetic by the brute-force comparison below.


@pytest.mark.parametrize("seed", range(20))
def test_pin9_sweep_matches_exact_flux_form(seed):
    rng = np.random.default_rng(100 + seed)
    N = 10
    f = [Fraction(int(x), 7) for x in rng.integers(0, 50, N)]
    C = Fraction(int(rng.integers(-9, 10)), 10)
    for lim in (0, 1, 2, 3, 4):
        exact = X.flux_step(f, C, lim)
        got = oracle.sweep(np.array([float(x) for x in f]), float(C), lim)
        scale = float(max(f)) or 1.0
        assert np.max(np.abs(got - np.array([float(x) for x in exact]))) <= 1e-15 * scale


@pytest.mark.parametrize("lim", ALL_LIMS[1:])
@pytest.mark.parametrize("seed", range(10))
def test_pin6_mirror_identity(seed, lim):
    rng = np.random.default_rng(200 + seed)
    f = _rand_profile(rng, 30)
    C = float(rng.uniform(0, 1))
    a = oracle.sweep(f, -C, lim)
    b = oracle.sweep(f[::-1].copy(), C, lim)[::-1]
    assert np.array_equal(a, b)


@pytest.mark.parametrize("lim", ALL_LIMS[1:])
@pytest.mark.parametrize("seed", range(30))
def test_pin8_positivity_and_tvd(seed, lim):
    """All limiters lie in Sweby's TVD region (0 <= phi <= min(2 theta, 2)), so the sweep is
    positivity preserving and total-variation diminishing for |C| <= 1."""
    rng = np.random.default_rng(300 + seed)
    f = _rand_profile(rng, 64) * 10.0 ** rng.uniform(-5, 5)
    C = float(rng.uniform(-1, 1))
    out = oracle.sweep(f, C, lim)
    tv = lambda v: np.sum(np.abs(np.diff(np.concatenate([[0, 0], v, [0, 0]]))))
    assert out.min() >= -1e-12 * f.max()
    assert tv(out) <= tv(f) * (1 + 1e-12)


# ------------------------------------------------------------------------------------
# PIN-9: full coupled march vs exact rational / 50-digit brute force on 10-bin meshes
# ------------------------------------------------------------------------------------
def _exact_args(w, s=0):
    return dict(N=w.N, dL=w.dL, L_lo=w.L_lo, limiter=w.limiter, courant=w.courant, dt_fixed=w.dt_fixed,
                dt_max=None if math.isinf(w.dt_max) else w.dt_max, law=w.law, theta=list(w.theta[s]),
                sol_kind=w.sol_kind, sol=list(w.sol), knot_t=list(w.knot_t), knot_T=list(w.knot_T[0]),
                n0=list(w.n0_for(s)), c0=w.c0[s], rho_c=w.rho_c, k_v=w.k_v,
                t_samples=list(w.t_samples), n_steps=w.n_steps)


def _compare_exact(w, num, rtol):
    r = oracle.run(w)
    recs, n_ex, steps = X.march(num, **_exact_args(w))
    assert r["status"][0] == 0 and r["steps"][0] == steps
    ex = np.array([[float(v) for v in rec] for rec in recs])
    assert np.allclose(r["samples"][0], ex, rtol=rtol, atol=0)
    n_ex = np.array([float(v) for v in n_ex])
    assert np.max(np.abs(r["n_final"][0] - n_ex)) <= rtol * np.max(np.abs(n_ex))


def _int_seed(rng, N):
    return np.array([float(x) for x in rng.integers(0, 40, N)], dtype=np.float64) * 0.5


@pytest.mark.parametrize("lim", [0, 1])
@pytest.mark.parametrize("G", [0.5, -0.5])
def test_pin9_const_growth_fixed_dt_exact(lim, G):
    rng = np.random.default_rng(7)
    n0 = _int_seed(rng, 10)
    n0[:2] = 0; n0[-2:] = 0
    w = _small(limiter=lim, theta=np.array([[G]]), dt_fixed=0.5, n0=n0[None, :],
               rho_c=1e-3, k_v=0.5, t_samples=np.array([0.5, 1.0, 1.5, 2.0]))
    _compare_exact(w, X.Num("fraction"), 1e-14)


@pytest.mark.parametrize("lim", [0, 1])
def test_pin9_poly_kinetics_cfl_coupled_exact(lim):
    # polynomial growth + polynomial solubility + CFL steps + sample landing + mass coupling:
    # every quantity stays rational.
    rng = np.random.default_rng(11)
    n0 = _int_seed(rng, 10)
    n0[:2] = 0
    w = _small(limiter=lim, law=W.LAW_POLY, theta=np.array([[0.5, 0.25]]),
               sol=np.array([2.0, 0.125, 0.0]), knot_t=np.array([0.0, 4.0]), knot_T=np.array([[0.0, 8.0]]),
               n0=n0[None, :], c0=np.array([4.0]), rho_c=1e-4, k_v=0.5,
               t_samples=np.array([0.75, 1.5]))
    _compare_exact(w, X.Num("fraction"), 1e-13)


@pytest.mark.parametrize("theta", [W.ARRHENIUS_DEFAULT, ARRH_DISTINCT])
@pytest.mark.parametrize("c0", [8.0, 4.0])
def test_pin9_arrhenius_growth_dissolution_50_digits(c0, theta):
    # exp-based kinetics (Eq. A.2 + R-12 dissolution), exponential solubility, dt_max cap,
    # time-varying T: brute force at 50 digits.  c0 = 4 < c*(15) -> dissolution.
    rng = np.random.default_rng(5)
    n0 = _int_seed(rng, 10) * 1e3
    w = _small(law=W.LAW_ARRHENIUS, theta=np.array([theta]), sol_kind=W.SOL_EXP,
               sol=np.array(W.SOL_EXP_DEFAULT), knot_t=np.array([0.0, 0.1]), knot_T=np.array([[15.0, 25.0]]),
               n0=n0[None, :], c0=np.array([c0]), dL=10.0, dt_max=0.02,
               t_samples=np.array([0.05, 0.1]))
    _compare_exact(w, X.Num("mp"), 1e-13)


def test_pin9_steps_mode_uncapped_cfl_exact():
    rng = np.random.default_rng(3)
    n0 = _int_seed(rng, 10)
    w = _small(law=W.LAW_POLY, theta=np.array([[1.0]]), sol=np.array([2.0, 0.0, 0.0]), n0=n0[None, :],
               c0=np.array([3.0]), rho_c=1e-4, k_v=1.0, n_steps=4)
    _compare_exact(w, X.Num("fraction"), 1e-13)


# ------------------------------------------------------------------------------------
# PIN-5 / PIN-7: upwind discrete-moment recurrence and conservation on C1 (full size)
# ------------------------------------------------------------------------------------
@pytest.mark.parametrize("G", [0.5, -0.5])
def test_pin5_upwind_moment_recurrence(G):
    w = W.c1_growth(W.LIM_UPWIND, M=1000)
    w.theta = np.array([[G]])
    w.t_samples = w.t_samples[:60]             # 60 steps: boundary outflow < 1e-20 relative
    r = oracle.run(w)
    smp = r["samples"][0]
    mu0_init = oracle.moments(w, w.n0[0])
    mu = np.vstack([mu0_init, smp[:, 2:6]])
    gdt, dL, s = G * 1.0, w.dL, np.sign(G)
    d = np.diff(mu, axis=0)
    pred1 = gdt * mu[:-1, 0]
    pred2 = gdt * (2 * mu[:-1, 1] + s * dL * mu[:-1, 0])
    pred3 = gdt * (3 * mu[:-1, 2] + 3 * s * dL * mu[:-1, 1] + dL ** 2 * mu[:-1, 0])
    assert np.max(np.abs(d[:, 0])) <= 1e-13 * mu[0, 0]
    assert np.allclose(d[:, 1], pred1, rtol=1e-11)
    assert np.allclose(d[:, 2], pred2, rtol=1e-10)
    assert np.allclose(d[:, 3], pred3, rtol=1e-10)
    # upwind numerical diffusion: Var += |G| dt dL (1 - |C|) per step (exact, SURVEY PIN-5)
    var = mu[:, 2] / mu[:, 0] - (mu[:, 1] / mu[:, 0]) ** 2
    C = abs(G) / dL
    assert np.allclose(np.diff(var), abs(G) * dL * (1 - C), rtol=1e-7)
    # mass coupling: c^{n+1} - c^n = -rho k_v (mu3^{n+1} - mu3^n)
    cs = np.concatenate([[w.c0[0]], smp[:, 1]])
    assert np.allclose(np.diff(cs), -w.rho_c * w.k_v * d[:, 3], rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("make", [lambda: W.c1_growth(W.LIM_VANLEER),
                                  lambda: W.c2_dissolution(t_max=120.0, M=120),
                                  lambda: W.c3_cycling(N=300, t_max=200.0, M=200, dt_max=0.02)])
def test_pin7_conservation(make):
    w = make()
    r = oracle.run(w)
    assert r["status"][0] == 0
    smp = r["samples"][0]
    mu_init = oracle.moments(w, w.n0[0])
    # number: no boundary flux while the distribution is far from both ends
    assert np.max(np.abs(smp[:, 2] - mu_init[0])) <= 1e-12 * mu_init[0]
    # solute + crystal mass: c + rho_c k_v mu3 is invariant (eq-discrete_mass_balance)
    inv = smp[:, 1] + w.rho_c * w.k_v * smp[:, 5]
    inv0 = w.c0[0] + w.rho_c * w.k_v * mu_init[3]
    assert np.max(np.abs(inv - inv0)) <= 1e-12 * inv0
    assert np.all(r["n_final"][0] >= 0)


# ------------------------------------------------------------------------------------
# PIN-10: the discrete seed moments are the Gaussian's raw moments (spectral accuracy)
# ------------------------------------------------------------------------------------
@pytest.mark.parametrize("N", [100, 1000, 2000])
def test_pin10_seed_moments(N):
    w = W.c4_sweep(N)
    mu = oracle.moments(w, w.n0[0])
    m, s = 400.0, 30.0
    assert mu[1] / mu[0] == pytest.approx(m, rel=1e-14)
    assert mu[2] / mu[0] == pytest.approx(m * m + s * s, rel=1e-14)
    assert mu[3] / mu[0] == pytest.approx(m ** 3 + 3 * m * s * s, rel=1e-14)
    assert W.RHO_C * W.K_V * mu[3] == pytest.approx(1.0, rel=1e-14)


@pytest.mark.parametrize("N,mean,sigma", [(1000, 400.0, 30.0), (2000, 300.0, 40.0)])   # tails beyond 1200 um < 1e-20
def test_pin10_lognormal_seed_moments(N, mean, sigma):
    """Log-normal seed (L882-883): the discrete moments are the log-normal raw moments
    E[L^k] = exp(k mu_l + k^2 s_l^2 / 2), with mean and std of L as given."""
    dL = 1200.0 / N
    n0 = W.lognormal_seed(N, dL, mean=mean, sigma=sigma)
    w = W.replace(W.c4_sweep(N), n0=n0[None, :])
    mu = oracle.moments(w, n0)
    s2 = math.log1p((sigma / mean) ** 2)
    ml = math.log(mean) - 0.5 * s2
    raw = [math.exp(k * ml + 0.5 * k * k * s2) for k in range(4)]
    assert mu[1] / mu[0] == pytest.approx(mean, rel=1e-13)
    assert mu[2] / mu[0] - (mu[1] / mu[0]) ** 2 == pytest.approx(sigma ** 2, rel=1e-9)
    for k in (2, 3):
        assert mu[k] / mu[0] == pytest.approx(raw[k], rel=1e-13)
    assert W.RHO_C * W.K_V * mu[3] == pytest.approx(1.0, rel=1e-13)


# ------------------------------------------------------------------------------------
# PIN-11 / PIN-13: constant-G exact translation n(L, t) = n0(L - G t); van Leer is
# second order away from extrema, upwind first order
# ------------------------------------------------------------------------------------
def _translation_error(N, lim, steps_per_unit=1):
    dL = 1200.0 / N
    G = 0.5
    dt = 0.5 * dL / G / steps_per_unit          # C = 0.5 at every resolution
    t_end = 200.0
    M = int(round(t_end / dt))
    w = W.Workload(name="tr", N=N, dL=dL, limiter=lim, dt_fixed=dt, law=W.LAW_CONST, theta=np.array([[G]]),
                   sol_kind=W.SOL_EXP, sol=np.array(W.SOL_EXP_DEFAULT), knot_t=np.array([0.0]),
                   knot_T=np.array([[15.0]]), n0=W.gaussian_seed(N, dL)[None, :], c0=np.array([8.0]),
                   t_samples=np.array([t_end]), max_steps=10 * M)
    r = oracle.run(w)
    m1 = 400.0 + G * t_end       # same crystal count N_c as the seed: undo the mass scaling
    exact = W.gaussian_seed(N, dL, mean=m1) * (m1 ** 3 + 3 * m1 * 900.0) / (400.0 ** 3 + 3 * 400.0 * 900.0)
    return np.sum(np.abs(r["n_final"][0] - exact)) * dL / (np.sum(exact) * dL)


@pytest.mark.parametrize("lim,order_lo,order_hi", [(W.LIM_VANLEER, 1.5, 2.5), (W.LIM_UPWIND, 0.8, 1.2)])
def test_pin13_translation_convergence(lim, order_lo, order_hi):
    e = [_translation_error(N, lim) for N in (200, 400, 800)]
    orders = np.log2(np.array(e[:-1]) / np.array(e[1:]))
    assert np.all(orders > order_lo) and np.all(orders < order_hi), (e, orders)


def test_pin11_constant_G_moments_approach_mom():
    # config 1 (van Leer): closed-form moments mu_k(t) = sum_j C(k,j) (G t)^(k-j) mu_j(0)
    errs = []
    for N in (100, 200, 400):
        w = W.c1_growth(W.LIM_VANLEER, N=N, M=10)
        w.dt_fixed = (1200.0 / N) / 12.0          # keep C = G dt / dL = 1/24 as in C1
        r = oracle.run(w)
        mu0 = oracle.moments(w, w.n0[0])
        Gt = 0.5 * 1000.0
        mu3 = sum(math.comb(3, j) * Gt ** (3 - j) * mu0[j] for j in range(4))
        errs.append(abs(r["samples"][0, -1, 5] - mu3) / mu3)
    assert errs[0] < 2e-3
    # monotone and better than first order over a 4x refinement (limiter clipping at the
    # extremum keeps van Leer below 2nd order in this norm)
    assert errs[2] < errs[1] < errs[0] and errs[0] / errs[2] > 4.0, errs


# ------------------------------------------------------------------------------------
# PIN-12: kinetics-coupled method of moments (SI eq-mom2D in 1D), RK4 with step halving
# ------------------------------------------------------------------------------------
def _mom_rk4(w, mu_init, t_end, n_steps, s=0):
    import tests.mom as mom
    return mom.solve(w, mu_init, t_end, n_steps, s)


@pytest.mark.parametrize("make", [lambda N, h: W.c3_cycling(N=N, t_max=100.0, M=100, dt_max=h),
                                  lambda N, h: W.c2_dissolution(N=N, t_max=200.0, M=200, dt_max=h),
                                  lambda N, h: W.c5_ensemble(n_sims=9, N=N, t_max=100.0, M=100,
                                                             dt_max=h).subset([5])])
def test_pin12_fvm_approaches_mom(make):
    # the FVM error is O(dL^p) + O(dt) (explicit coupling of c): refine both together
    errs = []
    for N, h in ((250, 0.08), (1000, 0.02)):
        w = make(N, h)
        r = oracle.run(w)
        assert r["status"][0] == 0
        mu_init = oracle.moments(w, w.n0_for(0))
        ref = _mom_rk4(w, mu_init, w.t_samples[-1], 20000)
        ref2 = _mom_rk4(w, mu_init, w.t_samples[-1], 40000)
        assert np.allclose(ref, ref2, rtol=1e-8)          # RK4 converged
        got = r["samples"][0, -1]
        errs.append(max(abs(got[1] - ref[0]) / ref[0], abs(got[5] - ref[4]) / ref[4]))
    assert errs[-1] < 1e-2, errs
    assert errs[-1] < errs[0], errs


# ------------------------------------------------------------------------------------
# PIN-14: forward-mode tangents = complex-step derivatives = central differences
# ------------------------------------------------------------------------------------
def _tangent_case():
    w = W.c5_ensemble(n_sims=9, N=200, t_max=30.0, M=30, n_tangents=8).subset([4])
    return w


def test_pin14_dual_equals_complex_step():
    w = _tangent_case()
    rd = oracle.run(w, mode=oracle.MODE_DUAL)
    rc = oracle.run(w, mode=oracle.MODE_CSTEP)
    assert np.array_equal(rd["samples"], rc["samples"])
    for p in range(w.n_tangents):
        a, b = rd["tsamples"][0, :, p, :], rc["tsamples"][0, :, p, :]
        for k in range(5):
            scale = np.max(np.abs(a[:, k]))
            if k == 1:      # d mu0: zero up to rounding (no boundary flux)
                continue
            assert np.max(np.abs(a[:, k] - b[:, k])) <= 1e-12 * scale
        sa = np.max(np.abs(rd["ndot_final"][0, p])); assert sa > 0
        assert np.max(np.abs(rd["ndot_final"][0, p] - rc["ndot_final"][0, p])) <= 1e-11 * sa


@pytest.mark.parametrize("lim", [W.LIM_MINMOD, W.LIM_SUPERBEE, W.LIM_MC])
def test_pin14_dual_equals_complex_step_extra_limiters(lim):
    """The piecewise-linear limiters' dual arithmetic (branch derivatives) equals complex-step."""
    w = W.replace(_tangent_case(), limiter=lim)
    rd = oracle.run(w, mode=oracle.MODE_DUAL)
    rc = oracle.run(w, mode=oracle.MODE_CSTEP)
    assert np.array_equal(rd["samples"], rc["samples"])
    for p in range(w.n_tangents):
        sa = np.max(np.abs(rd["ndot_final"][0, p])); assert sa > 0
        assert np.max(np.abs(rd["ndot_final"][0, p] - rc["ndot_final"][0, p])) <= 1e-11 * sa


def test_pin14_dual_matches_central_differences():
    w = _tangent_case()
    rd = oracle.run(w, mode=oracle.MODE_DUAL)
    for p in (0, 3, 7):
        h = 1e-3 * w.theta[0, p]          # O(h^2) truncation ~1e-6; rounding noise stays < 1e-4
        wp, wm = _tangent_case(), _tangent_case()
        wp.theta = w.theta.copy(); wp.theta[0, p] += h
        wm.theta = w.theta.copy(); wm.theta[0, p] -= h
        fd = (oracle.run(wp)["samples"][0, :, 1:] - oracle.run(wm)["samples"][0, :, 1:]) / (2 * h)
        ad = rd["tsamples"][0, :, p, :]
        for k in (0, 2, 3, 4):
            assert np.allclose(ad[:, k], fd[:, k], rtol=1e-4, atol=1e-6 * np.max(np.abs(ad[:, k])))


def test_pin14_uncapped_cfl_tangents_vanish():
    # AMB-9: with uncapped CFL steps C = nu sgn(G) exactly, so n and c do not depend on theta
    w = W.c4_sweep(500, batch=1, n_steps=50)
    w.n_tangents = 6
    r = oracle.run(w, mode=oracle.MODE_DUAL)
    assert np.all(r["ndot_final"] == 0.0)
    assert np.all(r["tsamples"][0, 0, :, 0] == 0.0)


# ------------------------------------------------------------------------------------
# row a7: loss and its gradient (from tangents) vs central differences of the loss
# ------------------------------------------------------------------------------------
def test_loss_gradient_matches_finite_differences():
    w = _tangent_case()
    rd = oracle.run(w, mode=oracle.MODE_DUAL)
    loss, grad = oracle.loss_and_grad(rd["samples"], rd["tsamples"], w.target)
    own = rd["samples"][:, :, [1, 3]].copy(); own[:, :, 1] /= rd["samples"][:, :, 2]
    assert oracle.loss_and_grad(rd["samples"], None, own)[0][0] == 0.0
    for p in (1, 5):
        h = 1e-3 * w.theta[0, p]
        lp = []
        for sgn in (1, -1):
            wp = _tangent_case(); wp.theta = w.theta.copy(); wp.theta[0, p] += sgn * h
            lp.append(oracle.loss_and_grad(oracle.run(wp)["samples"], None, w.target)[0][0])
        assert grad[0, p] == pytest.approx((lp[0] - lp[1]) / (2 * h), rel=1e-4)


# ------------------------------------------------------------------------------------
# runtime errors (per-simulation status)
# ------------------------------------------------------------------------------------
def test_status_cfl_violation_fixed_dt():
    w = W.c1_growth()
    w.dt_fixed = 30.0                      # C = 0.5 * 30 / 12 = 1.25 > 1
    r = oracle.run(w)
    assert r["status"][0] == 2 and r["steps"][0] == 0 and np.all(np.isnan(r["samples"]))


def test_status_infeasible_and_maxsteps():
    w = W.c1_growth()
    w.c0 = np.array([0.01])                # crystals grow at constant G: solute runs out
    r = oracle.run(w)
    assert r["status"][0] == 4
    w = W.c1_growth(); w.max_steps = 10
    r = oracle.run(w)
    assert r["status"][0] == 5 and r["steps"][0] == 10


def test_appb_targets_are_the_method_of_moments():
    # workloads/data/appb_targets.npy (tools/gen_appb_targets.py): spot-check experiment 4
    # (T = 15 C, S0 = 1.25) over its first 5 samples with an independent RK4 run at h = 0.01
    from tests import mom
    N = 2000
    dL = 1200.0 / N
    n0 = W.gaussian_seed(N, dL, m0=1.0)
    L = W.bin_centers(N, dL)
    y = np.array([W.APPB_S0[1] * W.APPB_CSAT[1]] + [np.sum(dL * L ** k * n0) for k in range(4)])
    w = W.Workload(name="appb", N=N, dL=dL, law=W.LAW_ARRHENIUS, theta=np.array([W.ARRHENIUS_DEFAULT[:3]]),
                   sol_kind=W.SOL_EXP, sol=np.array(W.SOL_EXP_DEFAULT), knot_t=np.array([0.0]),
                   knot_T=np.array([[15.0]]), n0=n0[None, :], c0=y[:1].copy())
    tg = W.appb_target(np.array([4]), np.arange(1.0, 6.0), y[:1])[0]
    for m in range(5):
        w.c0 = np.array([y[0]])
        y = mom.solve(w, y[1:], 1.0, 100)
        assert tg[m, 0] == pytest.approx(y[0], rel=1e-9) and tg[m, 1] == pytest.approx(y[2] / y[1], rel=1e-9)
