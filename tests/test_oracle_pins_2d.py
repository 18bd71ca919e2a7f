"""Pins for the 2D oracle (NEXT-1: the paper's 2D model with Godunov dimensional splitting,
PAPER.md L257-312, L291).  CPU only."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W
from tests import exact_march as X
from tests import mom2d


@pytest.mark.parametrize("lim", [W.LIM_UPWIND, W.LIM_VANLEER])
@pytest.mark.parametrize("C1,C2", [(0.3, 0.7), (-0.4, 0.9), (0.9, -0.2), (1.0, 1.0)])
def test_split_step_of_a_product_is_the_product_of_1d_steps(lim, C1, C2):
    # the limited slope is positively homogeneous (psi(la, lb) = l psi(a, b), l > 0), so one
    # split step of g (x) h is sweep_C1(g) (x) sweep_C2(h): pins rows-vs-columns and order
    rng = np.random.default_rng(int(10 * (C1 + 3 * C2)) + lim)
    g = rng.random(37) * (rng.random(37) < 0.9)
    h = rng.random(23) * (rng.random(23) < 0.9)
    out = oracle.split_step_2d(np.outer(h, g), C1, C2, lim)
    ref = np.outer(oracle.sweep(h, C2, lim), oracle.sweep(g, C1, lim))
    assert np.allclose(out, ref, rtol=1e-13, atol=1e-15 * np.abs(ref).max())


def test_unit_courant_moves_the_field_diagonally():
    rng = np.random.default_rng(5)
    f = rng.random((12, 15)); f[:, :2] = 0; f[:2, :] = 0
    out = oracle.split_step_2d(f, 1.0, 1.0, W.LIM_VANLEER)
    assert np.array_equal(out[1:, 1:], f[:-1, :-1]) and not out[0].any() and not out[:, 0].any()


def _tiny2d(law, theta, dt, c0=4.0):
    rng = np.random.default_rng(9)
    N1, N2 = 6, 5
    f0 = np.array([float(x) for x in rng.integers(0, 20, N1 * N2)]) * 0.5
    return W.Workload(name="t2", N=N1, dL=1.0, N2=N2, dL2=1.0, dt_fixed=dt, law=law, theta=np.array([theta]),
                      sol_kind=W.SOL_POLY, sol=np.array([2.0, 0.0, 0.0]), knot_t=np.array([0.0]),
                      knot_T=np.array([[15.0]]), n0=f0[None, :], c0=np.array([c0]), rho_c=1e-4, k_v=0.5,
                      t_samples=np.array([0.25, 0.5, 0.75]))


@pytest.mark.parametrize("lim", [0, 1])
def test_2d_march_matches_exact_rational_brute_force(lim):
    # polynomial growth in both dimensions, polynomial solubility, fixed dt: all rational
    w = _tiny2d(W.LAW_POLY, [0.5, 0.25, 0.75, 0.125], 0.25)
    w.limiter = lim
    if lim:
        w.t_samples = w.t_samples[:2]      # limiter denominators grow fast in exact arithmetic
    r = oracle.run2d(w)
    assert r["status"][0] == 0 and r["steps"][0] == len(w.t_samples)
    recs, f = X.march_2d(X.Num("fraction"), N1=6, N2=5, dL1=1.0, dL2=1.0, limiter=lim, dt_fixed=0.25,
                         law=W.LAW_POLY, theta=list(w.theta[0]), sol_kind=1, sol=[2.0, 0.0, 0.0], T=15.0,
                         f0=list(w.n0[0]), c0=4.0, rho_c=1e-4, k_v=0.5, t_samples=list(w.t_samples))
    ex = np.array([[float(v) for v in rec] for rec in recs])
    assert np.allclose(r["samples"][0], ex, rtol=1e-13, atol=0)
    fe = np.array([[float(v) for v in row] for row in f])
    assert np.max(np.abs(r["f_final"][0] - fe)) <= 1e-13 * np.max(fe)


@pytest.mark.parametrize("lim", [0, 1])
def test_2d_cfl_rule_matches_exact_rational_brute_force(lim):
    # SI L857-861: dt = nu min(dL1/|G1|, dL2/|G2|).  dL1 = 1 != dL2 = 0.5 and G2 = (S-1)^2 vs
    # G1 = S-1, with a mass coupling strong enough that the binding dimension switches from L2
    # to L1 as S falls: a dt taken from one dimension only, or with the wrong bin width,
    # changes every record.
    rng = np.random.default_rng(9)
    N1, N2 = 6, 5
    f0 = np.array([float(x) for x in rng.integers(0, 20, N1 * N2)]) * 0.5
    kw = dict(theta=[1.0, 0.0, 0.0, 1.0], sol=[2.0, 0.0, 0.0], rho_c=0.1, k_v=0.5, t_samples=[1.0, 2.0])
    w = W.Workload(name="t2cfl", N=N1, dL=1.0, N2=N2, dL2=0.5, dt_fixed=0.0, law=W.LAW_POLY,
                   theta=np.array([kw["theta"]]), sol_kind=W.SOL_POLY, sol=np.array(kw["sol"]),
                   knot_t=np.array([0.0]), knot_T=np.array([[15.0]]), n0=f0[None, :], c0=np.array([4.0]),
                   rho_c=kw["rho_c"], k_v=kw["k_v"], t_samples=np.array(kw["t_samples"]), limiter=lim,
                   courant=0.9)
    r = oracle.run2d(w)
    binding = []
    recs, f = X.march_2d(X.Num("fraction"), N1=N1, N2=N2, dL1=1.0, dL2=0.5, limiter=lim, dt_fixed=0,
                         law=W.LAW_POLY, sol_kind=1, T=15.0, f0=list(f0), c0=4.0, courant=0.9,
                         binding=binding, **kw)
    assert 1 in binding and 2 in binding, binding          # both dimensions limit dt at some step
    assert r["status"][0] == 0 and r["steps"][0] == len(binding)
    ex = np.array([[float(v) for v in rec] for rec in recs])
    assert np.allclose(r["samples"][0], ex, rtol=1e-13, atol=0)
    fe = np.array([[float(v) for v in row] for row in f])
    assert np.max(np.abs(r["f_final"][0] - fe)) <= 1e-13 * np.max(fe)


def test_2d_conservation_and_positivity():
    w = W.c2d_base(120, 60, t_max=20.0, M=20)
    r = oracle.run2d(w)
    assert r["status"][0] == 0
    s = r["samples"][0]
    mu00_0 = np.sum(w.n0[0]) * w.dL * w.dL2
    assert np.max(np.abs(s[:, 2] - mu00_0)) <= 1e-12 * mu00_0
    L1 = W.bin_centers(120, w.dL); L2 = W.bin_centers(60, w.dL2)
    mu12_0 = np.sum(np.outer(L2 ** 2, L1).reshape(-1) * w.n0[0]) * w.dL * w.dL2
    inv = s[:, 1] + w.rho_c * w.k_v * s[:, 7]
    assert np.allclose(inv, 8.0 + w.rho_c * w.k_v * mu12_0, rtol=1e-12)
    assert np.all(r["f_final"] >= 0)


def test_2d_fvm_approaches_2d_method_of_moments():
    errs = []
    for N1, N2 in ((60, 30), (240, 120)):
        w = W.c2d_base(N1, N2, t_max=10.0, M=5)
        r = oracle.run2d(w)
        assert r["status"][0] == 0
        f = w.n0[0].reshape(N2, N1)
        L1 = W.bin_centers(N1, w.dL); L2 = W.bin_centers(N2, w.dL2)
        wgt = w.dL * w.dL2
        mu0 = np.array([np.sum(f) * wgt, np.sum(f * L1[None, :]) * wgt, np.sum(f * L2[:, None]) * wgt,
                        np.sum(f * np.outer(L2, L1)) * wgt, np.sum(f * (L2 ** 2)[:, None]) * wgt,
                        np.sum(f * np.outer(L2 ** 2, L1)) * wgt])
        ref = mom2d.solve(w, mu0, 10.0, 20000)
        got = r["samples"][0, -1]
        errs.append(max(abs(got[1] - ref[0]) / ref[0], abs(got[7] - ref[6]) / ref[6]))
    assert errs[-1] < 1e-2 and errs[-1] < errs[0], errs


def test_2d_seed_mass():
    w = W.c2d_base(600, 300)
    L1 = W.bin_centers(600, w.dL); L2 = W.bin_centers(300, w.dL2)
    f = w.n0[0].reshape(300, 600)
    mu12 = np.sum(f * np.outer(L2 ** 2, L1)) * w.dL * w.dL2
    assert W.RHO_C * W.K_V * mu12 == pytest.approx(1.0, rel=1e-12)
