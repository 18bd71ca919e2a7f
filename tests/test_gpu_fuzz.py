"""Seeded randomized parity: configuration combinations the targeted tests do not cross —
mesh size, tangent lanes, the five limiters, the three growth laws (incl. long polynomials),
both solubility forms, constant and ramped temperature, fixed / capped / uncapped time steps,
sample and steps modes, Gaussian and log-normal seeds, and every 1D kernel (AUTO, resident,
cluster, stream) — each against the oracle with the same bars as test_gpu_parity.py.
Every case is drawn from numpy PCG64(seed) so failures reproduce exactly."""
import math
import os

import numpy as np
import pytest

import oracle
import workloads as W
from tests.test_gpu_parity import RTOL_TAN, _cmp_n, _cmp_samples, _cmp_tangents

pytestmark = pytest.mark.gpu

KERNELS = (0, 1, 2, 3)     # AUTO, RESIDENT, CLUSTER, STREAM


def random_case(seed):
    rng = np.random.Generator(np.random.PCG64(1000 + seed))
    kernel = int(rng.choice(KERNELS))
    if kernel == 2:
        N = int(rng.integers(3000, 9000))
    elif kernel == 3:
        N = int(rng.integers(300, 6000))
    else:
        N = int(rng.integers(3, 700))
    P = int(rng.integers(0, 5 if kernel == 3 else (9 if kernel == 2 else 11)))
    lim = int(rng.integers(0, 5))
    law = int(rng.choice([W.LAW_CONST, W.LAW_ARRHENIUS, W.LAW_POLY]))
    S = int(rng.integers(1, 4))
    dL = 1200.0 / N
    if law == W.LAW_CONST:
        theta = np.full((S, 1), float(rng.uniform(-0.8, 2.0)))
    elif law == W.LAW_ARRHENIUS:
        base = np.array(W.ARRHENIUS_DEFAULT)[: (6 if rng.random() < 0.6 else 3)]
        theta = base[None, :] * np.exp(0.1 * rng.standard_normal((S, base.shape[0])))
    else:
        k = int(rng.integers(1, 14))
        theta = np.abs(rng.standard_normal((S, k))) * np.array([20.0 / (j + 1) for j in range(k)])[None, :]
    sol_kind = int(rng.integers(0, 2))
    sol = np.array(W.SOL_EXP_DEFAULT) if sol_kind == 0 else np.array([3.37, 0.07, 0.002])
    if rng.random() < 0.5:
        knot_t, knot_T = np.array([0.0]), np.full((S, 1), float(rng.uniform(10.0, 25.0)))
    else:
        knot_t = np.array([0.0, float(rng.uniform(5.0, 30.0)), float(rng.uniform(31.0, 60.0))])
        knot_T = np.tile(np.array([[float(rng.uniform(10, 20)), float(rng.uniform(15, 25)), float(rng.uniform(10, 25))]]),
                         (S, 1))
    # concentration around saturation at the initial temperature: growth or dissolution
    T0 = knot_T[0, 0]
    csat = sol[0] * math.exp(sol[1] * T0) if sol_kind == 0 else sol[0] + sol[1] * T0 + sol[2] * T0 * T0
    c0 = csat * rng.uniform(0.85, 1.4, S)
    seed_fn = W.gaussian_seed if rng.random() < 0.6 else W.lognormal_seed
    mean = float(rng.uniform(150.0, 900.0))
    lo_sig = max(3 * dL, 20.0)
    n0 = seed_fn(N, dL, mean=mean, sigma=float(rng.uniform(lo_sig, max(lo_sig + 1.0, 80.0))), m0=float(rng.uniform(0.2, 2.0)))
    mode = rng.choice(["fixed", "capped", "uncapped"])
    dt_fixed = float(rng.uniform(0.01, 0.3)) * dL if mode == "fixed" else 0.0
    dt_max = float(rng.uniform(0.02, 0.5)) if mode == "capped" else math.inf
    steps_mode = kernel == 3 and rng.random() < 0.5 or rng.random() < 0.2
    t_max = float(rng.uniform(2.0, 30.0))
    M = int(rng.integers(1, 12))
    w = W.Workload(
        name=f"fuzz{seed}", N=N, dL=dL, limiter=lim, dt_fixed=dt_fixed, dt_max=dt_max, max_steps=4000,
        n_steps=int(rng.integers(20, 150)) if steps_mode else 0, law=law, theta=theta, sol_kind=sol_kind, sol=sol,
        knot_t=knot_t, knot_T=knot_T, n0=n0[None, :], c0=c0,
        t_samples=np.array([t_max]) if steps_mode else np.linspace(t_max / M, t_max, M),
        target=None, n_tangents=P)
    return w, kernel


NF = int(os.environ.get("PBE_FUZZ_N", "40"))       # case counts (larger one-off sweeps: PBE_FUZZ_N=200)


@pytest.mark.parametrize("seed", range(NF))
def test_fuzz_matches_oracle(seed):
    import paper_2411_00742_b200 as pb
    w, kernel = random_case(seed)
    mode = oracle.MODE_DUAL if w.n_tangents else oracle.MODE_DOUBLE
    o = oracle.run(w, mode=mode, threads=4)
    try:
        g = pb.run_workload(w, kernel=kernel)
    except pb.PBEError as e:            # only documented argument limits may refuse a case
        pytest.skip(f"refused: {e}")
    assert np.array_equal(g["status"], o["status"]), (g["status"], o["status"])
    assert np.array_equal(g["steps"], o["steps"]), (g["steps"], o["steps"])
    _cmp_samples(g, o)
    _cmp_n(g, o)
    if w.n_tangents:
        _cmp_tangents(g, o)
        for s in range(w.n_sims):
            if o["status"][s] != 0:
                continue
            for p in range(w.n_tangents):
                sc = np.max(np.abs(o["ndot_final"][s, p]))
                assert np.max(np.abs(g["ndot_final"][s, p] - o["ndot_final"][s, p])) <= RTOL_TAN * max(sc, 1e-300)


# ---------------------------------------------------------------------------------------------
# 2D model (NEXT-1) and the adjoint (NEXT-3)
# ---------------------------------------------------------------------------------------------
def random_case_2d(seed):
    rng = np.random.Generator(np.random.PCG64(5000 + seed))
    N1, N2 = int(rng.integers(8, 260)), int(rng.integers(8, 200))
    S = int(rng.integers(1, 4))
    lim = int(rng.integers(0, 5))
    law = int(rng.choice([W.LAW_CONST, W.LAW_ARRHENIUS, W.LAW_POLY]))
    if law == W.LAW_CONST:
        theta = np.tile(np.array([[rng.uniform(0.1, 2.0), rng.uniform(-0.5, 1.0)]]), (S, 1))
    elif law == W.LAW_ARRHENIUS:
        theta = np.tile(np.array(W.ARRHENIUS_2D)[None, :], (S, 1)) * np.exp(0.1 * rng.standard_normal((S, 6)))
    else:
        k = int(rng.integers(1, 5))
        theta = np.abs(rng.standard_normal((S, 2 * k))) * 10.0
    w = W.c2d_base(N1, N2, t_max=float(rng.uniform(1.0, 8.0)), M=int(rng.integers(1, 5)), n_sims=S,
                   dt_max=float(rng.uniform(0.05, 0.5)) if rng.random() < 0.5 else math.inf, limiter=lim)
    w = W.replace(w, law=law, theta=theta, c0=8.0 * rng.uniform(0.7, 1.3, S), max_steps=3000)
    if rng.random() < 0.5:
        w = W.replace(w, knot_t=np.array([0.0, 4.0]), knot_T=np.array([[float(rng.uniform(10, 20)), float(rng.uniform(10, 25))]]))
    return w


DRAIN = 1e-4     # R-33: a moment below 1e-4 of its run maximum has lost > 99.99% of its mass


@pytest.mark.parametrize("seed", range(max(12, NF // 4)))
def test_fuzz_2d_matches_oracle(seed):
    import paper_2411_00742_b200 as pb
    w = random_case_2d(seed)
    o = oracle.run2d(w, threads=4)
    g = pb.run_workload(w)
    assert np.array_equal(g["status"], o["status"]) and np.array_equal(g["steps"], o["steps"]), (g["status"], o["status"])
    a, b = g["samples"], o["samples"]
    assert np.array_equal(np.isnan(a), np.isnan(b))
    # element-wise 1e-10 relative (north star), except for a moment the outflow boundary has drained
    # below DRAIN of its largest value over the run: its absolute error is the rounding of the
    # fluxes that carried that mass out, so it is compared at 1e-10 of its run maximum (reading
    # R-33)
    runmax = np.nanmax(np.abs(b), axis=1, keepdims=True)
    drained = np.abs(b) < DRAIN * runmax
    scale = np.where(drained, runmax, np.abs(b))
    ok = ~np.isnan(b)
    if ok.any():
        assert np.max((np.abs(a - b) / np.maximum(scale, 1e-300))[ok]) <= 1e-10
    for s in range(w.n_sims):
        if o["status"][s] == 0:
            f = o["f_final"][s].reshape(-1)
            sc = np.max(np.abs(f))
            if sc < DRAIN * np.max(np.abs(w.n0)):            # the whole field drained (R-33)
                sc = np.max(np.abs(w.n0))
            assert np.max(np.abs(g["n_final"][s] - f)) <= 1e-9 * sc


@pytest.mark.parametrize("seed", range(max(10, NF // 4)))
def test_fuzz_adjoint_matches_oracle(seed):
    from tests.test_gpu_adjoint import RTOL_GRAD, RTOL_LOSS, gpu_adjoint, oracle_grad
    rng = np.random.Generator(np.random.PCG64(9000 + seed))
    w, _ = random_case(seed)
    if w.n_steps:                                     # the adjoint differentiates sample mode only
        w = W.replace(w, n_steps=0, t_samples=np.linspace(2.0, 2.0 * int(rng.integers(2, 7)), int(rng.integers(1, 6))))
    N = min(w.N, 600)
    if N != w.N:
        w = W.replace(w, N=N, dL=1200.0 / N, n0=W.gaussian_seed(N, 1200.0 / N, mean=400.0)[None, :])
    w = W.replace(w, n_tangents=0, tangent_seed=None, target=W._target(w.c0, w.t_samples))
    lo, go = oracle_grad(W.replace(w, max_steps=4000), allow_fail=True)
    ok = np.isfinite(lo)
    g, rec, _ = gpu_adjoint(w)
    o_status = oracle.run(w, want_n=False)["status"]
    assert np.array_equal(rec["status"], o_status)
    if not ok.any():
        return
    assert np.all(np.abs(g["loss"][ok] - lo[ok]) <= RTOL_LOSS * np.abs(lo[ok]))
    scale = np.max(np.abs(go[ok]), axis=1, keepdims=True)
    assert (np.abs(g["grad"][ok] - go[ok]) / np.maximum(scale, 1e-300)).max() <= RTOL_GRAD


def _cluster_size_for(N):
    """The CS in {16, 8, 4, 2} for which libpbe's cluster adjoint (64 threads x K in {2, 4, 8} bins
    per CTA, every CTA but the last full) takes N, or 0."""
    for c in (16, 8, 4, 2):
        for K in (2, 4, 8):
            nb = 64 * K
            if c * nb >= N and (c - 1) * nb < N:
                return c
    return 0


@pytest.mark.parametrize("seed", range(max(8, NF // 5)))
def test_fuzz_adjoint_cluster_matches_oracle(seed, monkeypatch):
    """The cluster adjoint (CTAs exchanging halos and partials with st.async) on random cases."""
    from tests.test_gpu_adjoint import RTOL_GRAD, RTOL_LOSS, gpu_adjoint, oracle_grad
    rng = np.random.Generator(np.random.PCG64(9500 + seed))
    w, _ = random_case(seed + 100)
    if w.n_steps:
        w = W.replace(w, n_steps=0, t_samples=np.linspace(2.0, 2.0 * int(rng.integers(2, 7)), int(rng.integers(1, 6))))
    N = int(rng.integers(129, 1025))
    cs = _cluster_size_for(N)
    if cs == 0:
        N, cs = 200, 2
    w = W.replace(w, N=N, dL=1200.0 / N, n0=W.gaussian_seed(N, 1200.0 / N, mean=float(rng.uniform(300, 900)))[None, :],
                  n_tangents=0, tangent_seed=None, target=W._target(w.c0, w.t_samples))
    monkeypatch.setenv("PBE_ADJ_CLUSTER", str(cs))
    lo, go = oracle_grad(W.replace(w, max_steps=4000), allow_fail=True)
    ok = np.isfinite(lo)
    g, rec, info = gpu_adjoint(w)
    assert info["cluster"] == cs, (N, cs, info)
    o_status = oracle.run(w, want_n=False)["status"]
    assert np.array_equal(rec["status"], o_status)
    if not ok.any():
        return
    assert np.all(np.abs(g["loss"][ok] - lo[ok]) <= RTOL_LOSS * np.abs(lo[ok]))
    scale = np.max(np.abs(go[ok]), axis=1, keepdims=True)
    assert (np.abs(g["grad"][ok] - go[ok]) / np.maximum(scale, 1e-300)).max() <= RTOL_GRAD
