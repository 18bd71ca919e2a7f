"""NEXT-3 parity: the reverse-mode gradient of libpbe (pbe_run_adjoint, k_adjoint) against the
oracle's forward-mode gradient of the same discrete loss (oracle/pbe_oracle.cpp in dual
arithmetic, pinned against complex-step and finite differences in test_oracle_pins.py).
Reverse and forward mode differentiate the same discrete march with the same branch decisions,
so they agree up to rounding: the bar is 1e-8 x max |grad| per simulation (R-21 style, the
kinetic partials span many orders of magnitude) plus the loss to 1e-10 relative.
Dual lanes are limited to 10, so the oracle gradient over n_params > 10 parameters is
assembled from ceil(n_params / 10) runs with unit seed blocks."""
import math

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

RTOL_GRAD = 1e-8
RTOL_LOSS = 1e-10


def oracle_grad(w, allow_fail=False):
    """(loss [S], grad [S][n_params]) of workload w from the oracle in dual arithmetic (failed
    simulations give NaN when allow_fail)."""
    P, Q = w.n_params, w.sol.shape[0]
    grads = []
    loss = None
    for j0 in range(0, P, 10):
        nl = min(10, P - j0)
        seed = np.zeros((nl, P + Q))
        seed[np.arange(nl), j0 + np.arange(nl)] = 1.0
        wk = W.replace(w, n_tangents=nl, tangent_seed=seed)
        o = oracle.run(wk, oracle.MODE_DUAL, threads=8, want_n=False)
        assert allow_fail or (o["status"] == 0).all(), o["status"]
        lo, g = oracle.loss_and_grad(o["samples"], o["tsamples"], w.target)
        loss = lo if loss is None else loss
        grads.append(g)
    return loss, np.concatenate(grads, axis=1)


def gpu_adjoint(w, checkpoint_every=0):
    import torch

    import paper_2411_00742_b200 as pb
    wg = W.replace(w, n_tangents=0, tangent_seed=None)
    ctx = pb.context_for(wg)
    n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).cuda()
    ctx.run_adjoint(n0, w.c0, w.t_samples, w.target, checkpoint_every=checkpoint_every)
    g = ctx.adjoint_gradient(w.n_params)
    rec = ctx.moments()
    info = ctx.last_run_info()
    ctx.close()
    return g, rec, info


def _check(w, checkpoint_every=0):
    lo, go = oracle_grad(w)
    g, rec, info = gpu_adjoint(w, checkpoint_every)
    assert info["kernel"] == 5
    assert (rec["status"] == 0).all(), rec["status"]
    assert np.all(np.abs(g["loss"] - lo) <= RTOL_LOSS * np.abs(lo)), (g["loss"], lo)
    scale = np.max(np.abs(go), axis=1, keepdims=True)
    err = np.abs(g["grad"] - go) / scale
    assert err.max() <= RTOL_GRAD, f"max grad err {err.max():.3e} (per-sim scale {scale.ravel()})"
    return g, go


def small_ensemble(n_params=8, n_sims=9, N=200, t_max=60.0, M=30, dt_max=0.5, limiter=W.LIM_VANLEER):
    """C5-shaped (App. B experiments, polynomial growth) at test size; parameters beyond the
    8 of POLY_A get small coefficients so the long polynomial stays physical."""
    w = W.c5_ensemble(n_sims=n_sims, N=N, t_max=t_max, M=M, dt_max=dt_max, n_tangents=0)
    if n_params != w.n_params:
        th = np.zeros((n_sims, n_params))
        k = min(n_params, w.n_params)
        th[:, :k] = w.theta[:, :k]
        if n_params > w.n_params:
            rng = np.random.Generator(np.random.PCG64(7))
            th[:, w.n_params:] = 0.05 * rng.random((n_sims, n_params - w.n_params))
        w = W.replace(w, theta=th)
    return W.replace(w, limiter=limiter, max_steps=20000)


def test_adjoint_poly_ensemble_matches_oracle():
    _check(small_ensemble())


def test_adjoint_long_polynomial_matches_oracle():
    """n_params = 40 > MAXTH: the runtime-loop POLY path on both sides."""
    _check(small_ensemble(n_params=40, n_sims=3))


def test_adjoint_upwind_matches_oracle():
    _check(small_ensemble(n_sims=3, limiter=W.LIM_UPWIND))


@pytest.mark.parametrize("lim", [W.LIM_MINMOD, W.LIM_SUPERBEE, W.LIM_MC])
def test_adjoint_extra_limiters_match_oracle(lim):
    _check(small_ensemble(n_sims=3, limiter=lim))


def test_adjoint_uncapped_cfl_matches_oracle():
    """dt = nu dL/|G| (C = nu sgn G, R-9): the parameters act through the clock only."""
    _check(small_ensemble(n_sims=3, dt_max=math.inf, t_max=120.0, M=12))


def test_adjoint_dissolution_ramp_matches_oracle():
    """C2-shaped: Arrhenius growth + dissolution (6 parameters), temperature ramp (dG/dt via
    T(t)), C < 0 sweeps, landing steps."""
    w = W.c2_dissolution()
    N = 150
    dL = 1200.0 / N
    t = np.linspace(4.0, 120.0, 30)
    w = W.replace(w, N=N, dL=dL, n0=W.gaussian_seed(N, dL, m0=3.0)[None, :], t_samples=t, dt_max=0.5,
                  target=W._target(w.c0, t), max_steps=20000)
    _check(w)


def test_adjoint_fixed_dt_constant_growth_matches_oracle():
    w = W.c1_growth(W.LIM_VANLEER, N=100, M=25)
    t = np.linspace(8.0, 200.0, 25)
    w = W.replace(w, t_samples=t, target=W._target(w.c0, t), max_steps=5000)
    _check(w)


def test_adjoint_checkpoint_interval_is_bitwise_neutral():
    w = small_ensemble(n_sims=2, M=10, t_max=20.0)
    g1, _, _ = gpu_adjoint(w, checkpoint_every=1)
    g7, _, _ = gpu_adjoint(w, checkpoint_every=7)
    g0, _, _ = gpu_adjoint(w, checkpoint_every=0)
    assert np.array_equal(g1["grad"], g7["grad"]) and np.array_equal(g1["grad"], g0["grad"])


@pytest.mark.parametrize("N", [97, 128])
def test_adjoint_trajectory_mode_matches_recompute_mode(N, monkeypatch):
    """checkpoint_every=0 keeps every state in HBM (cp.async ring, no re-march); the O(sqrt K)
    checkpoint mode re-marches each segment.  Same arithmetic -> bitwise equal (odd N: the
    8-byte tail copy of the ring prefetch)."""
    w = small_ensemble(n_sims=3, N=N, M=10, t_max=20.0)
    g0, _, info0 = gpu_adjoint(w, checkpoint_every=0)
    monkeypatch.setenv("PBE_ADJ_RECOMPUTE", "1")
    g1, _, _ = gpu_adjoint(w, checkpoint_every=0)
    assert np.array_equal(g0["grad"], g1["grad"]) and np.array_equal(g0["loss"], g1["loss"])


@pytest.mark.parametrize("N", [1500, 3001, 6000])
def test_adjoint_large_mesh_matches_oracle(N):
    """The wider CTA variants (K = 4 at 384-512 threads, K = 16, K = 24 at 256 threads) with
    their padded shared-memory rows; N = 6000 also takes the segment re-march (the 3-state ring
    does not fit next to the K = 24 rows)."""
    _check(small_ensemble(n_sims=2, N=N, t_max=4.0, M=4))


def test_adjoint_agrees_with_gpu_tangents():
    """The two GPU differentiation modes (k_resident tangent lanes, k_adjoint) agree."""
    import paper_2411_00742_b200 as pb
    w = small_ensemble(n_sims=4)
    wt = W.replace(w, n_tangents=8)
    r = pb.run_workload(wt, want_n=False)
    g, rec, _ = gpu_adjoint(w)
    scale = np.max(np.abs(r["grad"]), axis=1, keepdims=True)
    assert (np.abs(g["grad"] - r["grad"]) / scale).max() <= RTOL_GRAD
    ok = ~np.isnan(r["samples"])
    assert np.allclose(rec["moments"][ok], r["samples"][ok], rtol=1e-12, atol=0)


def test_adjoint_failed_simulation_gives_nan():
    """A simulation that exceeds max_steps has no gradient (NaN) and status MAXSTEPS."""
    w = W.replace(small_ensemble(n_sims=2), max_steps=50)
    g, rec, _ = gpu_adjoint(w)
    assert (rec["status"] == 5).all()
    assert np.isnan(g["grad"]).all() and np.isnan(g["loss"]).all()


def test_adjoint_rejects_bad_arguments():
    import torch

    import paper_2411_00742_b200 as pb
    w = small_ensemble(n_sims=1)
    ctx = pb.context_for(w)
    n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).cuda()
    with pytest.raises(pb.PBEError):
        ctx.run_adjoint(n0, w.c0, w.t_samples, None)                       # no target
    with pytest.raises(pb.PBEError):
        ctx.adjoint_gradient(w.n_params)                                   # no adjoint run yet
    ctx.close()


def test_adjoint_full_size_matches_gpu_tangents():
    """NEXT-3 exactly as bench.py times it (9 experiments, N = 2000, 12,000 steps, 1000 POLY
    coefficients): the adjoint gradient of coefficients 0..9 and 990..999 against forward-mode
    tangent lanes on the same parameters (the tangent path is itself pinned to the oracle)."""
    import paper_2411_00742_b200 as pb
    w = W.next3_estimation(n_params=1000)
    g, rec, _ = gpu_adjoint(w)
    assert (rec["status"] == 0).all()
    Q = w.sol.shape[0]
    for js in (np.arange(10), np.arange(990, 1000)):
        seed = np.zeros((10, 1000 + Q))
        seed[np.arange(10), js] = 1.0
        r = pb.run_workload(W.replace(w, n_tangents=10, tangent_seed=seed), want_n=False)
        scale = np.max(np.abs(g["grad"]), axis=1)
        err = np.abs(g["grad"][:, js] - r["grad"]) / scale[:, None]
        assert err.max() <= RTOL_GRAD, err.max()


@pytest.mark.parametrize("N", [60, 61, 128, 129])
def test_adjoint_outflow_boundary_matches_oracle(N):
    """Mass leaving through the outflow face at L = 1200 um, with N a multiple of the bins per
    thread and not (found by the fuzz sweep: the outflow face's dF/dC term was counted twice
    when N % K == 0)."""
    w = small_ensemble(n_sims=2, N=N, t_max=20.0, M=5)
    w = W.replace(w, n0=W.gaussian_seed(N, 1200.0 / N, mean=1100.0, sigma=70.0)[None, :])
    _check(w)


@pytest.mark.parametrize("N", [64, 65])
def test_adjoint_dissolution_outflow_at_zero(N):
    """Dissolution (C < 0, Arrhenius 6 parameters) with mass leaving through L = 0."""
    w = W.c2_dissolution()
    dL = 1200.0 / N
    t = np.linspace(3.0, 30.0, 10)
    c0 = np.array([4.0])                                   # well undersaturated: strong dissolution
    w = W.replace(w, N=N, dL=dL, n0=W.gaussian_seed(N, dL, mean=60.0, sigma=40.0, m0=0.5)[None, :], c0=c0,
                  t_samples=t, dt_max=0.5, target=W._target(c0, t), max_steps=20000)
    _check(w)


# ---- cluster mode (k_adjoint<K, 64, true>: CS CTAs per simulation, DSMEM halos) -------------------
@pytest.mark.parametrize("cs,N", [(2, 200), (4, 450), (8, 1000), (16, 2000), (16, 1950)])
def test_adjoint_cluster_matches_oracle(cs, N, monkeypatch):
    """The cluster variant forced at CS = 2..16 (bins split over CTAs, edge values pushed into the
    neighbours' ghost cells, partial sums added across the cluster) against the oracle."""
    monkeypatch.setenv("PBE_ADJ_CLUSTER", str(cs))
    w = small_ensemble(n_sims=3, N=N, t_max=20.0, M=6)
    lo, go = oracle_grad(w)
    g, rec, info = gpu_adjoint(w)
    assert info["cluster"] == cs, info
    assert (rec["status"] == 0).all(), rec["status"]
    assert np.all(np.abs(g["loss"] - lo) <= RTOL_LOSS * np.abs(lo)), (g["loss"], lo)
    err = np.abs(g["grad"] - go) / np.max(np.abs(go), axis=1, keepdims=True)
    assert err.max() <= RTOL_GRAD, f"max grad err {err.max():.3e}"


@pytest.mark.parametrize("cs,N", [(2, 129), (2, 256)])
def test_adjoint_cluster_outflow_and_dissolution(cs, N, monkeypatch):
    """Cluster mode with mass at the outflow face (last CTA partial or full) and with dissolution
    (C < 0: the sweep runs the other way across the CTA boundary)."""
    monkeypatch.setenv("PBE_ADJ_CLUSTER", str(cs))
    w = small_ensemble(n_sims=2, N=N, t_max=20.0, M=5)
    w = W.replace(w, n0=W.gaussian_seed(N, 1200.0 / N, mean=1100.0, sigma=70.0)[None, :])
    _check(w)
    wd = W.c2_dissolution()
    dL = 1200.0 / N
    t = np.linspace(3.0, 30.0, 10)
    c0 = np.array([4.0])
    wd = W.replace(wd, N=N, dL=dL, n0=W.gaussian_seed(N, dL, mean=60.0, sigma=40.0, m0=0.5)[None, :], c0=c0,
                   t_samples=t, dt_max=0.5, target=W._target(c0, t), max_steps=20000)
    _check(wd)


def test_adjoint_cluster_failed_simulation_gives_nan(monkeypatch):
    monkeypatch.setenv("PBE_ADJ_CLUSTER", "2")
    w = W.replace(small_ensemble(n_sims=2), max_steps=50)
    g, rec, info = gpu_adjoint(w)
    assert info["cluster"] == 2
    assert (rec["status"] == 5).all()
    assert np.isnan(g["grad"]).all() and np.isnan(g["loss"]).all()


def test_adjoint_cluster_is_the_default_for_next3():
    """NEXT-3 (9 experiments, N = 2000) runs 16-CTA clusters (144 SMs) by default."""
    w = W.next3_estimation(n_params=40, t_max=30.0, M=30)
    g, rec, info = gpu_adjoint(w)
    assert info["cluster"] == 16 and info["ctas"] == 144, info
    assert (rec["status"] == 0).all()
