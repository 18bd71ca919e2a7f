"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Tolerances (BASELINE.json north star):
    moments and concentration   1e-10 relative
    distribution n              1e-9 * max(n)
    tangent records / ndot      1e-8 * max |lane|     (R-21: per lane)
    loss / gradient             1e-9 relative
Integers (status, step counts) must match exactly."""
import math
import os

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

RTOL_MOM = 1e-10
RTOL_N = 1e-9
RTOL_TAN = 1e-8


def _gpu(w, **kw):
    import paper_2411_00742_b200 as pb
    return pb.run_workload(w, **kw)


def _cmp_samples(g, o, rtol=RTOL_MOM):
    a, b = g["samples"], o["samples"]
    assert a.shape == b.shape
    assert np.array_equal(np.isnan(a), np.isnan(b))
    ok = ~np.isnan(b)
    if not ok.any():
        return
    err = np.abs(a[ok] - b[ok]) / np.maximum(np.abs(b[ok]), 1e-300)
    # time stamps and moments: relative; mu0's tiny drift terms are compared relative to mu0
    assert err.max() <= rtol, f"max rel err {err.max():.3e}"


def _cmp_n(g, o, rtol=RTOL_N):
    # failed simulations: the oracle keeps the last good state, the kernel stops after the
    # failing step (include/pbe.h) -> compare n only where status == OK
    for s in range(o["n_final"].shape[0]):
        if o["status"][s] != 0:
            continue
        scale = np.max(np.abs(o["n_final"][s]))
        assert np.max(np.abs(g["n_final"][s] - o["n_final"][s])) <= rtol * scale


def _cmp_tangents(g, o, rtol=RTOL_TAN):
    a, b = g["tsamples"], o["tsamples"]
    assert np.array_equal(np.isnan(a), np.isnan(b))
    S, M, P, _ = b.shape
    for s in range(S):
        for p in range(P):
            for k in range(5):
                x, y = a[s, :, p, k], b[s, :, p, k]
                ok = ~np.isnan(y)
                if not ok.any():
                    continue
                scale = np.max(np.abs(y[ok]))
                if scale == 0:
                    assert np.all(x[ok] == 0)
                    continue
                if k == 1:   # d mu0 is 0 up to rounding (no boundary flux): compare on the lane's
                    # natural scale sum_i dL |ndot_i| ~ |d mu1| / Lbar, Lbar = mu1/mu0 from the
                    # oracle's own records at the same sample times
                    Lbar = o["samples"][s, :, 3] / o["samples"][s, :, 2]
                    scale = max(scale, np.max(np.abs(b[s, :, p, 2][ok]) / Lbar[ok]))
                assert np.max(np.abs(x[ok] - y[ok])) <= rtol * scale, (s, p, k)


def _check(w, mode=oracle.MODE_DOUBLE, **kw):
    o = oracle.run(w, mode=mode, threads=8)
    g = _gpu(w, **kw)
    assert np.array_equal(g["status"], o["status"]), (g["status"], o["status"])
    assert np.array_equal(g["steps"], o["steps"]), (g["steps"], o["steps"])
    _cmp_samples(g, o)
    _cmp_n(g, o)
    if mode != oracle.MODE_DOUBLE:
        _cmp_tangents(g, o)
        for s in range(w.n_sims):
            if o["status"][s] != 0:
                continue
            for p in range(w.n_tangents):
                sc = np.max(np.abs(o["ndot_final"][s, p]))
                assert np.max(np.abs(g["ndot_final"][s, p] - o["ndot_final"][s, p])) <= RTOL_TAN * max(sc, 1e-300)
    return g, o


# ---------------------------------------------------------------------------------------
# BASELINE configs at full size (C1-C3), reduced sims for C4/C5 plus sampled full-size runs
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("lim", [W.LIM_UPWIND, W.LIM_VANLEER])
def test_c1_growth_constant_G(lim):
    _check(W.c1_growth(lim, M=1000))


def test_c2_dissolution_full():
    g, o = _check(W.c2_dissolution())
    assert o["steps"][0] == 6000


def test_c3_temperature_cycling_full():
    g, o = _check(W.c3_cycling())
    assert o["steps"][0] == 100_000


@pytest.mark.parametrize("N", [1000, 4000])
def test_c4_steps_mode(N):
    _check(W.c4_sweep(N, batch=3, n_steps=200))


def test_c5_tangents_small():
    w = W.c5_ensemble(n_sims=18, N=300, t_max=60.0, M=60)
    g, o = _check(w, mode=oracle.MODE_DUAL)
    lo, go = oracle.loss_and_grad(o["samples"], o["tsamples"], w.target)
    assert np.allclose(g["loss"], lo, rtol=1e-9, atol=0)
    assert np.allclose(g["grad"], go, rtol=1e-8, atol=1e-9 * np.max(np.abs(go)))


@pytest.mark.parametrize("kernel", [0, 3])
def test_lognormal_seed_matches_oracle(kernel):
    """Log-normal seed through the resident (AUTO) and streaming kernels,
    with tangents."""
    w = W.c5_ensemble(n_sims=9, N=300, t_max=40.0, M=40, n_tangents=4 if kernel == 3 else 8)
    w = W.replace(w, n0=W.lognormal_seed(300, w.dL, mean=380.0, sigma=45.0)[None, :])
    g, o = _check(w, mode=oracle.MODE_DUAL, kernel=kernel)
    lo, go = oracle.loss_and_grad(o["samples"], o["tsamples"], w.target)
    assert np.allclose(g["loss"], lo, rtol=1e-9, atol=0)


EXTRA_LIMS = [W.LIM_MINMOD, W.LIM_SUPERBEE, W.LIM_MC]


@pytest.mark.parametrize("lim", EXTRA_LIMS)
def test_extra_limiters_resident_tangents(lim):
    """NEXT-4 limiters (R-31) in the resident kernel with 8 tangent lanes (branch partials)."""
    w = W.replace(W.c5_ensemble(n_sims=9, N=300, t_max=40.0, M=40), limiter=lim)
    _check(w, mode=oracle.MODE_DUAL)


@pytest.mark.parametrize("lim", EXTRA_LIMS)
def test_extra_limiters_dissolution_and_stream(lim):
    """C < 0 sweeps (dissolution) in the resident kernel and the streaming kernel."""
    w = W.replace(W.c2_dissolution(N=400, t_max=30.0, M=30), limiter=lim)
    _check(w)
    w4 = W.replace(W.c4_sweep(3000, batch=2, n_steps=200), limiter=lim)
    _check(w4, kernel=3)


@pytest.mark.parametrize("lim", EXTRA_LIMS)
def test_extra_limiters_cluster(lim):
    w = W.replace(W.c4_sweep(10000, batch=2, n_steps=100), limiter=lim)
    g, o = _check(w, kernel=2)
    assert g["info"]["kernel"] == 2


@pytest.mark.parametrize("n_params", [40, 1000])
def test_long_polynomial_primal_matches_oracle(n_params):
    """NEXT-3's long polynomials (n_params > 10) through the primal resident kernel (the
    warp-cooperative evaluation) against the oracle's power-sum loop."""
    w = W.next3_estimation(n_params=n_params, N=300, t_max=40.0, M=40)
    _check(w)


def test_long_polynomial_tangents_match_oracle():
    """Tangent lanes on a 40-term polynomial (warp-cooperative seeded evaluation): unit seeds
    on low and high coefficients plus one mixed direction."""
    w = W.next3_estimation(n_params=40, N=300, t_max=40.0, M=40)
    Q = w.sol.shape[0]
    seed = np.zeros((5, 40 + Q))
    for p, j in enumerate((0, 3, 9, 27)):
        seed[p, j] = 1.0
    seed[4, :40] = np.linspace(1.0, 0.1, 40)
    w = W.replace(w, n_tangents=5, tangent_seed=seed)
    _check(w, mode=oracle.MODE_DUAL)


def test_c5_full_size_sampled_sims():
    """C5 exactly as bench.py runs it (4096 sims x 2000 bins, 8 tangents) — oracle on 64 sims
    (stride 64; every App. B experiment and both ends of the batch)."""
    w = W.c5_ensemble()
    g = _gpu(w, want_n=False)
    assert np.all(g["status"] == 0)
    sims = list(range(0, 4096, 64)) + [4095]
    o = oracle.run(w.subset(sims), mode=oracle.MODE_DUAL, threads=os.cpu_count() or 8, want_n=False)
    gs = {k: g[k][sims] for k in ("samples", "tsamples", "status", "steps")}
    assert np.array_equal(gs["steps"], o["steps"])
    _cmp_samples(gs, o)
    _cmp_tangents(gs, o)


def test_c4_full_size_sampled_sims():
    """C4 exactly as bench.py's secondary/next4 entries run it (64 x 10^6 bins, 1000 uncapped CFL
    steps, temporal blocking by default): final records and distributions of 2 sampled sims
    against the oracle (results never depend on the batch)."""
    import torch

    import paper_2411_00742_b200 as pb
    w = W.c4_sweep(1_000_000, batch=64, n_steps=1000)
    ctx = pb.context_for(w)
    n0 = torch.from_numpy(np.ascontiguousarray(w.n0)).cuda()
    nf = torch.empty((64, w.N), dtype=torch.float64, device="cuda")
    ctx.run_batch(n0, w.c0, None, None, nf)
    r = ctx.moments()
    assert ctx.last_run_info()["steps_per_pass"] == 8
    ctx.close()
    assert np.all(r["status"] == 0) and np.all(r["steps"] == 1000)
    sims = list(range(0, 64, 4)) + [41, 63]             # 18 of 64 simulations
    o = oracle.run(w.subset(sims), threads=os.cpu_count() or 8)
    g = dict(samples=r["moments"][sims], n_final=nf[sims].cpu().numpy(), status=r["status"][sims],
             steps=r["steps"][sims])
    _cmp_samples(g, o)
    _cmp_n(g, o)


# ---------------------------------------------------------------------------------------
# edge cases
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("N", [3, 5, 31, 33, 257, 1023, 2049])
def test_ragged_sizes(N):
    w = W.c3_cycling(N=N, t_max=5.0, M=5, dt_max=0.05)
    w.n0 = np.abs(np.random.default_rng(N).standard_normal((1, N))) * 100.0
    _check(w)


@pytest.mark.parametrize("P", [1, 3, 8, 10])
def test_tangent_lane_counts(P):
    w = W.c5_ensemble(n_sims=4, N=150, t_max=20.0, M=20, n_tangents=P)
    _check(w, mode=oracle.MODE_DUAL)


def test_custom_tangent_seed_over_solubility():
    w = W.c5_ensemble(n_sims=2, N=120, t_max=10.0, M=10, n_tangents=2)
    seed = np.zeros((2, 8 + 2))
    seed[0, 8] = 1.0          # d/da (solubility prefactor)
    seed[1, 0] = 0.5; seed[1, 9] = -2.0
    w.tangent_seed = seed
    _check(w, mode=oracle.MODE_DUAL)


def test_dissolution_outflow_at_L0():
    # strong dissolution drives mass through the L = 0 face (R-25)
    w = W.c2_dissolution(N=400, t_max=200.0, M=50, dt_max=0.2)
    w.n0 = W.gaussian_seed(400, 3.0, mean=40.0, sigma=10.0, m0=0.5)[None, :]
    w.c0 = np.array([3.0])
    g, o = _check(w)
    assert o["samples"][0, -1, 2] < o["samples"][0, 0, 2]      # number left the domain


def test_per_sim_n0_and_host_n0():
    w = W.c4_sweep(2000, batch=4, n_steps=50)
    rng = np.random.default_rng(0)
    w.n0 = w.n0 * rng.uniform(0.5, 1.5, size=(4, 1))
    _check(w)
    _check(w, host_n0=True)


def test_status_codes():
    w = W.c1_growth(); w.dt_fixed = 30.0
    _check(w)                                     # CFL error before the first step
    w = W.c1_growth(); w.c0 = np.array([0.01])
    _check(w)                                     # infeasible (c < 0)
    w = W.c1_growth(); w.max_steps = 10
    _check(w)                                     # max steps


def test_determinism_independent_of_batch():
    w = W.c5_ensemble(n_sims=40, N=200, t_max=20.0, M=20)
    g_all = _gpu(w)
    g_one = _gpu(w.subset([17]))
    assert np.array_equal(g_all["samples"][17], g_one["samples"][0])
    assert np.array_equal(g_all["tsamples"][17], g_one["tsamples"][0])
    assert np.array_equal(g_all["n_final"][17], g_one["n_final"][0])
    g_again = _gpu(w)
    assert np.array_equal(g_all["samples"], g_again["samples"])


def test_uncapped_cfl_tangents_vanish():
    w = W.c4_sweep(500, batch=2, n_steps=50)
    w.n_tangents = 6
    g = _gpu(w)
    assert np.all(g["ndot_final"] == 0.0)


# ---------------------------------------------------------------------------------------
# k_stream (grid-wide HBM streaming kernel, forced) vs the oracle
# ---------------------------------------------------------------------------------------
def _stream(w, mode=oracle.MODE_DOUBLE):
    import paper_2411_00742_b200 as pb
    return _check(w, mode=mode, kernel=pb.KERNEL_STREAM)


@pytest.fixture
def plain_stream(monkeypatch):
    monkeypatch.setenv("PBE_TEMPORAL_BLOCK", "0")     # steps mode without temporal blocking


@pytest.mark.parametrize("N", [4000, 4001, 20000])
def test_stream_c4_steps_mode(N, plain_stream):
    g, o = _stream(W.c4_sweep(N, batch=3, n_steps=120))
    assert g["info"]["kernel"] == 3 and g["info"]["steps_per_pass"] == 1


def test_stream_landing_and_temperature_profile():
    _stream(W.c3_cycling(N=3000, t_max=20.0, M=20, dt_max=0.05))
    _stream(W.c2_dissolution(N=2500, t_max=30.0, M=30, dt_max=0.1))


def test_stream_dissolution_outflow():
    w = W.c2_dissolution(N=4000, t_max=100.0, M=25, dt_max=0.2)
    w.n0 = W.gaussian_seed(4000, 0.3, mean=40.0, sigma=10.0, m0=0.5)[None, :]
    w.dL = 0.3
    w.c0 = np.array([3.0])
    _stream(w)


@pytest.mark.parametrize("P", [2, 4])
def test_stream_tangent_lanes(P):
    w = W.c5_ensemble(n_sims=5, N=3000, t_max=10.0, M=10, n_tangents=P)
    _stream(w, mode=oracle.MODE_DUAL)


def test_stream_many_sims_and_statuses():
    w = W.c5_ensemble(n_sims=37, N=1500, t_max=5.0, M=5, n_tangents=0)
    w.c0 = w.c0.copy(); w.c0[3] = 0.001        # infeasible
    w.max_steps = 40                           # some sims hit MAXSTEPS
    _stream(w)


def test_stream_matches_resident():
    import paper_2411_00742_b200 as pb
    w = W.c5_ensemble(n_sims=6, N=2000, t_max=30.0, M=30, n_tangents=4)
    a = _gpu(w, kernel=pb.KERNEL_RESIDENT)
    b = _gpu(w, kernel=pb.KERNEL_STREAM)
    assert np.array_equal(a["steps"], b["steps"])
    _cmp_samples(a, b)
    _cmp_n(a, dict(b, status=b["status"]))


# ---------------------------------------------------------------------------------------
# k_cluster (thread-block cluster + DSMEM mode of the resident kernel, forced) vs the oracle
# ---------------------------------------------------------------------------------------
def _cluster(w, mode=oracle.MODE_DOUBLE):
    import paper_2411_00742_b200 as pb
    g, o = _check(w, mode=mode, kernel=pb.KERNEL_CLUSTER)
    assert g["info"]["kernel"] == 2 and g["info"]["cluster"] >= 2
    return g, o


@pytest.mark.parametrize("N", [9000, 12001, 40000])
def test_cluster_c4_steps_mode(N):
    _cluster(W.c4_sweep(N, batch=2, n_steps=100))


def test_cluster_landing_dissolution_and_cycling():
    _cluster(W.c3_cycling(N=10000, t_max=5.0, M=5, dt_max=0.02))
    _cluster(W.c2_dissolution(N=10000, t_max=20.0, M=20, dt_max=0.1))


@pytest.mark.parametrize("P", [2, 8])
def test_cluster_tangents(P):
    w = W.c5_ensemble(n_sims=3, N=5000, t_max=6.0, M=6, n_tangents=P)
    _cluster(w, mode=oracle.MODE_DUAL)


def test_cluster_statuses():
    w = W.c5_ensemble(n_sims=6, N=9000, t_max=4.0, M=4, n_tangents=0)
    w.c0 = w.c0.copy(); w.c0[2] = 0.001
    w.max_steps = 30
    _cluster(w)


# ---------------------------------------------------------------------------------------
# NEXT-4: temporal blocking of uncapped CFL steps in k_stream (steps mode, primal)
# ---------------------------------------------------------------------------------------
@pytest.fixture
def temporal_blocking(monkeypatch):
    monkeypatch.setenv("PBE_TEMPORAL_BLOCK", "1")     # read by pbe_create


@pytest.mark.parametrize("N,batch,steps", [(4000, 3, 7), (4000, 3, 8), (9001, 2, 61), (30000, 5, 100),
                                           (70001, 2, 19), (200003, 2, 17)])   # tiles 512 / 1024 / 2048
def test_temporal_blocking_matches_oracle(N, batch, steps, temporal_blocking):
    import paper_2411_00742_b200 as pb
    g, o = _check(W.c4_sweep(N, batch=batch, n_steps=steps), kernel=pb.KERNEL_STREAM)
    assert g["info"]["steps_per_pass"] == 8


def test_temporal_blocking_sign_flips_redo(temporal_blocking):
    """Supersaturation barely above 1: G changes sign every one or two steps, so most 8-step
    blocks are invalidated and their valid prefix is redone (bitwise the same sub-steps)."""
    import paper_2411_00742_b200 as pb
    w = W.c4_sweep(4000, batch=3, n_steps=40)
    w.c0 = np.array([5.782943125562973 * 1.0003, 5.782943125562973 * 1.001, 8.0])
    g, o = _check(w, kernel=pb.KERNEL_STREAM)
    assert g["info"]["steps_per_pass"] == 8


def test_temporal_blocking_max_steps_and_failure(temporal_blocking):
    """k_stream_tb stops at exactly max_steps (not at the end of its 8-step block) and, on a
    failure inside a block, redoes the valid prefix so n_final holds the failing step's state
    like every other kernel (R-26; include/pbe.h)."""
    import paper_2411_00742_b200 as pb
    w = W.c4_sweep(4000, batch=3, n_steps=40)
    w.max_steps = 13                                     # not a multiple of the block depth
    g, o = _check(w, kernel=pb.KERNEL_STREAM)
    assert g["info"]["steps_per_pass"] == 8
    assert np.all(g["status"] == 5) and np.all(g["steps"] == 13)
    # crystal mass 5000x the seed mass: the first step drives c below 0 (INFEASIBLE in step 1,
    # which is not counted: steps = completed steps)
    wf = W.c4_sweep(4000, batch=2, n_steps=40)
    wf.rho_c = 1.11e-12 * 5000.0
    g, o = _check(wf, kernel=pb.KERNEL_STREAM)
    assert np.all(g["status"] == 4) and np.all(g["steps"] == 0)
    r = _gpu(wf, kernel=pb.KERNEL_RESIDENT)             # same semantics in the resident kernel
    assert np.array_equal(r["status"], g["status"]) and np.array_equal(r["steps"], g["steps"])
    assert np.max(np.abs(r["n_final"] - g["n_final"])) <= RTOL_N * np.max(np.abs(r["n_final"]))


@pytest.mark.parametrize("kernel,N,P,steps_mode", [(1, 64, 8, False), (1, 1024, 4, False), (1, 1000, 0, True),
                                                     (2, 8192, 4, False), (3, 4096, 2, False), (3, 4096, 0, True),
                                                     (3, 131072, 0, True)])
def test_outflow_boundary_all_kernels(kernel, N, P, steps_mode, monkeypatch):
    """Mass leaving through the outflow face at L = 1200 um, N a multiple of the bins per thread
    / tile, tangents where the kernel supports them (the adjoint had a bug exactly there)."""
    if steps_mode:
        w = W.c4_sweep(N, batch=2, n_steps=60)
    else:
        w = W.c5_ensemble(n_sims=2, N=N, t_max=10.0, M=5, n_tangents=P)
    w = W.replace(w, n0=W.gaussian_seed(N, 1200.0 / N, mean=1120.0, sigma=50.0)[None, :])
    g, o = _check(w, mode=oracle.MODE_DUAL if P else oracle.MODE_DOUBLE, kernel=kernel)
    assert g["info"]["kernel"] == kernel


# ---------------------------------------------------------------------------------------
# k_resident_ws (scalar chain overlapped with the tangent sweep) and the lockstep k_resident
# ---------------------------------------------------------------------------------------
@pytest.fixture(params=["ws", "lockstep"])
def resident_kind(request, monkeypatch):
    monkeypatch.setenv("PBE_WS", "1" if request.param == "ws" else "0")   # read by pbe_create
    return request.param


def _expect_kind(g, kind):
    assert g["info"]["kernel"] == 1 and g["info"]["warp_specialized"] == (1 if kind == "ws" else 0)


def test_resident_kinds_cycling_sign_changes(resident_kind):
    """C3-shaped temperature cycling with 8 tangent lanes: G changes sign with T, so the march
    alternates between the two sweep directions (separate step loops in k_resident_ws)."""
    w = W.c3_cycling(N=600, t_max=240.0, M=24, dt_max=0.05)
    w = W.replace(w, n_tangents=6, n0=W.gaussian_seed(600, 2.0, mean=300.0, sigma=40.0)[None, :])
    g, o = _check(w, mode=oracle.MODE_DUAL)
    _expect_kind(g, resident_kind)
    s = o["samples"][0]
    assert np.any(np.diff(s[:, 1]) > 0) and np.any(np.diff(s[:, 1]) < 0)   # growth and dissolution


def test_resident_kinds_c5_loss_gradient(resident_kind):
    w = W.c5_ensemble(n_sims=12, N=900, t_max=30.0, M=30)
    g, o = _check(w, mode=oracle.MODE_DUAL)
    _expect_kind(g, resident_kind)
    lo, go = oracle.loss_and_grad(o["samples"], o["tsamples"], w.target)
    assert np.allclose(g["loss"], lo, rtol=1e-9, atol=0)
    assert np.allclose(g["grad"], go, rtol=1e-8, atol=1e-9 * np.max(np.abs(go)))


def test_resident_kinds_failure_with_tangents(resident_kind):
    """INFEASIBLE part-way through a tangent run: earlier records valid, later ones NaN (R-26),
    loss and gradient NaN, the other simulations unaffected."""
    w = W.c5_ensemble(n_sims=3, N=400, t_max=20.0, M=20)
    # constant G = 3 um/min regardless of S: the crystal mass grows until sim 1 (c0 = 0.05 g/kg)
    # runs out of solute; 8 lanes seeded over (G, a, b) so every lane is non-trivial
    seed = np.random.default_rng(5).standard_normal((8, 3))
    w = W.replace(w, law=W.LAW_CONST, theta=np.full((3, 1), 3.0), c0=np.array([w.c0[0], 0.05, w.c0[2]]),
                  tangent_seed=seed)
    g, o = _check(w, mode=oracle.MODE_DUAL)
    _expect_kind(g, resident_kind)
    assert g["status"][1] == 4 and g["status"][0] == 0 and g["status"][2] == 0
    assert np.isnan(g["loss"][1]) and np.all(np.isnan(g["grad"][1])) and np.all(np.isfinite(g["grad"][0]))


def test_resident_kinds_steps_mode_and_lane_counts(resident_kind):
    """Steps mode with capped steps (tangents do not vanish) and 5 lanes of an 8-lane kernel."""
    w = W.c5_ensemble(n_sims=2, N=500, t_max=10.0, M=10, n_tangents=5)
    w = W.replace(w, n_steps=77, t_samples=np.array([1.0]), target=None)
    g, o = _check(w, mode=oracle.MODE_DUAL)
    _expect_kind(g, resident_kind)
    assert np.all(g["steps"] == 77) and np.any(g["ndot_final"] != 0.0)


def test_tail_wave_half_lane_ctas_bitwise():
    """A last partial wave of <= 74 simulations runs as two 4-lane CTAs per simulation (second
    launch, kp.G = 2).  Results must be bitwise those of the one-CTA march of the same simulation
    (the primal is recomputed identically; every tangent reduction has the same order)."""
    w = W.c5_ensemble(n_sims=148, N=300, t_max=15.0, M=15)
    g_full = _gpu(w)                                     # 148 sims: one full wave, no split
    assert g_full["info"]["launches"] == 1 and g_full["info"]["ctas"] == 148
    for sims in ([17], [3, 90, 147]):                    # tails of 1 and 3 simulations: split
        g = _gpu(w.subset(sims))
        assert g["info"]["launches"] == 1 and g["info"]["ctas"] == 2 * len(sims)
        for k in ("samples", "tsamples", "n_final", "ndot_final", "loss", "grad", "status", "steps"):
            assert np.array_equal(g[k], g_full[k][sims], equal_nan=True), k
    w150 = W.c5_ensemble(n_sims=150, N=300, t_max=15.0, M=15)
    g150 = _gpu(w150)                                    # 148 full CTAs + 2 x 2 half CTAs
    assert g150["info"]["launches"] == 2 and g150["info"]["ctas"] == 152
    o = oracle.run(w150.subset([0, 148, 149]), mode=oracle.MODE_DUAL, threads=3)
    gs = {k: g150[k][[0, 148, 149]] for k in ("samples", "tsamples", "status", "steps")}
    _cmp_samples(gs, o)
    _cmp_tangents(gs, o)
