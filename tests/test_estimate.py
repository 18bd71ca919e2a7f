"""NEXT-2: batched Adam parameter estimation on the tangent ensemble.
CPU: Adam arithmetic (App. C).  GPU: gradient = finite differences of the GPU loss,
trajectory = an oracle-driven Adam on the same data, loss decreases over the paper's 100
iterations."""
import numpy as np
import pytest

import workloads as W
from paper_2411_00742_b200.estimate import AdamState


def test_adam_zero_gradient_keeps_theta():
    a = AdamState(np.array([[0.3, 0.7]]))
    a.step(np.zeros((1, 2)))
    assert np.array_equal(a.theta, [[0.3, 0.7]])


def test_adam_first_step_is_lr_sized_and_projected():
    a = AdamState(np.array([[1.0, 0.005]]), lr=0.01)
    a.step(np.array([[2.5, 1.0]]))
    # bias-corrected m = g, v = g^2 -> step lr * g / (|g| + eps); theta >= 0 (L762)
    assert a.theta[0, 0] == pytest.approx(1.0 - 0.01 * 2.5 / (2.5 + 1e-8), rel=1e-15)
    assert a.theta[0, 1] == 0.0


def test_adam_matches_textbook_recurrence():
    rng = np.random.default_rng(0)
    th = rng.random((3, 4)); a = AdamState(th.copy(), lr=0.01)
    m = np.zeros_like(th); v = np.zeros_like(th)
    for it in range(1, 6):
        g = rng.standard_normal(th.shape)
        a.step(g)
        m = 0.9 * m + 0.1 * g; v = 0.999 * v + 0.001 * g * g
        th = np.maximum(th - 0.01 * (m / (1 - 0.9 ** it)) / (np.sqrt(v / (1 - 0.999 ** it)) + 1e-8), 0)
        assert np.allclose(a.theta, th, rtol=1e-14, atol=0)


@pytest.fixture(scope="module")
def exps():
    from paper_2411_00742_b200.estimate import make_experiments
    N = 240
    return make_experiments(N, W.gaussian_seed(N, 1200.0 / N), t_max=60.0, M=60)


THETA0 = np.array([[0.4, 4.0, 16.0, 40.0]])


@pytest.mark.gpu
def test_estimator_gradient_matches_finite_differences(exps):
    from paper_2411_00742_b200.estimate import Estimator
    est = Estimator(exps, THETA0)
    loss, grad, st = est.loss_and_grad(est.theta0)
    assert np.all(st == 0)
    for j in range(4):
        h = 1e-4 * THETA0[0, j]
        tp = THETA0.copy(); tp[0, j] += h
        tm = THETA0.copy(); tm[0, j] -= h
        fd = (est.loss_and_grad(tp)[0][0] - est.loss_and_grad(tm)[0][0]) / (2 * h)
        assert grad[0, j] == pytest.approx(fd, rel=2e-4)
    est.close()


@pytest.mark.gpu
def test_estimator_trajectory_matches_oracle_adam(exps):
    import oracle
    from paper_2411_00742_b200.estimate import Estimator
    est = Estimator(exps, THETA0)
    est.run(3)
    # oracle-driven Adam on the same data
    th = THETA0.copy(); m = np.zeros_like(th); v = np.zeros_like(th)
    for it in range(1, 4):
        w = W.Workload(name="est", N=exps.N, dL=exps.dL, dt_max=exps.dt_max, law=W.LAW_POLY,
                       theta=np.repeat(th, 9, axis=0), sol_kind=W.SOL_EXP, sol=np.array(exps.sol),
                       knot_t=np.array([0.0]), knot_T=exps.T[:, None], n0=exps.n0[None, :], c0=exps.c0,
                       t_samples=exps.t_samples, target=exps.target, n_tangents=4)
        r = oracle.run(w, mode=oracle.MODE_DUAL, threads=9, want_n=False)
        _, g = oracle.loss_and_grad(r["samples"], r["tsamples"], exps.target)
        g = g.sum(axis=0, keepdims=True)
        m = 0.9 * m + 0.1 * g; v = 0.999 * v + 0.001 * g * g
        th = np.maximum(th - 0.01 * (m / (1 - 0.9 ** it)) / (np.sqrt(v / (1 - 0.999 ** it)) + 1e-8), 0)
        assert np.allclose(est.history[it]["theta"], th, rtol=1e-9, atol=0), it
    est.close()


@pytest.mark.gpu
def test_multistart_estimation_reduces_loss(exps):
    from paper_2411_00742_b200.estimate import Estimator
    rng = np.random.default_rng(3)
    theta0 = THETA0 * np.exp(0.3 * rng.standard_normal((6, 4)))
    est = Estimator(exps, theta0, lr=0.05)
    theta, loss = est.run(100)
    l0 = est.history[0]["loss"]
    assert np.all(np.isfinite(loss)) and np.all(theta >= 0)
    assert np.all(loss < 0.5 * l0), (l0, loss)
    est.close()


@pytest.mark.gpu
def test_adjoint_estimator_matches_tangent_estimator(exps):
    """grad_mode='adjoint' (NEXT-3) drives the same Adam trajectory as the tangent lanes."""
    from paper_2411_00742_b200.estimate import Estimator
    et = Estimator(exps, THETA0, grad_mode="tangent")
    ea = Estimator(exps, THETA0, grad_mode="adjoint")
    lt, gt, _ = et.loss_and_grad(THETA0)
    la, ga, _ = ea.loss_and_grad(THETA0)
    assert np.allclose(la, lt, rtol=1e-12, atol=0)
    assert np.allclose(ga, gt, rtol=1e-9, atol=1e-12 * np.abs(gt).max())
    et.run(3); ea.run(3)
    for it in range(4):
        assert np.allclose(ea.history[it]["theta"], et.history[it]["theta"], rtol=1e-9, atol=0), it
    et.close(); ea.close()


@pytest.mark.gpu
def test_adjoint_estimator_many_coefficients(exps):
    """40 polynomial coefficients (beyond the 10 tangent lanes): Adam on adjoint gradients
    lowers the RSS."""
    from paper_2411_00742_b200.estimate import Estimator
    th0 = np.zeros((2, 40))
    th0[:, :4] = THETA0 * np.array([[1.0], [1.3]])
    th0[:, 4:] = 0.01
    est = Estimator(exps, th0, lr=0.05)
    assert est.grad_mode == "adjoint"
    theta, loss = est.run(20)
    assert np.all(np.isfinite(loss)) and np.all(theta >= 0)
    assert np.all(loss < est.history[0]["loss"]), (est.history[0]["loss"], loss)
    est.close()
