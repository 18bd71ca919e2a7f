"""NEXT-2: batched parameter estimation on the tangent ensemble (§4.1, App. B
L734-744, App. C).

The paper fits the polynomial growth law (eq-poly_growth_rate, L565-571) to 9 in-silico
experiments (T in {10, 15, 20} C x S0 in {1.15, 1.25, 1.5}) by Adam (lr 0.01, beta1 0.9,
beta2 0.999, 100 iterations, theta >= 0, L756-762) on the residual sum of squares (L764).

B200 design: R independent estimations (e.g. multi-start) advance together.  One Adam
iteration = ONE pbe_run_batch of R x 9 simulations with k forward-mode tangent lanes (one
per coefficient) — the loss of every simulation and its exact gradient come out of the same
launch (row a7/a8) — then the Adam update of the R parameter vectors (host, R x k numbers).
No finite differences and no reverse pass are needed for k <= 10.  For more coefficients
(the paper's 1000-parameter regime, L599) grad_mode="adjoint" takes the gradient from the
discrete adjoint instead (pbe_run_adjoint, NEXT-3): same loss, cost independent of k.

In-silico data (R-28): the paper generated its targets with the method of moments and the
Arrhenius truth (L741-743).  Here the targets are produced by the same FVM march with the
Arrhenius truth (Table A.1 dimension-1 constants), on the GPU; tests/test_oracle_pins.py
(PIN-12) shows FVM and MOM agree within 1% at these resolutions.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import LAW_ARRHENIUS_GD, LAW_POLY, SOL_EXP, Context

APPB_T = (10.0, 15.0, 20.0)
APPB_S0 = (1.15, 1.25, 1.5)
# c*(T) = 3.37 exp(0.036 T) at APPB_T (Eq. A.1, Table A.1 constants) as input data: the product
# evaluates no kinetics on the host (workloads.APPB_CSAT holds the same numbers; a CPU test
# re-derives them through the oracle)
APPB_CSAT = (4.8303201270683465, 5.782943125562973, 6.923439919869901)
SOL_DEFAULT = (3.37, 0.036)


@dataclass
class Experiments:
    """The 9 App. B experiments on one grid: per-experiment T, c0 and target traces."""
    N: int
    dL: float
    n0: np.ndarray          # [N] seed (shared)
    T: np.ndarray           # [9]
    c0: np.ndarray          # [9]
    t_samples: np.ndarray   # [M]
    target: np.ndarray      # [9][M][2] (c, mean length)
    sol: tuple = (3.37, 0.036)
    dt_max: float = 0.05
    rho_c: float = 1.11e-12
    k_v: float = math.pi / 4


def make_experiments(N: int, n0: np.ndarray, t_max: float = 600.0, M: int = 600, dt_max: float = 0.05,
                     truth=(8.86e6, 2.45e3, 3.7), sol=SOL_DEFAULT, csat=None, device: int = 0) -> Experiments:
    """App. B in-silico campaign: c0 = S0 c*(T) for the 3 x 3 grid, targets (c, mu1/mu0)
    sampled at M uniform times from the GPU FVM with the Arrhenius truth (R-28).  csat: c*(T)
    at the three temperatures APPB_T (input data; defaults to APPB_CSAT for the Table A.1
    solubility, required for any other `sol`)."""
    import torch
    dL = 1200.0 / N
    if csat is None:
        if tuple(sol) != SOL_DEFAULT:
            raise ValueError("make_experiments: pass csat = c*(T) at APPB_T for a non-default solubility")
        csat = APPB_CSAT
    T = np.repeat(np.array(APPB_T), 3)
    S0 = np.tile(np.array(APPB_S0), 3)
    c0 = S0 * np.repeat(np.asarray(csat, dtype=np.float64), 3)
    t = np.linspace(t_max / M, t_max, M)
    ctx = Context(N, dL, dt_max=dt_max, n_samples=M, max_sims=9, device=device)
    ctx.set_kinetics(LAW_ARRHENIUS_GD, np.tile(np.array(truth), (9, 1)), SOL_EXP, np.array(sol),
                     np.array([0.0]), T[:, None])
    ctx.run_batch(torch.from_numpy(np.ascontiguousarray(n0[None, :])).cuda(device), c0, t)
    out = ctx.moments()
    ctx.close()
    if not np.all(out["status"] == 0):
        raise RuntimeError(f"truth simulation failed: {out['status']}")
    m = out["moments"]
    target = np.stack([m[:, :, 1], m[:, :, 3] / m[:, :, 2]], axis=-1)
    return Experiments(N=N, dL=dL, n0=n0, T=T, c0=c0, t_samples=t, target=target, sol=sol, dt_max=dt_max)


@dataclass
class AdamState:
    """Adam (L756-762) for R parameter vectors of length k, with theta >= 0 projection."""
    theta: np.ndarray                       # [R][k]
    lr: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    m: Optional[np.ndarray] = None
    v: Optional[np.ndarray] = None
    it: int = 0

    def step(self, grad: np.ndarray) -> None:
        if self.m is None:
            self.m = np.zeros_like(self.theta)
            self.v = np.zeros_like(self.theta)
        self.it += 1
        self.m = self.beta1 * self.m + (1.0 - self.beta1) * grad
        self.v = self.beta2 * self.v + (1.0 - self.beta2) * grad * grad
        mh = self.m / (1.0 - self.beta1 ** self.it)
        vh = self.v / (1.0 - self.beta2 ** self.it)
        self.theta = np.maximum(self.theta - self.lr * mh / (np.sqrt(vh) + self.eps), 0.0)


@dataclass
class Estimator:
    """R independent fits of the k-coefficient polynomial growth law to the experiments."""
    exps: Experiments
    theta0: np.ndarray                      # [R][k] initial parameters (>= 0)
    lr: float = 0.01
    device: int = 0
    grad_mode: str = "auto"                 # "tangent" (k <= 10), "adjoint", "auto"
    history: list = field(default_factory=list)

    def __post_init__(self):
        import torch
        self.theta0 = np.atleast_2d(np.asarray(self.theta0, dtype=np.float64))
        self.R, self.k = self.theta0.shape
        if self.grad_mode == "auto":
            self.grad_mode = "tangent" if self.k <= 10 else "adjoint"
        if self.grad_mode == "tangent" and self.k > 10:
            raise ValueError("at most 10 parameters with tangent lanes (use grad_mode='adjoint')")
        e = self.exps
        M = e.t_samples.shape[0]
        adj = self.grad_mode == "adjoint"
        # the adjoint's trace is sized by max_steps: bound it by the sample horizon
        max_steps = int(1.2 * e.t_samples[-1] / e.dt_max) + 1000 if adj else 10_000_000
        self.ctx = Context(e.N, e.dL, dt_max=e.dt_max, n_samples=M, n_tangents=0 if adj else self.k,
                           max_sims=self.R * 9, device=self.device, rho_c=e.rho_c, k_v=e.k_v, max_steps=max_steps)
        self.n0 = torch.from_numpy(np.ascontiguousarray(e.n0[None, :])).cuda(self.device)
        self.c0 = np.tile(e.c0, self.R)
        self.T = np.tile(e.T, self.R)[:, None]
        self.target = np.tile(e.target, (self.R, 1, 1))
        self.adam = AdamState(self.theta0.copy(), lr=self.lr)

    def loss_and_grad(self, theta: np.ndarray):
        """Total RSS over the 9 experiments and its gradient for every fit: one launch of
        R x 9 simulations with k tangent lanes."""
        e = self.exps
        th = np.repeat(theta, 9, axis=0)                    # sim r*9 + j runs fit r on experiment j
        self.ctx.set_kinetics(LAW_POLY, th, SOL_EXP, np.array(e.sol), np.array([0.0]), self.T)
        if self.grad_mode == "adjoint":
            self.ctx.run_adjoint(self.n0, self.c0, e.t_samples, self.target)
            g = self.ctx.adjoint_gradient(self.k)["grad"]
            out = self.ctx.moments()
        else:
            self.ctx.run_batch(self.n0, self.c0, e.t_samples, self.target)
            out = self.ctx.moments()
            g = self.ctx.tangents()["grad"]
        ok = out["status"] == 0
        loss = np.where(ok, out["loss"], np.inf).reshape(self.R, 9).sum(axis=1)
        grad = np.where(ok[:, None], g, 0.0).reshape(self.R, 9, self.k).sum(axis=1)
        return loss, grad, out["status"].reshape(self.R, 9)

    def run(self, iterations: int = 100):
        """App. C: `iterations` Adam steps with no convergence test (L760)."""
        for _ in range(iterations):
            loss, grad, status = self.loss_and_grad(self.adam.theta)
            self.history.append(dict(theta=self.adam.theta.copy(), loss=loss.copy(), status=status))
            self.adam.step(grad)
        loss, _, status = self.loss_and_grad(self.adam.theta)
        self.history.append(dict(theta=self.adam.theta.copy(), loss=loss.copy(), status=status))
        return self.adam.theta, loss

    def close(self):
        self.ctx.close()
