"""1D method of moments (SI eq-mom2D, reduced to one length):
    d mu_k / dt = k G mu_{k-1}          (k = 0..3, size-independent growth)
    d c / dt    = -rho_c k_v d mu_3/dt = -3 rho_c k_v G mu_2      (eq-mass_balance, L271)
with G = G(S = c/c*(T(t)), T(t)), integrated by classical fixed-step RK4 (the paper used
scipy odeint, L463; fixed-step RK4 is verifiable by step halving).  Used only as a pin for
the oracle (DESIGN.md PIN-12).  Kinetics are re-typed here from Eq. A.1/A.2 and
eq-poly_growth_rate so the check does not route through oracle/."""
import math

import numpy as np


def _T(w, s, t):
    kt, kT = w.knot_t, w.knot_T[s if w.knot_T.shape[0] > 1 else 0]
    if len(kt) == 1 or t <= kt[0]:
        return kT[0]
    if t >= kt[-1]:
        return kT[-1]
    return float(np.interp(t, kt, kT))


def _G(w, s, c, t):
    T = _T(w, s, t)
    sol = w.sol
    cs = sol[0] * math.exp(sol[1] * T) if w.sol_kind == 0 else sol[0] + sol[1] * T + sol[2] * T * T
    S = c / cs
    th = w.theta[s]
    if w.law == 0:
        return th[0]
    if w.law == 1:
        if S > 1:
            return th[0] * math.exp(-th[1] / (T + 273.15)) * (S - 1) ** th[2]
        if S < 1 and len(th) >= 6:
            return -th[3] * math.exp(-th[4] / (T + 273.15)) * (1 - S) ** th[5]
        return 0.0
    return sum(th[j] * (S - 1) ** (j + 1) for j in range(len(th))) if S > 1 else 0.0


def rhs(w, s, y, t):
    c, mu = y[0], y[1:]
    G = _G(w, s, c, t)
    dmu = np.array([0.0, G * mu[0], 2 * G * mu[1], 3 * G * mu[2]])
    return np.concatenate([[-w.rho_c * w.k_v * dmu[3]], dmu])


def solve(w, mu_init, t_end, n_steps, s=0):
    """Returns (c, mu0, mu1, mu2, mu3) at t_end, starting from the discrete seed moments."""
    y = np.concatenate([[w.c0[s]], np.asarray(mu_init, dtype=np.float64)])
    h = t_end / n_steps
    t = 0.0
    for _ in range(n_steps):
        k1 = rhs(w, s, y, t)
        k2 = rhs(w, s, y + 0.5 * h * k1, t + 0.5 * h)
        k3 = rhs(w, s, y + 0.5 * h * k2, t + 0.5 * h)
        k4 = rhs(w, s, y + h * k3, t + h)
        y = y + (h / 6.0) * (k1 + 2 * k2 + 2 * k3 + k4)
        t += h
    return y
