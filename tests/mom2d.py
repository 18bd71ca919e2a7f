"""2D method of moments (SI eq-mom2D): for the six cross moments
(p, q) in {(0,0),(1,0),(0,1),(1,1),(0,2),(1,2)}:  d mu_pq/dt = p G1 mu_{p-1,q} + q G2 mu_{p,q-1},
and dc/dt = -rho_c k_v d mu_12/dt (eq-mass_balance, L271) = -rho_c k_v (G1 mu_02 + 2 G2 mu_11).
Fixed-step RK4; a pin for the 2D oracle (kinetics re-typed from Eq. A.1/A.2)."""
import math

import numpy as np


def _G(th, S, T):
    if S <= 1:
        return 0.0
    return th[0] * math.exp(-th[1] / (T + 273.15)) * (S - 1) ** th[2]


def solve(w, mu_init, t_end, n_steps, s=0):
    T = w.knot_T[0][0]
    cs = w.sol[0] * math.exp(w.sol[1] * T)
    th = w.theta[s]
    H = len(th) // 2
    rk = w.rho_c * w.k_v

    def rhs(y):
        c, m00, m10, m01, m11, m02, m12 = y
        G1, G2 = _G(th[:H], c / cs, T), _G(th[H:], c / cs, T)
        d = np.array([0.0, G1 * m00, G2 * m00, G1 * m01 + G2 * m10, 2 * G2 * m01, G1 * m02 + 2 * G2 * m11])
        return np.concatenate([[-rk * d[5]], d])

    y = np.concatenate([[w.c0[s]], mu_init])
    h = t_end / n_steps
    for _ in range(n_steps):
        k1 = rhs(y); k2 = rhs(y + 0.5 * h * k1); k3 = rhs(y + 0.5 * h * k2); k4 = rhs(y + h * k3)
        y = y + (h / 6.0) * (k1 + 2 * k2 + 2 * k3 + k4)
    return y
