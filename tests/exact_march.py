"""Brute-force march in exact rational (fractions.Fraction) or 50-digit (mpmath) arithmetic.

A PIN for the oracle (DESIGN.md PIN-9), written independently of oracle/pbe_oracle.cpp:
  * the FVM step is in FLUX form with the one-division harmonic limited slope
        psi(a, b) = 2ab/(a+b) if ab > 0 else 0        (= phi_vanLeer(a/b) * b, SI L853-856)
        C >= 0: F_{i-1/2} = C n_{i-1} + kappa psi(d_{i-1}, d_i)
        C <  0: F_{i-1/2} = C n_i     + kappa psi(d_{i+1}, d_i)      (LeVeque's wave form)
        n_i <- n_i - (F_{i+1/2} - F_{i-1/2}),  kappa = |C|(1-|C|)/2,  d_i = n_i - n_{i-1}
    whereas the oracle evaluates eq-highRes_growth literally with theta/phi and obtains
    the dissolution branch by mirroring — so an index, sign or limiter mistake in either
    shows up as a mismatch;
  * no rounding at all (Fraction) or 50 significant digits (mpmath, for exp-based kinetics).
Sized for ~10 bins and a handful of steps (denominators grow fast under the coupling).
"""
from __future__ import annotations

import math
from fractions import Fraction

import mpmath


class Num:
    """Number system: exact rationals or mpmath at `dps` digits."""

    def __init__(self, kind: str = "fraction", dps: int = 50):
        self.kind = kind
        if kind == "mp":
            self.ctx = mpmath.mp.clone()
            self.ctx.dps = dps

    def __call__(self, x):
        if self.kind == "fraction":
            return Fraction(x)
        return self.ctx.mpf(x)

    def exp(self, x):
        assert self.kind == "mp", "exp needs the mpmath number system"
        return self.ctx.exp(x)

    def log(self, x):
        assert self.kind == "mp", "log needs the mpmath number system"
        return self.ctx.log(x)


def psi(a, b, limiter):
    if limiter == 0:
        return 0
    if not a * b > 0:
        return 0
    if limiter == 1:
        return 2 * a * b / (a + b)
    # NEXT-4 limiters as slope limiters on |a|, |b| with the sign of b (R-31): minmod,
    # superbee, MC (Sweby's region; LeVeque, "Finite Volume Methods", eqs. 6.39-6.44)
    A, B = abs(a), abs(b)
    sgn = 1 if b > 0 else -1
    if limiter == 2:
        m = min(A, B)
    elif limiter == 3:
        m = max(min(2 * A, B), min(A, 2 * B))
    else:
        m = min(2 * A, (A + B) / 2, 2 * B)
    return sgn * m


def flux_step(n, Cn, limiter):
    """One step in flux form (exact in the chosen number system)."""
    N = len(n)
    g = lambda i: n[i] if 0 <= i < N else 0
    d = lambda i: g(i) - g(i - 1)
    aC = Cn if Cn >= 0 else -Cn
    kappa = aC * (1 - aC) / 2
    F = []
    for i in range(N + 1):          # face i - 1/2
        if Cn >= 0:
            F.append(Cn * g(i - 1) + kappa * psi(d(i - 1), d(i), limiter))
        else:
            F.append(Cn * g(i) + kappa * psi(d(i + 1), d(i), limiter))
    return [n[i] - (F[i + 1] - F[i]) for i in range(N)]


def temperature(num, knot_t, knot_T, t):
    if len(knot_t) == 1 or t <= knot_t[0]:
        return num(knot_T[0])
    if t >= knot_t[-1]:
        return num(knot_T[-1])
    k = max(j for j in range(len(knot_t) - 1) if knot_t[j] <= t)
    slope = (num(knot_T[k + 1]) - num(knot_T[k])) / (num(knot_t[k + 1]) - num(knot_t[k]))
    return num(knot_T[k]) + slope * (t - num(knot_t[k]))


def solubility(num, sol_kind, sol, T):
    if sol_kind == 0:
        return num(sol[0]) * num.exp(num(sol[1]) * T)
    return num(sol[0]) + num(sol[1]) * T + num(sol[2]) * T * T


def growth(num, law, theta, S, T):
    th = [num(x) for x in theta]
    if law == 0:
        return th[0]
    if law == 1:
        if S > 1:
            return th[0] * num.exp(-th[1] / (T + num("273.15"))) * num.exp(th[2] * num.log(S - 1))
        if S < 1 and len(th) >= 6:
            return -(th[3] * num.exp(-th[4] / (T + num("273.15"))) * num.exp(th[5] * num.log(1 - S)))
        return num(0)
    if S > 1:
        return sum(th[j] * (S - 1) ** (j + 1) for j in range(len(th)))
    return num(0)


def march(num, *, N, dL, L_lo, limiter, courant, dt_fixed, dt_max, law, theta, sol_kind, sol,
          knot_t, knot_T, n0, c0, rho_c, k_v, t_samples=None, n_steps=0):
    """Returns (records [(t, c, mu0..mu3)], n_final, steps).  Inputs may be Fractions,
    strings or floats (converted exactly)."""
    n = [num(x) for x in n0]
    c = num(c0)
    t = num(0)
    L = [num(L_lo) + (num(i) + num("0.5")) * num(dL) for i in range(N)]
    dLn = num(dL)
    rk = num(rho_c) * num(k_v)

    def mom(v):
        return [sum(dLn * L[i] ** k * v[i] for i in range(N)) for k in range(4)]

    mu3_prev = mom(n)[3]
    recs, steps, m = [], 0, 0
    while (n_steps and steps < n_steps) or (not n_steps and m < len(t_samples)):
        T = temperature(num, knot_t, knot_T, t)
        S = c / solubility(num, sol_kind, sol, T)
        G = growth(num, law, theta, S, T)
        inf = None
        if dt_fixed:
            dt = num(dt_fixed)
            Cn = G * dt / dLn
            assert abs(Cn) <= 1
        elif G != 0:
            dt_cfl = num(courant) * dLn / abs(G)
            if dt_max is not None and num(dt_max) < dt_cfl:
                dt = num(dt_max)
                Cn = G * dt / dLn
            else:
                dt = dt_cfl
                Cn = num(courant) if G > 0 else -num(courant)
        else:
            dt = num(dt_max) if dt_max is not None else inf
            Cn = num(0)
        landing = False
        if n_steps and dt is None:
            dt = num(0)                      # steps mode, G = 0, no cap: a no-op step
        if not n_steps:
            tn = num(t_samples[m])
            if dt is None or t + dt >= tn - num("1e-9") * dt:
                dtl = tn - t
                Cl = G * dtl / dLn
                if abs(Cl) <= 1:
                    dt, Cn, landing = dtl, Cl, True
        n = flux_step(n, Cn, limiter)
        assert min(n) >= 0, "exact arithmetic never produces a negative density (TVD)"
        mu = mom(n)
        c = c - rk * (mu[3] - mu3_prev)
        mu3_prev = mu[3]
        t = tn if landing else t + dt
        steps += 1
        if landing:
            recs.append((t, c, *mu))
            m += 1
    if n_steps:
        recs.append((t, c, *mom(n)))
    return recs, n, steps


def march_2d(num, *, N1, N2, dL1, dL2, limiter, dt_fixed, law, theta, sol_kind, sol, T, f0, c0, rho_c, k_v,
             t_samples, courant=None, dt_max=None, binding=None):
    """Exact 2D Godunov-split march (rows along L1, then columns along L2, flux form) landing
    on the sample times; returns records (t, c, mu00, mu10, mu01, mu11, mu02, mu12) and the
    final field [N2][N1].  dt_fixed > 0: fixed dt; otherwise the SI's CFL rule (PAPER.md
    L857-861) dt = nu min(dL1/|G1|, dL2/|G2|) (a zero rate does not limit), capped by dt_max.
    `binding` (a list) receives, per CFL step, which dimension set dt (1, 2 or 0 = dt_max)."""
    f = [[num(f0[j * N1 + i]) for i in range(N1)] for j in range(N2)]
    c, t = num(c0), num(0)
    L1 = [(num(i) + num("0.5")) * num(dL1) for i in range(N1)]
    L2 = [(num(j) + num("0.5")) * num(dL2) for j in range(N2)]
    w = num(dL1) * num(dL2)
    PQ = [(0, 0), (1, 0), (0, 1), (1, 1), (0, 2), (1, 2)]
    mom = lambda g: [sum(w * L1[i] ** p * L2[j] ** q * g[j][i] for j in range(N2) for i in range(N1)) for p, q in PQ]
    H = len(theta) // 2
    mu12 = mom(f)[5]
    recs, m = [], 0
    Tn = num(T)
    while m < len(t_samples):
        S = c / solubility(num, sol_kind, sol, Tn)
        G1 = growth(num, law, theta[:H], S, Tn)
        G2 = growth(num, law, theta[H:], S, Tn)
        if dt_fixed:
            dt = num(dt_fixed)
        else:
            cand = []
            if G1 != 0:
                cand.append((num(courant) * num(dL1) / abs(G1), 1))
            if G2 != 0:
                cand.append((num(courant) * num(dL2) / abs(G2), 2))
            if dt_max is not None:
                cand.append((num(dt_max), 0))
            dt, who = min(cand, key=lambda e: e[0]) if cand else (None, -1)   # None: unbounded
            if binding is not None:
                binding.append(who)
        tn = num(t_samples[m])
        landing = dt is None or t + dt >= tn - num("1e-9") * dt
        if landing:
            dt = tn - t
        C1, C2 = G1 * dt / num(dL1), G2 * dt / num(dL2)
        f = [flux_step(row, C1, limiter) for row in f]
        cols = [flux_step([f[j][i] for j in range(N2)], C2, limiter) for i in range(N1)]
        f = [[cols[i][j] for i in range(N1)] for j in range(N2)]
        mu = mom(f)
        c = c - num(rho_c) * num(k_v) * (mu[5] - mu12)
        mu12 = mu[5]
        t = tn if landing else t + dt
        if landing:
            recs.append((t, c, *mu))
            m += 1
    return recs, f
