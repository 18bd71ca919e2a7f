// =====================================================================================
//  oracle/pbe_oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
//  A plain, slow, serial CPU implementation of the explicit high-resolution FVM
//  time-march of the 1D crystal population balance + solute mass balance of
//  arXiv 2411.00742 (§2.1, SI §S1).  It exists so
//  that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg can check
//  and time the CUDA path.  The product path (paper_2411_00742_b200/) never loads
//  this file or its .so; the two share no code, headers, tables or helpers.
//
//  Scalar type is a template parameter so the SAME march runs on
//     double                       (primal),
//     Dual  (value + 10 tangents)  (forward-mode AD, Table S1),
//     std::complex<double>         (complex-step derivative, used only as a pin).
//
//  Every step follows DESIGN.md "Oracle definition" in the paper's order:
//     1. kinetics at t^n  : T(t^n), c* (Eq. A.1), S = c/c* (L285),
//                           G (Eq. A.2, L699-705 / Eq. poly_growth_rate)
//     2. time step        : CFL  dt = nu*dL/|G|  (SI L857-861, nu = 0.9 L301),
//                           capped by dt_max and by the next sample time (R-8)
//     3. FVM update       : eq-highRes_growth (L292-298) with the van Leer limiter
//                           (SI L849-856), written out literally (theta, phi);
//                           G < 0 uses the mirror image of the same formula (R-6)
//     4. clip of round-off negatives (R-17)
//     5. moments          : mu_k = sum_i dL * L_i^k * n_i (SI eq-moment2D L871-875,
//                           midpoint rule R-11), Neumaier-compensated
//     6. mass balance     : c^{n+1} = c^n - rho_c k_v (mu3^{n+1} - mu3^n)
//                           (eq-discrete_mass_balance, L304-312)
//     7. sampling         : record (t, c, mu0..mu3) when t^{n+1} lands on a sample time
//
//  Parity pins for this file live in tests/test_oracle_pins.py (closed forms, exact
//  rational brute force, method of moments, conservation, translation, complex step).
// =====================================================================================
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

namespace oracle {

constexpr int MAXP = 10;  // tangent lanes carried by Dual (north star: 6-10 parameters)

// ----------------------------------------------------------------------------------
// Scalar types.  Dual: forward-mode AD ("each primitive is augmented
// with its corresponding derivative (called a tangent)").  All lanes are always
// carried; unused lanes stay zero.
// ----------------------------------------------------------------------------------
struct Dual {
    double v;
    double d[MAXP];
    Dual() : v(0.0) { for (int p = 0; p < MAXP; ++p) d[p] = 0.0; }
    Dual(double x) : v(x) { for (int p = 0; p < MAXP; ++p) d[p] = 0.0; }
};
inline Dual operator+(const Dual& a, const Dual& b) { Dual r(a.v + b.v); for (int p = 0; p < MAXP; ++p) r.d[p] = a.d[p] + b.d[p]; return r; }
inline Dual operator-(const Dual& a, const Dual& b) { Dual r(a.v - b.v); for (int p = 0; p < MAXP; ++p) r.d[p] = a.d[p] - b.d[p]; return r; }
inline Dual operator-(const Dual& a) { Dual r(-a.v); for (int p = 0; p < MAXP; ++p) r.d[p] = -a.d[p]; return r; }
inline Dual operator*(const Dual& a, const Dual& b) { Dual r(a.v * b.v); for (int p = 0; p < MAXP; ++p) r.d[p] = a.d[p] * b.v + a.v * b.d[p]; return r; }
inline Dual operator/(const Dual& a, const Dual& b) {
    // (a/b)' = (a' - (a/b) b') / b   (no b^2: b can be ~1e-160 in Gaussian tails)
    Dual r(a.v / b.v);
    for (int p = 0; p < MAXP; ++p) r.d[p] = (a.d[p] - r.v * b.d[p]) / b.v;
    return r;
}
inline Dual operator+(const Dual& a, double b) { return a + Dual(b); }
inline Dual operator+(double a, const Dual& b) { return Dual(a) + b; }
inline Dual operator-(const Dual& a, double b) { return a - Dual(b); }
inline Dual operator-(double a, const Dual& b) { return Dual(a) - b; }
inline Dual operator*(const Dual& a, double b) { return a * Dual(b); }
inline Dual operator*(double a, const Dual& b) { return Dual(a) * b; }
inline Dual operator/(const Dual& a, double b) { return a / Dual(b); }
inline Dual operator/(double a, const Dual& b) { return Dual(a) / b; }
inline Dual dexp(const Dual& a) { Dual r(std::exp(a.v)); for (int p = 0; p < MAXP; ++p) r.d[p] = r.v * a.d[p]; return r; }
inline Dual dlog(const Dual& a) { Dual r(std::log(a.v)); for (int p = 0; p < MAXP; ++p) r.d[p] = a.d[p] / a.v; return r; }
inline Dual dsin(const Dual& a) { Dual r(std::sin(a.v)); for (int p = 0; p < MAXP; ++p) r.d[p] = std::cos(a.v) * a.d[p]; return r; }

using cplx = std::complex<double>;

// real part ("primal") of each scalar type — every branch of the algorithm is decided on it
inline double re(double x) { return x; }
inline double re(const Dual& x) { return x.v; }
inline double re(const cplx& x) { return x.real(); }

inline double sexp(double x) { return std::exp(x); }
inline Dual sexp(const Dual& x) { return dexp(x); }
inline cplx sexp(const cplx& x) { return std::exp(x); }
inline double slog(double x) { return std::log(x); }
inline Dual slog(const Dual& x) { return dlog(x); }
inline cplx slog(const cplx& x) { return std::log(x); }

// |x| with the AD convention d|x| = sgn(x) dx, sgn(0) = 0 (R-20); for the
// complex step this is |z| := sgn(Re z) z.
template <class S> inline S sabs(const S& x) {
    if (re(x) > 0) return x;
    if (re(x) < 0) return -x;
    return x * 0.0;
}

// ----------------------------------------------------------------------------------
// Problem description (the oracle's own struct; NOT shared with include/pbe.h).
// ----------------------------------------------------------------------------------
enum { LIM_UPWIND = 0, LIM_VANLEER = 1, LIM_MINMOD = 2, LIM_SUPERBEE = 3, LIM_MC = 4 };
enum { LAW_CONST = 0, LAW_ARRHENIUS = 1, LAW_POLY = 2 };
enum { SOL_EXP = 0, SOL_POLY = 1 };
enum { ST_OK = 0, ST_CFL = 2, ST_NEGATIVE = 3, ST_INFEASIBLE = 4, ST_MAXSTEPS = 5 };

}  // namespace oracle

extern "C" {
typedef struct {
    int32_t N;            // number of bins
    double L_lo, dL;      // bin i has center L_lo + (i + 1/2) dL
    int32_t limiter;      // 0 upwind (phi = 0), 1 van Leer, 2 minmod, 3 superbee, 4 MC
    double courant;       // nu (0.9)
    double dt_fixed;      // > 0: fixed time step; 0: CFL time step
    double dt_max;        // cap on the CFL time step (INFINITY = paper behaviour)
    int64_t max_steps;    // runaway guard
    int64_t n_steps;      // > 0: "steps mode": exactly n_steps steps, no sample landing
    double rho_c, k_v;    // crystal density, shape factor (Table 1)
    int32_t law, n_params;
    int32_t sol_kind, n_sol;
    const double* sol;    // [n_sol]
    int32_t n_knots;      // temperature profile T(t), piecewise linear (R-14)
    const double* knot_t;     // [n_knots] shared by all simulations
    const double* knot_T;     // [n_sims or 1][n_knots]
    int64_t knot_T_stride;    // n_knots (per-simulation profiles) or 0 (shared)
    int32_t M;            // number of sample times
    const double* t_samples;  // [M] strictly increasing, > 0
    int32_t n_tan;            // tangent lanes (0..10)
    const double* tangent_seed;  // [n_tan][n_params + n_sol]; NULL => unit vectors over theta
    // 2D model (NEXT-1): N2 > 0 adds the second length L2 (bins j, centers L2_lo + (j+1/2) dL2);
    // theta = [dimension-1 law | dimension-2 law] (n_params even)
    int32_t N2;
    double L2_lo, dL2;
} oracle_problem;
}

namespace oracle {

// ----------------------------------------------------------------------------------
// Kinetics (row a1).  Evaluated at the start of the step (eq-highRes_growth uses G^n).
// ----------------------------------------------------------------------------------
template <class S> S temperature(const oracle_problem& pb, const S& t) {
    // piecewise-linear through (knot_t[k], knot_T[k]); constant outside the knots (R-14)
    const int K = pb.n_knots;
    if (K == 1) return S(pb.knot_T[0]);
    if (re(t) <= pb.knot_t[0]) return S(pb.knot_T[0]);
    if (re(t) >= pb.knot_t[K - 1]) return S(pb.knot_T[K - 1]);
    int k = 0;
    while (!(re(t) >= pb.knot_t[k] && re(t) < pb.knot_t[k + 1])) ++k;
    const double slope = (pb.knot_T[k + 1] - pb.knot_T[k]) / (pb.knot_t[k + 1] - pb.knot_t[k]);
    return pb.knot_T[k] + slope * (t - pb.knot_t[k]);
}

template <class S> S solubility(const oracle_problem& pb, const S* sol, const S& T) {
    if (pb.sol_kind == SOL_EXP) return sol[0] * sexp(sol[1] * T);   // Eq. A.1: c* = a exp(bT)
    return sol[0] + sol[1] * T + sol[2] * T * T;                     // R-13: polynomial c*
}

// x^y for x > 0 as exp(y ln x) (R-18)
template <class S> S spow(const S& x, const S& y) { return sexp(y * slog(x)); }

template <class S> S growth_rate(const oracle_problem& pb, const S* th, const S& Ssat, const S& T) {
    if (pb.law == LAW_CONST) return th[0];
    if (pb.law == LAW_ARRHENIUS) {
        // Eq. A.2 (L699-705): G = k1 exp(-k2/(T+273.15)) (S-1)^k3, "only applies when S exceeds one"
        if (re(Ssat) > 1.0) return th[0] * sexp(-th[1] / (T + 273.15)) * spow(Ssat - 1.0, th[2]);
        // R-12: mirrored dissolution branch G = -kd exp(-Ed/(T+273.15)) (1-S)^d for S < 1
        if (re(Ssat) < 1.0 && pb.n_params >= 6)
            return -(th[3] * sexp(-th[4] / (T + 273.15)) * spow(1.0 - Ssat, th[5]));
        return S(0.0) * Ssat;
    }
    // eq-poly_growth_rate (L565-571): G = sum_{j=1..k} a_j (S-1)^j, growth only (S <= 1 -> 0)
    if (re(Ssat) > 1.0) {
        S g(0.0), x = Ssat - 1.0, xp = x;
        for (int j = 0; j < pb.n_params; ++j) { g = g + th[j] * xp; xp = xp * x; }
        return g;
    }
    return S(0.0) * Ssat;
}

// ----------------------------------------------------------------------------------
// FVM update (rows a3, a4): eq-highRes_growth written out literally for C >= 0.
// Ghost cells f_{-2} = f_{-1} = f_N = f_{N+1} = 0 (boundary conditions L278-280, R-25).
// ----------------------------------------------------------------------------------
// min / max on the real part; the result (value and derivative) is the chosen argument,
// ties take the second argument.
template <class S> S smin(const S& x, const S& y) { return re(x) < re(y) ? x : y; }
template <class S> S smax(const S& x, const S& y) { return re(x) > re(y) ? x : y; }

// phi(theta) * den with theta = num/den (SI L851, L855).  den == 0 -> 0 (R-4).
// van Leer (SI L855) is the paper's limiter (L299-300).  NEXT-4 adds three classical Sweby-region
// limiters in the same phi(theta) form (R-31; every one is 0 for theta <= 0):
//   minmod    phi = max(0, min(1, theta))
//   superbee  phi = max(0, min(2 theta, 1), min(theta, 2))
//   MC        phi = max(0, min(2 theta, (1 + theta)/2, 2))
template <class S> S phi_times_den(const S& num, const S& den, int limiter) {
    if (limiter == LIM_UPWIND) return S(0.0);   // first-order upwind: phi = 0 (R-5)
    if (re(den) == 0.0) return S(0.0);
    const S theta = num / den;
    if (!(re(theta) > 0.0)) return S(0.0);      // every limiter is 0 for theta <= 0
    if (std::isinf(re(theta)))                   // lim_{theta -> inf} phi
        return (limiter == LIM_MINMOD ? S(1.0) : S(2.0)) * den;
    S phi;
    if (limiter == LIM_VANLEER) phi = (theta + sabs(theta)) / (1.0 + sabs(theta));
    else if (limiter == LIM_MINMOD) phi = smin(S(1.0), theta);
    else if (limiter == LIM_SUPERBEE) phi = smax(smin(2.0 * theta, S(1.0)), smin(theta, S(2.0)));
    else phi = smin(smin(2.0 * theta, (1.0 + theta) * 0.5), S(2.0));   // MC
    return phi * den;
}

// One growth sweep (C >= 0) of eq-highRes_growth:
//   f_i^{n+1} = f_i - C (f_i - f_{i-1})
//             - 1/2 C (1 - C) [ phi_{i+1/2} (f_{i+1} - f_i) - phi_{i-1/2} (f_i - f_{i-1}) ]
//   phi_{i-1/2} = phi(theta_{i-1/2}),  theta_{i-1/2} = (f_{i-1} - f_{i-2}) / (f_i - f_{i-1})
template <class S> void sweep_growth(const std::vector<S>& f, const S& C, int limiter, std::vector<S>& out) {
    const int N = (int)f.size();
    auto F = [&](int i) -> S { return (i < 0 || i >= N) ? S(0.0) : f[i]; };
    for (int i = 0; i < N; ++i) {
        const S fm2 = F(i - 2), fm1 = F(i - 1), f0 = F(i), fp1 = F(i + 1);
        const S lim_plus = phi_times_den(f0 - fm1, fp1 - f0, limiter);    // phi_{i+1/2} (f_{i+1} - f_i)
        const S lim_minus = phi_times_den(fm1 - fm2, f0 - fm1, limiter);  // phi_{i-1/2} (f_i - f_{i-1})
        out[i] = f0 - C * (f0 - fm1) - 0.5 * C * (1.0 - C) * (lim_plus - lim_minus);
    }
}

// Full sweep for either sign of C.  C < 0 (dissolution, R-6): the mirror image of the
// growth formula — reverse the bins, sweep with |C|, reverse back.
template <class S> void sweep(const std::vector<S>& f, const S& C, int limiter, std::vector<S>& out) {
    if (re(C) >= 0.0) { sweep_growth(f, C, limiter, out); return; }
    const int N = (int)f.size();
    std::vector<S> r(N), ro(N);
    for (int i = 0; i < N; ++i) r[i] = f[N - 1 - i];
    sweep_growth(r, -C, limiter, ro);
    for (int i = 0; i < N; ++i) out[i] = ro[N - 1 - i];
}

// ----------------------------------------------------------------------------------
// Moments (row a5): mu_k = sum_i dL L_i^k n_i, Neumaier-compensated per real component.
// ----------------------------------------------------------------------------------
struct Neumaier {
    double s = 0.0, comp = 0.0;
    void add(double x) {
        const double t = s + x;
        if (std::fabs(s) >= std::fabs(x)) comp += (s - t) + x; else comp += (x - t) + s;
        s = t;
    }
    double get() const { return s + comp; }
};
inline void moment_sum(const std::vector<double>& terms, double& out) {
    Neumaier a; for (double x : terms) a.add(x); out = a.get();
}
inline void moment_sum(const std::vector<Dual>& terms, Dual& out) {
    Neumaier a, b[MAXP];
    for (const Dual& x : terms) { a.add(x.v); for (int p = 0; p < MAXP; ++p) b[p].add(x.d[p]); }
    out = Dual(a.get()); for (int p = 0; p < MAXP; ++p) out.d[p] = b[p].get();
}
inline void moment_sum(const std::vector<cplx>& terms, cplx& out) {
    Neumaier a, b; for (const cplx& x : terms) { a.add(x.real()); b.add(x.imag()); }
    out = cplx(a.get(), b.get());
}
template <class S> void moments(const oracle_problem& pb, const std::vector<S>& n, S mu[4]) {
    std::vector<S> terms(n.size());
    for (int k = 0; k < 4; ++k) {
        for (size_t i = 0; i < n.size(); ++i) {
            const double L = pb.L_lo + ((double)i + 0.5) * pb.dL;   // bin center (R-2)
            terms[i] = pb.dL * std::pow(L, (double)k) * n[i];
        }
        moment_sum(terms, mu[k]);
    }
}

// ----------------------------------------------------------------------------------
// One simulation (rows a1-a8).
// ----------------------------------------------------------------------------------
template <class S> struct Result {
    std::vector<std::vector<S>> rec;   // [M][6]
    std::vector<S> n_final;
    int32_t status = ST_OK;
    int64_t steps = 0;
};

template <class S>
Result<S> simulate(const oracle_problem& pb, const S* theta, const S* sol, const double* n0, double c0) {
    const int N = pb.N;
    Result<S> R;
    R.rec.assign(pb.n_steps > 0 ? 1 : pb.M, std::vector<S>(6, S(std::numeric_limits<double>::quiet_NaN())));
    std::vector<S> n(N), nn(N);
    double n_scale = 0.0;
    for (int i = 0; i < N; ++i) { n[i] = S(n0[i]); n_scale = std::max(n_scale, n0[i]); }
    S c(c0), t(0.0);
    S mu[4];
    moments(pb, n, mu);
    S mu3_prev = mu[3];
    int m = 0;  // next sample index
    const double nu = pb.courant;

    while (true) {
        if (pb.n_steps > 0) { if (R.steps >= pb.n_steps) break; }
        else if (m >= pb.M) break;
        if (R.steps >= pb.max_steps) { R.status = ST_MAXSTEPS; break; }

        // 1. kinetics at t^n
        const S T = temperature(pb, t);
        const S cs = solubility(pb, sol, T);
        const S Ssat = c / cs;                       // S = c / c*  (L285)
        const S G = growth_rate(pb, theta, Ssat, T);

        // 2. time step
        S dt, C;
        if (pb.dt_fixed > 0.0) {
            dt = S(pb.dt_fixed);
            C = G * dt / pb.dL;
            if (std::fabs(re(C)) > 1.0) { R.status = ST_CFL; break; }
        } else if (re(G) != 0.0) {
            const S dt_cfl = nu * pb.dL / sabs(G);   // SI L859 with |G| (R-7)
            if (pb.dt_max < re(dt_cfl)) { dt = S(pb.dt_max); C = G * dt / pb.dL; }
            else { dt = dt_cfl; C = S(re(G) > 0 ? nu : -nu); }   // C = nu sgn(G) exactly (R-9)
        } else {
            dt = S(pb.dt_max);                        // may be +inf: jump to the next sample
            C = S(0.0);
        }
        bool landing = false;
        if (pb.n_steps <= 0) {
            const double tn = pb.t_samples[m];
            if (re(t) + re(dt) >= tn - 1e-9 * re(dt)) {          // R-8
                const S dtl = tn - t;
                const S Cl = G * dtl / pb.dL;
                if (std::fabs(re(Cl)) <= 1.0) { dt = dtl; C = Cl; landing = true; }
            }
        } else if (std::isinf(re(dt))) {
            dt = S(0.0);                              // steps mode with G = 0 and no cap: no-op step
        }

        // 3. FVM update (eq-highRes_growth, mirrored for C < 0)
        sweep(n, C, pb.limiter, nn);

        // 4. round-off clip (R-17)
        bool bad = false;
        for (int i = 0; i < N; ++i) {
            if (re(nn[i]) < 0.0) {
                if (re(nn[i]) >= -1e-12 * n_scale) nn[i] = S(0.0);
                else bad = true;
            }
        }
        if (bad) { R.status = ST_NEGATIVE; break; }

        // 5. moments of f^{n+1}
        S mun[4];
        moments(pb, nn, mun);

        // 6. mass balance (eq-discrete_mass_balance, L304-312)
        const S cn = c - pb.rho_c * pb.k_v * (mun[3] - mu3_prev);
        if (re(cn) < 0.0) { R.status = ST_INFEASIBLE; break; }

        // commit
        n.swap(nn);
        c = cn;
        mu3_prev = mun[3];
        for (int k = 0; k < 4; ++k) mu[k] = mun[k];
        t = landing ? S(pb.t_samples[m]) : t + dt;
        R.steps += 1;

        // 7. sampling
        if (landing) {
            R.rec[m] = {t, c, mu[0], mu[1], mu[2], mu[3]};
            ++m;
        }
    }
    if (pb.n_steps > 0 && R.status == ST_OK) R.rec[0] = {t, c, mu[0], mu[1], mu[2], mu[3]};
    R.n_final = n;
    return R;
}

}  // namespace oracle

// =====================================================================================
//  C entry points (ctypes, from oracle/__init__.py)
// =====================================================================================
namespace oracle {

template <class S> void seed_inputs(const oracle_problem& pb, const double* th_s, int lane_mode, int lane,
                                    double h, std::vector<S>& th, std::vector<S>& sol);

// Dual: lane p of theta/sol carries seed[p] (NULL seed => unit vectors e_p over theta).
template <> void seed_inputs<Dual>(const oracle_problem& pb, const double* th_s, int, int, double,
                                   std::vector<Dual>& th, std::vector<Dual>& sol) {
    const int P = pb.n_params, Q = pb.n_sol;
    th.assign(P, Dual()); sol.assign(Q, Dual());
    for (int j = 0; j < P; ++j) th[j] = Dual(th_s[j]);
    for (int j = 0; j < Q; ++j) sol[j] = Dual(pb.sol[j]);
    for (int p = 0; p < pb.n_tan; ++p) {
        for (int j = 0; j < P + Q; ++j) {
            // NULL seed: unit vectors e_p over theta only (include/pbe.h); lanes p >= n_params are 0
            const double s = pb.tangent_seed ? pb.tangent_seed[p * (P + Q) + j] : (j == p && j < P ? 1.0 : 0.0);
            if (j < P) th[j].d[p] = s; else sol[j - P].d[p] = s;
        }
    }
}
template <> void seed_inputs<double>(const oracle_problem& pb, const double* th_s, int, int, double,
                                     std::vector<double>& th, std::vector<double>& sol) {
    th.assign(th_s, th_s + pb.n_params);
    sol.assign(pb.sol, pb.sol + pb.n_sol);
}
// complex step along lane `lane`: x + i h seed
template <> void seed_inputs<cplx>(const oracle_problem& pb, const double* th_s, int, int lane, double h,
                                   std::vector<cplx>& th, std::vector<cplx>& sol) {
    const int P = pb.n_params, Q = pb.n_sol;
    th.assign(P, cplx(0)); sol.assign(Q, cplx(0));
    for (int j = 0; j < P + Q; ++j) {
        const double s = pb.tangent_seed ? pb.tangent_seed[lane * (P + Q) + j] : (j == lane && j < P ? 1.0 : 0.0);
        if (j < P) th[j] = cplx(th_s[j], h * s); else sol[j - P] = cplx(pb.sol[j - P], h * s);
    }
}

struct BatchIO {
    const double* theta; const double* n0; int64_t n0_stride; const double* c0;
    double* samples; double* tsamples; int32_t* status; int64_t* steps; double* n_final; double* ndot_final;
};

inline void run_one(const oracle_problem& pb, const BatchIO& io, int s, int mode) {
    const int N = pb.N, P = pb.n_tan;
    const int Mr = pb.n_steps > 0 ? 1 : pb.M;
    const double* th_s = io.theta + (size_t)s * pb.n_params;
    const double* n0 = io.n0 + (size_t)s * io.n0_stride;
    const double c0 = io.c0[s];
    oracle_problem pbs = pb;                      // this simulation's temperature profile
    pbs.knot_T = pb.knot_T + (size_t)s * pb.knot_T_stride;
    double* smp = io.samples + (size_t)s * Mr * 6;
    if (mode == 0) {
        std::vector<double> th, sol; seed_inputs<double>(pb, th_s, 0, 0, 0, th, sol);
        Result<double> R = simulate<double>(pbs, th.data(), sol.data(), n0, c0);
        for (int m = 0; m < Mr; ++m) for (int k = 0; k < 6; ++k) smp[m * 6 + k] = R.rec[m][k];
        io.status[s] = R.status; io.steps[s] = R.steps;
        if (io.n_final) for (int i = 0; i < N; ++i) io.n_final[(size_t)s * N + i] = R.n_final[i];
    } else if (mode == 1) {
        std::vector<Dual> th, sol; seed_inputs<Dual>(pb, th_s, 0, 0, 0, th, sol);
        Result<Dual> R = simulate<Dual>(pbs, th.data(), sol.data(), n0, c0);
        for (int m = 0; m < Mr; ++m) for (int k = 0; k < 6; ++k) smp[m * 6 + k] = R.rec[m][k].v;
        // unreached samples (R-26: a failed simulation's later records are NaN) have NaN tangents too
        if (io.tsamples)
            for (int m = 0; m < Mr; ++m) for (int p = 0; p < P; ++p) for (int k = 0; k < 5; ++k)
                io.tsamples[(((size_t)s * Mr + m) * P + p) * 5 + k] =
                    std::isnan(R.rec[m][k + 1].v) ? R.rec[m][k + 1].v : R.rec[m][k + 1].d[p];
        io.status[s] = R.status; io.steps[s] = R.steps;
        if (io.n_final) for (int i = 0; i < N; ++i) io.n_final[(size_t)s * N + i] = R.n_final[i].v;
        if (io.ndot_final)
            for (int p = 0; p < P; ++p) for (int i = 0; i < N; ++i)
                io.ndot_final[((size_t)s * P + p) * N + i] = R.n_final[i].d[p];
    } else {
        // complex-step derivative (pin only): one run per lane, d = Im(out) / h
        const double h = 1e-40;
        for (int p = 0; p < P; ++p) {
            std::vector<cplx> th, sol; seed_inputs<cplx>(pb, th_s, 0, p, h, th, sol);
            Result<cplx> R = simulate<cplx>(pbs, th.data(), sol.data(), n0, c0);
            if (p == 0) {
                for (int m = 0; m < Mr; ++m) for (int k = 0; k < 6; ++k) smp[m * 6 + k] = R.rec[m][k].real();
                io.status[s] = R.status; io.steps[s] = R.steps;
                if (io.n_final) for (int i = 0; i < N; ++i) io.n_final[(size_t)s * N + i] = R.n_final[i].real();
            }
            if (io.tsamples)
                for (int m = 0; m < Mr; ++m) for (int k = 0; k < 5; ++k)
                    io.tsamples[(((size_t)s * Mr + m) * P + p) * 5 + k] =
                        std::isnan(R.rec[m][k + 1].real()) ? R.rec[m][k + 1].real() : R.rec[m][k + 1].imag() / h;
            if (io.ndot_final)
                for (int i = 0; i < N; ++i) io.ndot_final[((size_t)s * P + p) * N + i] = R.n_final[i].imag() / h;
        }
    }
}

}  // namespace oracle

extern "C" {

// Run n_sims independent simulations (rows a1-a8).  mode 0: double, 1: Dual tangents,
// 2: complex-step tangents.  n_threads > 1 runs one simulation per std::thread.
int oracle_run_batch(const oracle_problem* pb, int32_t n_sims, const double* theta, const double* n0,
                     int64_t n0_stride, const double* c0, double* samples, double* tsamples, int32_t* status,
                     int64_t* steps, double* n_final, double* ndot_final, int32_t mode, int32_t n_threads) {
    if (!pb || pb->N < 1 || pb->n_tan < 0 || pb->n_tan > oracle::MAXP) return 1;
    oracle::BatchIO io{theta, n0, n0_stride, c0, samples, tsamples, status, steps, n_final, ndot_final};
    if (n_threads <= 1) {
        for (int s = 0; s < n_sims; ++s) oracle::run_one(*pb, io, s, mode);
        return 0;
    }
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    for (int w = 0; w < n_threads; ++w)
        pool.emplace_back([&]() {
            for (int s = next++; s < n_sims; s = next++) oracle::run_one(*pb, io, s, mode);
        });
    for (auto& th : pool) th.join();
    return 0;
}

// Kinetics probe (row a1): out = (T, c*, S, G) at time t and concentration c.
void oracle_kinetics(const oracle_problem* pb, const double* theta, double t, double c, double* out) {
    std::vector<double> sol(pb->sol, pb->sol + pb->n_sol);
    const double T = oracle::temperature<double>(*pb, t);
    const double cs = oracle::solubility<double>(*pb, sol.data(), T);
    const double S = c / cs;
    out[0] = T; out[1] = cs; out[2] = S; out[3] = oracle::growth_rate<double>(*pb, theta, S, T);
}

// Sweep probe (rows a3-a4 without clip): out = one eq-highRes_growth step of f with Courant C.
void oracle_sweep(int32_t N, const double* f, double C, int32_t limiter, double* out) {
    std::vector<double> a(f, f + N), b(N);
    oracle::sweep<double>(a, C, limiter, b);
    std::copy(b.begin(), b.end(), out);
}

// Moment probe (row a5).
void oracle_moments(const oracle_problem* pb, const double* n, double* out) {
    std::vector<double> a(n, n + pb->N);
    double mu[4];
    oracle::moments<double>(*pb, a, mu);
    for (int k = 0; k < 4; ++k) out[k] = mu[k];
}

// SI Table S1 worked example, evaluated with the oracle's Dual type (pins Dual arithmetic):
// y1 = sin(x1) / (x1 + x2), y2 = (x1 + x2) exp(x2), tangent direction (v1, v2).
void oracle_dual_si_example(double x1, double x2, double v1, double v2, double* out) {
    oracle::Dual a(x1), b(x2);
    a.d[0] = v1; b.d[0] = v2;
    const oracle::Dual s = a + b;
    const oracle::Dual y1 = oracle::dsin(a) / s;
    const oracle::Dual y2 = s * oracle::dexp(b);
    out[0] = y1.v; out[1] = y2.v; out[2] = y1.d[0]; out[3] = y2.d[0];
}

}  // extern "C"

// =====================================================================================
//  NEXT-1: the paper's 2D model (eq-PBE_batch_2d, L257-266) with Godunov dimensional
//  splitting (L291: "update the PSSD ... along each spatial dimension separately (i.e.
//  twice)"): every row along L1 with C1 = G1 dt / dL1, then every column along L2 with
//  C2 = G2 dt / dL2, each with eq-highRes_growth.  dt = nu min(dL1/|G1|, dL2/|G2|) (SI L859),
//  mass balance with mu_12 = sum dL1 dL2 L1 L2^2 f (eq-discrete_mass_balance, L304-312).
//  Records (t, c, mu00, mu10, mu01, mu11, mu02, mu12) (SPEC MomentVector).  double only.
// =====================================================================================
namespace oracle {

struct Rec2D { double t, c, mu[6]; };

inline void moments2d(const oracle_problem& pb, const std::vector<double>& f, double mu[6]) {
    // (p, q) = (0,0) (1,0) (0,1) (1,1) (0,2) (1,2)  (SI eq-moment2D, L873)
    static const int PQ[6][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}, {0, 2}, {1, 2}};
    const int N1 = pb.N, N2 = pb.N2;
    for (int k = 0; k < 6; ++k) {
        Neumaier acc;
        for (int j = 0; j < N2; ++j) {
            const double L2 = pb.L2_lo + ((double)j + 0.5) * pb.dL2;
            for (int i = 0; i < N1; ++i) {
                const double L1 = pb.L_lo + ((double)i + 0.5) * pb.dL;
                acc.add(pb.dL * pb.dL2 * std::pow(L1, (double)PQ[k][0]) * std::pow(L2, (double)PQ[k][1]) *
                        f[(size_t)j * N1 + i]);
            }
        }
        mu[k] = acc.get();
    }
}

inline int simulate2d(const oracle_problem& pb, const double* theta, const double* f0, double c0,
                      std::vector<Rec2D>& rec, std::vector<double>& f, int64_t& steps) {
    const int N1 = pb.N, N2 = pb.N2, H = pb.n_params / 2;
    oracle_problem p1 = pb;
    p1.n_params = H;
    std::vector<double> sol(pb.sol, pb.sol + pb.n_sol);
    f.assign(f0, f0 + (size_t)N1 * N2);
    double nscale = 0.0;
    for (double v : f) nscale = std::max(nscale, v);
    double c = c0, t = 0.0, mu[6];
    moments2d(pb, f, mu);
    double mu12p = mu[5];
    int m = 0;
    steps = 0;
    rec.assign(pb.n_steps > 0 ? 1 : pb.M, Rec2D{NAN, NAN, {NAN, NAN, NAN, NAN, NAN, NAN}});
    std::vector<double> line, out;
    while (true) {
        if (pb.n_steps > 0) { if (steps >= pb.n_steps) break; }
        else if (m >= pb.M) break;
        if (steps >= pb.max_steps) return ST_MAXSTEPS;
        const double T = temperature<double>(pb, t);
        const double cs = solubility<double>(pb, sol.data(), T);
        const double S = c / cs;
        const double G1 = growth_rate<double>(p1, theta, S, T);
        const double G2 = growth_rate<double>(p1, theta + H, S, T);
        // SI L859: dt = nu min(dL1/|G1|, dL2/|G2|) (a zero rate does not limit), capped (R-7, R-8)
        double dt = pb.dt_max;
        if (pb.dt_fixed > 0.0) dt = pb.dt_fixed;
        else {
            double dtc = INFINITY;
            if (G1 != 0.0) dtc = std::min(dtc, pb.courant * pb.dL / std::fabs(G1));
            if (G2 != 0.0) dtc = std::min(dtc, pb.courant * pb.dL2 / std::fabs(G2));
            dt = std::min(dtc, pb.dt_max);
        }
        bool landing = false;
        if (pb.n_steps <= 0) {
            const double tn = pb.t_samples[m];
            if (t + dt >= tn - 1e-9 * dt) { dt = tn - t; landing = true; }   // land on the sample (R-8)
        } else if (std::isinf(dt)) {
            dt = 0.0;
        }
        const double C1 = G1 * dt / pb.dL, C2 = G2 * dt / pb.dL2;
        if (std::fabs(C1) > 1.0 || std::fabs(C2) > 1.0) return ST_CFL;
        // sweep 1: every row along L1
        std::vector<double> g(f.size());
        line.resize(N1); out.resize(N1);
        for (int j = 0; j < N2; ++j) {
            for (int i = 0; i < N1; ++i) line[i] = f[(size_t)j * N1 + i];
            sweep<double>(line, C1, pb.limiter, out);
            for (int i = 0; i < N1; ++i) g[(size_t)j * N1 + i] = out[i];
        }
        // sweep 2: every column along L2, on the result of sweep 1
        line.resize(N2); out.resize(N2);
        for (int i = 0; i < N1; ++i) {
            for (int j = 0; j < N2; ++j) line[j] = g[(size_t)j * N1 + i];
            sweep<double>(line, C2, pb.limiter, out);
            for (int j = 0; j < N2; ++j) g[(size_t)j * N1 + i] = out[j];
        }
        bool bad = false;
        for (double& v : g)
            if (v < 0.0) { if (v >= -1e-12 * nscale) v = 0.0; else bad = true; }
        if (bad) return ST_NEGATIVE;
        double mun[6];
        moments2d(pb, g, mun);
        const double cn = c - pb.rho_c * pb.k_v * (mun[5] - mu12p);
        if (cn < 0.0) return ST_INFEASIBLE;
        f.swap(g);
        c = cn;
        mu12p = mun[5];
        for (int k = 0; k < 6; ++k) mu[k] = mun[k];
        t = landing ? pb.t_samples[m] : t + dt;
        ++steps;
        if (landing) { rec[m] = Rec2D{t, c, {mu[0], mu[1], mu[2], mu[3], mu[4], mu[5]}}; ++m; }
    }
    if (pb.n_steps > 0) rec[0] = Rec2D{t, c, {mu[0], mu[1], mu[2], mu[3], mu[4], mu[5]}};
    return ST_OK;
}

}  // namespace oracle

extern "C" {
// 2D march of n_sims simulations: samples [S][M][8], f_final [S][N2][N1] (nullable).
int oracle_run_batch_2d(const oracle_problem* pb, int32_t n_sims, const double* theta, const double* f0,
                        int64_t f0_stride, const double* c0, double* samples, int32_t* status, int64_t* steps,
                        double* f_final, int32_t n_threads) {
    if (!pb || pb->N2 < 1 || (pb->n_params % 2) != 0) return 1;
    const int Mr = pb->n_steps > 0 ? 1 : pb->M;
    std::atomic<int> next{0};
    auto work = [&]() {
        for (int s = next++; s < n_sims; s = next++) {
            oracle_problem pbs = *pb;
            pbs.knot_T = pb->knot_T + (size_t)s * pb->knot_T_stride;
            std::vector<oracle::Rec2D> rec;
            std::vector<double> f;
            int64_t st = 0;
            status[s] = oracle::simulate2d(pbs, theta + (size_t)s * pb->n_params, f0 + (size_t)s * f0_stride, c0[s],
                                           rec, f, st);
            steps[s] = st;
            for (int m = 0; m < Mr; ++m) {
                double* o = samples + ((size_t)s * Mr + m) * 8;
                o[0] = rec[m].t; o[1] = rec[m].c;
                for (int k = 0; k < 6; ++k) o[2 + k] = rec[m].mu[k];
            }
            if (f_final) std::copy(f.begin(), f.end(), f_final + (size_t)s * pb->N * pb->N2);
        }
    };
    std::vector<std::thread> pool;
    for (int w = 0; w < std::max(1, (int)n_threads); ++w) pool.emplace_back(work);
    for (auto& th : pool) th.join();
    return 0;
}

// one Godunov-split step of a 2D field (probe): rows along L1 with C1, then columns with C2
void oracle_split_step_2d(int32_t N1, int32_t N2, const double* f, double C1, double C2, int32_t limiter, double* out) {
    std::vector<double> g(f, f + (size_t)N1 * N2), line, o;
    line.resize(N1); o.resize(N1);
    for (int j = 0; j < N2; ++j) {
        for (int i = 0; i < N1; ++i) line[i] = g[(size_t)j * N1 + i];
        oracle::sweep<double>(line, C1, limiter, o);
        for (int i = 0; i < N1; ++i) g[(size_t)j * N1 + i] = o[i];
    }
    line.resize(N2); o.resize(N2);
    for (int i = 0; i < N1; ++i) {
        for (int j = 0; j < N2; ++j) line[j] = g[(size_t)j * N1 + i];
        oracle::sweep<double>(line, C2, limiter, o);
        for (int j = 0; j < N2; ++j) g[(size_t)j * N1 + i] = o[j];
    }
    std::copy(g.begin(), g.end(), out);
}
}  // extern "C"
