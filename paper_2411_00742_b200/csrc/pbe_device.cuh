// =====================================================================================
//  pbe_device.cuh — device-side building blocks shared by the libpbe kernels
//  (k_resident, k_cluster, k_stream).  sm_100a, FP64 on the SIMT pipes (nothing on the
//  path is a dense contraction, so no tensor cores).
//
//  Contents
//    KParams        kernel arguments (device pointers + problem constants)
//    D1             one-lane forward-mode dual number: warp lane p carries tangent p, so
//                   one warp evaluates the scalar kinetics for all P <= 10 directions at
//                   once (primal + tangent in one pass)
//    kinetics       row a1: T(t), c*(T), S = c/c*, G(S, T; theta)   (L285, L693-705, L565-571)
//    time step      row a2: CFL / dt_max / fixed dt / landing on sample times (R-7..R-9)
//    limited slope  row a3: psi(a,b) = 2ab/(a+b) for ab > 0, else 0  (= phi_vL(a/b) b)
//    warp_transpose_reduce   V partial sums over 32 lanes in ~V+5 shuffles
// =====================================================================================
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pbe {

constexpr int MAXP = 10;   // tangent lanes
constexpr int MAXTH = 10;  // kinetic parameters held in registers (POLY may have more: runtime loop)
constexpr int MAX_PARAMS = 4096;   // PBE_MAX_PARAMS (include/pbe.h)

enum { LIM_UPWIND = 0, LIM_VANLEER = 1, LIM_MINMOD = 2, LIM_SUPERBEE = 3, LIM_MC = 4 };
enum { LAW_CONST = 0, LAW_ARRH = 1, LAW_POLY = 2 };
enum { SOL_EXP = 0, SOL_POLY = 1 };
enum { ST_OK = 0, ST_CFL = 2, ST_NEG = 3, ST_INFEAS = 4, ST_MAXSTEPS = 5 };

struct KParams {
    // grid and scheme
    int N;
    double L_lo, dL, inv_dL;
    int limiter;
    double courant, dt_fixed, dt_max;
    long long max_steps, n_steps;
    double rho_kv;          // rho_c * k_v
    // kinetics
    int law, n_params, sol_kind, n_sol, n_knots;
    long long knotT_stride; // 0 (shared profile) or n_knots
    const double* theta;    // [S][n_params]
    const double* sol;      // [n_sol]
    const double* knot_t;   // [n_knots]
    const double* knot_T;   // [S or 1][n_knots]
    const double* seed;     // [P][n_params + n_sol]
    // batch
    int n_sims, M, P;       // P = tangent lanes of a simulation
    int G;                  // lane groups per simulation (CTAs per simulation)
    int sim0;               // first simulation of the launch (k_resident_ws tail launches)
    const double* n0; long long n0_stride;
    const double* c0;       // [S]
    const double* t_samples;// [M]
    const double* target;   // [S][M][2] or nullptr
    // outputs
    double* rec;            // [S][M][6]
    double* trec;           // [S][M][P][5]
    int* status;            // [S]
    long long* steps;       // [S]
    double* loss;           // [S]
    double* grad;           // [S][P]
    double* n_final;        // [S][N] or nullptr
    double* ndot_final;     // [S][P][N] or nullptr
};

// 1/x to ~1 ulp without the IEEE-division slow path (no branches): MUFU.RCP64H seed +
// two Newton steps.  Callers guarantee 1e-300 < |x| < 1e300.
__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// ------------------------------------------------------------------------------------
// D1: value + one tangent (this lane's direction).  Divisions use rcp_nr (<= ~1 ulp off the
// correctly rounded quotient, no slow path); operands are c*, S-like ratios and |G| > 1e-300.
// ------------------------------------------------------------------------------------
// Every operation is an explicitly rounded intrinsic (no FMA contraction left to the compiler),
// so the primal value of an expression never depends on the code around it: kernels that
// evaluate the same kinetics with different tangent seedings (k_resident_ws full and half-lane
// CTAs) take bitwise identical primal decisions.
struct D1 { double v, d; };
__device__ __forceinline__ D1 mk(double v, double d = 0.0) { return D1{v, d}; }
__device__ __forceinline__ D1 operator+(D1 a, D1 b) { return {__dadd_rn(a.v, b.v), __dadd_rn(a.d, b.d)}; }
__device__ __forceinline__ D1 operator-(D1 a, D1 b) { return {__dsub_rn(a.v, b.v), __dsub_rn(a.d, b.d)}; }
__device__ __forceinline__ D1 operator-(D1 a) { return {-a.v, -a.d}; }
__device__ __forceinline__ D1 operator*(D1 a, D1 b) {
    return {__dmul_rn(a.v, b.v), __fma_rn(a.d, b.v, __dmul_rn(a.v, b.d))};
}
__device__ __forceinline__ D1 operator/(D1 a, D1 b) {
    const double r = rcp_nr(b.v), q = __dmul_rn(a.v, r);
    return {q, __dmul_rn(__fma_rn(-q, b.d, a.d), r)};
}
__device__ __forceinline__ D1 operator+(D1 a, double b) { return {__dadd_rn(a.v, b), a.d}; }
__device__ __forceinline__ D1 operator-(D1 a, double b) { return {__dsub_rn(a.v, b), a.d}; }
__device__ __forceinline__ D1 operator+(double a, D1 b) { return {__dadd_rn(a, b.v), b.d}; }
__device__ __forceinline__ D1 operator-(double a, D1 b) { return {__dsub_rn(a, b.v), -b.d}; }
__device__ __forceinline__ D1 operator*(D1 a, double b) { return {__dmul_rn(a.v, b), __dmul_rn(a.d, b)}; }
__device__ __forceinline__ D1 operator*(double a, D1 b) { return {__dmul_rn(a, b.v), __dmul_rn(a, b.d)}; }
__device__ __forceinline__ D1 operator/(double a, D1 b) {
    const double r = rcp_nr(b.v), q = __dmul_rn(a, r);
    return {q, __dmul_rn(__dmul_rn(-q, b.d), r)};
}
__device__ __forceinline__ D1 dexp(D1 a) { const double e = exp(a.v); return {e, __dmul_rn(e, a.d)}; }
__device__ __forceinline__ D1 dlog(D1 a) { return {log(a.v), __ddiv_rn(a.d, a.v)}; }
// |x| with d|x| = sgn(x) dx, sgn(0) = 0 (R-20)
__device__ __forceinline__ D1 dabs(D1 a) { return a.v > 0.0 ? a : (a.v < 0.0 ? -a : D1{0.0, 0.0}); }

// ------------------------------------------------------------------------------------
// Row a1: kinetics.  `th`/`so` hold theta and solubility parameters as D1 (this lane's
// seed), `kT` points at this simulation's temperature knots.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ D1 temperature(const KParams& kp, const double* __restrict__ kT, D1 t) {
    const int K = kp.n_knots;
    if (K == 1 || t.v <= kp.knot_t[0]) return mk(kT[0]);
    if (t.v >= kp.knot_t[K - 1]) return mk(kT[K - 1]);
    int k = 0;
    while (!(t.v >= kp.knot_t[k] && t.v < kp.knot_t[k + 1])) ++k;
    const double slope = (kT[k + 1] - kT[k]) / (kp.knot_t[k + 1] - kp.knot_t[k]);
    return kT[k] + slope * (t - kp.knot_t[k]);
}

// Parameters are read on demand through a loader (this lane's seed) so no D1 array of
// theta has to live in registers next to the resident state.
struct KinLoader {
    const double* th;     // this simulation's theta
    const double* sol;    // solubility parameters
    const double* seed;   // [P][n_params + n_sol]
    int lane_p;           // tangent lane of this thread (-1: none)
    int n_params, nsd;
    __device__ __forceinline__ D1 theta(int j) const {
        return mk(__ldg(th + j), lane_p >= 0 ? __ldg(seed + lane_p * nsd + j) : 0.0);
    }
    __device__ __forceinline__ D1 so(int j) const {
        return mk(__ldg(sol + j), lane_p >= 0 ? __ldg(seed + lane_p * nsd + n_params + j) : 0.0);
    }
};

// The same parameters staged in shared memory by the CTA (k_resident: read every step by every
// warp, so the per-step kinetics sees shared-memory latency instead of L1/L2 latency).
struct KinLoaderS {
    const double* th;     // smem [n_params]
    const double* sol;    // smem [n_sol]
    const double* seed;   // smem [P][nsd] (rows of this CTA's lane group)
    int lane_p, n_params, nsd;
    __device__ __forceinline__ D1 theta(int j) const { return mk(th[j], lane_p >= 0 ? seed[lane_p * nsd + j] : 0.0); }
    __device__ __forceinline__ D1 so(int j) const { return mk(sol[j], lane_p >= 0 ? seed[lane_p * nsd + n_params + j] : 0.0); }
};

template <class LD>
__device__ __forceinline__ D1 solubility(const KParams& kp, const LD& L, D1 T) {
    if (kp.sol_kind == SOL_EXP) return L.so(0) * dexp(L.so(1) * T);          // Eq. A.1
    return L.so(0) + L.so(1) * T + L.so(2) * T * T;                           // R-13
}

__device__ __forceinline__ D1 dpow(D1 x, D1 y) { return dexp(y * dlog(x)); }   // R-18

template <class LD>
__device__ __forceinline__ D1 growth_rate(const KParams& kp, const LD& L, D1 S, D1 T) {
    if (kp.law == LAW_CONST) return L.theta(0);
    if (kp.law == LAW_ARRH) {
        if (S.v > 1.0)                                                                 // Eq. A.2
            return L.theta(0) * dexp(-L.theta(1) / (T + 273.15)) * dpow(S - 1.0, L.theta(2));
        if (S.v < 1.0 && kp.n_params >= 6)                                             // R-12
            return -(L.theta(3) * dexp(-L.theta(4) / (T + 273.15)) * dpow(1.0 - S, L.theta(5)));
        return mk(0.0);
    }
    if (S.v > 1.0) {                                                      // eq-poly_growth_rate
        const D1 x = S - 1.0;
        if (kp.n_params > MAXTH) {        // long polynomials (NEXT-3: up to PBE_MAX_PARAMS terms)
            D1 g = mk(0.0);
            for (int j = kp.n_params - 1; j >= 0; --j) g = g * x + L.theta(j);
            return g * x;
        }
        // sum_{j=1..k} a_j x^j in Horner form (short dependency chain on the step's critical
        // path); parameters are loaded up front (independent of the chain)
        D1 a[MAXTH];
#pragma unroll
        for (int j = 0; j < MAXTH; ++j) a[j] = (j < kp.n_params) ? L.theta(j) : mk(0.0);
        D1 g = mk(0.0);
#pragma unroll
        for (int j = MAXTH - 1; j >= 0; --j)
            if (j < kp.n_params) g = g * x + a[j];
        return g * x;
    }
    return mk(0.0);
}

// x^e for an integer e >= 0 by binary exponentiation (<= 2 log2(e) multiplications instead of
// pow()'s exp/log: the long-polynomial chunk offsets and the adjoint's d G / d a_j = x^(j+1)).
__device__ __forceinline__ double ipow(double x, int e) {
    // binary exponentiation with a select instead of a branch per bit (lanes of a warp take
    // different exponents; a divergent branch per bit cost ~50 cycles per iteration): the same
    // products in the same order as the branchy form, so bitwise the same result
    double r = 1.0, b = x;
    while (e > 0) {
        const double rb = r * b;
        r = (e & 1) ? rb : r;
        e >>= 1;
        b = e ? b * b : b;
    }
    return r;
}

// Long polynomial growth law (n > MAXTH terms; NEXT-3's 1000-coefficient regime) evaluated
// cooperatively by the 32 lanes of a warp, for lanes WITHOUT parameter seeds: lane l sums the
// terms j in [l m, l m + m), m = ceil(n/32), by Horner (value and d/dx), scales by x^(l m + 1),
// and a symmetric xor butterfly gives every lane the same G = sum_j a_j x^(j+1) and dG/dx;
// the lane's tangent is dG/dx * dS (chain rule).  O(n/32) dependent steps instead of O(n).
// Must be called by all 32 lanes (warp-uniform S).
__device__ __forceinline__ D1 poly_long_warp(const double* __restrict__ a, int n, D1 S) {
    if (!(S.v > 1.0)) return mk(0.0);
    const int lane = threadIdx.x & 31;
    const double x = S.v - 1.0;
    const int m = (n + 31) >> 5;
    const int j0 = lane * m;
    double q = 0.0, dq = 0.0;
    for (int i = m - 1; i >= 0; --i) {
        const int j = j0 + i;
        const double aj = j < n ? __ldg(a + j) : 0.0;
        dq = fma(dq, x, q);
        q = fma(q, x, aj);
    }
    const double xl = ipow(x, j0);                    // x^(l m)
    double t = xl * x * q;                             // x^(l m + 1) q(x)
    double dt = xl * fma((double)(j0 + 1), q, x * dq); // (l m + 1) x^(l m) q + x^(l m + 1) q'
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        t += __shfl_xor_sync(0xffffffffu, t, off);
        dt += __shfl_xor_sync(0xffffffffu, dt, off);
    }
    return {t, dt * S.d};
}

// Kinetics inputs that are constant when the temperature profile is constant (one knot):
// T and 1/c*(T) are computed once, so a step needs no exp and no division for S.
struct KinCache {
    bool const_T;
    D1 T, ics;
};
template <class LD>
__device__ __forceinline__ KinCache kin_cache(const KParams& kp, const LD& L, const double* kT) {
    KinCache k;
    k.const_T = (kp.n_knots == 1);
    k.T = mk(kT[0]);
    k.ics = k.const_T ? 1.0 / solubility(kp, L, k.T) : mk(0.0);
    return k;
}
// S = c / c*(T(t)) (L285) and T
template <class LD>
__device__ __forceinline__ D1 supersaturation(const KParams& kp, const LD& L, const double* kT,
                                              const KinCache& kc, D1 t, D1 c, D1& T) {
    if (kc.const_T) { T = kc.T; return c * kc.ics; }
    T = temperature(kp, kT, t);
    return c / solubility(kp, L, T);
}

// Fixed-order sum of n values base[0], base[stride], ... (n <= 32): four interleaved chains
// then a pairwise combine — the same order everywhere (deterministic), shorter latency
// than one sequential chain.
// The same sum, unrolled up to MAXW terms (identical order and result for n <= MAXW).
template <int MAXW>
__device__ __forceinline__ double sum4u(const double* base, int stride, int n) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int w = 0; w < MAXW; w += 4) {
        if (w < n) a0 += base[w * stride];
        if (w + 1 < n) a1 += base[(w + 1) * stride];
        if (w + 2 < n) a2 += base[(w + 2) * stride];
        if (w + 3 < n) a3 += base[(w + 3) * stride];
    }
    return (a0 + a1) + (a2 + a3);
}
__device__ __forceinline__ double sum4(const double* base, int stride, int n) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int w = 0; w < n; w += 4) {
        a0 += base[(size_t)w * stride];
        if (w + 1 < n) a1 += base[(size_t)(w + 1) * stride];
        if (w + 2 < n) a2 += base[(size_t)(w + 2) * stride];
        if (w + 3 < n) a3 += base[(size_t)(w + 3) * stride];
    }
    return (a0 + a1) + (a2 + a3);
}

// Per-step scalars produced by the kinetics warp and consumed by every thread.
struct StepScalars {
    D1 C;        // Courant number G dt / dL (+ this lane's tangent)
    D1 kap;      // 1/2 |C| (1 - |C|)
    D1 dt;       // time step
    bool landing;
    int err;     // ST_CFL if fixed-dt |C| > 1
};

// Row a2: the time step at (t, G) toward sample time tn (R-7, R-8, R-9).
__device__ __forceinline__ StepScalars time_step(const KParams& kp, D1 G, D1 t, double tn, bool steps_mode) {
    StepScalars r;
    r.landing = false; r.err = ST_OK;
    D1 dt, C;
    if (kp.dt_fixed > 0.0) {
        dt = mk(kp.dt_fixed);
        C = G * dt * kp.inv_dL;
        if (fabs(C.v) > 1.0) r.err = ST_CFL;
    } else if (fabs(G.v) > 1e-300) {                 // |G| <= 1e-300 moves nothing: treated as 0
        const D1 dt_cfl = (kp.courant * kp.dL) / dabs(G);
        if (kp.dt_max < dt_cfl.v) { dt = mk(kp.dt_max); C = G * dt * kp.inv_dL; }
        else { dt = dt_cfl; C = mk(G.v > 0.0 ? kp.courant : -kp.courant); }   // C = nu sgn G (R-9)
    } else {
        dt = mk(kp.dt_max);
        C = mk(0.0);
    }
    if (!steps_mode) {
        if (__dadd_rn(t.v, dt.v) >= __dsub_rn(tn, __dmul_rn(1e-9, dt.v))) {
            const D1 dtl = tn - t;
            const D1 Cl = G * dtl * kp.inv_dL;
            if (fabs(Cl.v) <= 1.0) { dt = dtl; C = Cl; r.landing = true; }
        }
    } else if (isinf(dt.v)) {
        dt = mk(0.0);
    }
    const D1 aC = dabs(C);
    r.C = C; r.dt = dt;
    r.kap = 0.5 * aC * (1.0 - aC);
    return r;
}

// ------------------------------------------------------------------------------------
// Row a3: limited slope psi(a, b) = phi_vanLeer(a/b) * b = 2ab/(a+b) (ab > 0), else 0,
// plus the partials pa = d psi/da = 2 (b/(a+b))^2 and pb = 2 (a/(a+b))^2 for tangents.
// ------------------------------------------------------------------------------------
// theta = a/b > 0  <=>  ab > 0.  (If ab underflows, |a|,|b| < 1.5e-154 and psi <= 3e-154 is
// taken as 0; if ab > 0 then |a+b| >= sqrt(ab) > 1.4e-154, safe for rcp_nr.)
__device__ __forceinline__ double psi_vl(double a, double b) {
    const double ab = a * b;
    const double r = ab > 0.0 ? rcp_nr(a + b) : 0.0;
    return 2.0 * ab * r;
}
// Half-slope and partials for the tangent lanes:  h = ab/(a+b) = psi/2,
// qa = (b/(a+b))^2 = (d psi/da)/2,  qb = (a/(a+b))^2 = (d psi/db)/2  (0 for ab <= 0).
__device__ __forceinline__ void psi_half_d(double a, double b, double& h, double& qa, double& qb) {
    const double ab = a * b;
    const double r = ab > 0.0 ? rcp_nr(a + b) : 0.0;   // inactive face: r = 0 zeroes all three
    const double br = b * r, ar = a * r;
    h = ab * r;
    qa = br * br;
    qb = ar * ar;
}

// The same three values without a branch around the reciprocal (the divisor is replaced by 1
// on inactive faces and the result selected afterwards): bitwise identical to psi_half_d, but
// the faces of a sweep stay in one basic block, so their reciprocal chains can overlap.
__device__ __forceinline__ void psi_half_d_bf(double a, double b, double& h, double& qa, double& qb) {
    const double ab = a * b;
    const bool act = ab > 0.0;
    const double r0 = rcp_nr(act ? a + b : 1.0);
    const double r = act ? r0 : 0.0;
    const double br = b * r, ar = a * r;
    h = ab * r;
    qa = br * br;
    qb = ar * ar;
}

// Select-free van Leer half slope (primal paths): h = ab/(a+b) for ab > 0, else exactly 0,
// as (a|b| + |a|b) / (2 (|a| + |b|)).  The two products are rounded separately (no FMA
// contraction), so for ab < 0 they cancel exactly and for ab > 0 the numerator is 2 round(ab);
// +1e-300 keeps 0/0 out (it changes no quotient with |a| + |b| > 1e-284).
__device__ __forceinline__ double psi_half_vl_sf(double a, double b) {
    const double num = __dadd_rn(__dmul_rn(fabs(a), b), __dmul_rn(a, fabs(b)));
    return num * (0.5 * rcp_nr((fabs(a) + fabs(b)) + 1e-300));
}

// NEXT-4 limiters (R-31; the paper fixes van Leer, L299-300) as slope limiters psi(a, b) =
// phi(a/b) b for ab > 0, with A = |a|, B = |b| and the sign of b:
//   minmod   m = A <= B ? A : B
//   superbee m = max(min(2A, B), min(A, 2B))
//   MC       m = min(2A, (A + B)/2, 2B)
// Branch choices follow the oracle's min/max (ties take the second argument of min(x, y) =
// x < y ? x : y on phi's argument order).  Half slope h = psi/2 and partials qa, qb = half
// d psi/da, d psi/db (piecewise constant).
__device__ __forceinline__ void psi_half_other(int lim, double a, double b, double& h, double& qa, double& qb) {
    h = qa = qb = 0.0;
    if (!(a * b > 0.0)) return;
    const double A = fabs(a), B = fabs(b), s = b > 0.0 ? 0.5 : -0.5;
    double m, dA, dB;
    if (lim == LIM_MINMOD) {                          // phi = min(1, theta): theta < 1 ... tie -> theta
        if (B < A) { m = B; dA = 0.0; dB = 1.0; } else { m = A; dA = 1.0; dB = 0.0; }
    } else if (lim == LIM_SUPERBEE) {                 // max(min(2 theta, 1), min(theta, 2))
        double m1, a1, b1, m2, a2, b2;
        if (2.0 * A < B) { m1 = 2.0 * A; a1 = 2.0; b1 = 0.0; } else { m1 = B; a1 = 0.0; b1 = 1.0; }
        if (A < 2.0 * B) { m2 = A; a2 = 1.0; b2 = 0.0; } else { m2 = 2.0 * B; a2 = 0.0; b2 = 2.0; }
        if (m1 > m2) { m = m1; dA = a1; dB = b1; } else { m = m2; dA = a2; dB = b2; }
    } else {                                          // MC: min(min(2 theta, (1+theta)/2), 2)
        const double mid = (A + B) * 0.5;
        if (2.0 * A < mid) { m = 2.0 * A; dA = 2.0; dB = 0.0; } else { m = mid; dA = 0.5; dB = 0.5; }
        if (!(m < 2.0 * B)) { m = 2.0 * B; dA = 0.0; dB = 2.0; }
    }
    h = s * m;
    qa = 0.5 * dA;         // d psi/da = dm/dA (sgn a = sgn b), halved
    qb = 0.5 * dB;
}
// Half limited slope h = psi/2 for limiter `lim` (upwind: 0); van Leer first (hot path).
__device__ __forceinline__ double psi_half(int lim, double a, double b) {
    if (lim == LIM_VANLEER) return 0.5 * psi_vl(a, b);
    if (lim == LIM_UPWIND) return 0.0;
    double h, qa, qb;
    psi_half_other(lim, a, b, h, qa, qb);
    return h;
}
// h and the half partials for the tangent / adjoint lanes, any limiter.
__device__ __forceinline__ void psi_half_dl(int lim, double a, double b, double& h, double& qa, double& qb) {
    if (lim == LIM_VANLEER) { psi_half_d_bf(a, b, h, qa, qb); return; }
    if (lim == LIM_UPWIND) { h = qa = qb = 0.0; return; }
    psi_half_other(lim, a, b, h, qa, qb);
}

// ------------------------------------------------------------------------------------
// Transpose-reduce V per-lane values across a warp in ~V + 5 FP64 shuffles (instead of
// 5 V): each level halves the list a lane keeps.  On exit, lane l holds in v[0] the warp
// total of value index reduce_index<V>(l) (== V for padding lanes).  Fully compile-time
// (template recursion), so the list stays in registers.
// ------------------------------------------------------------------------------------
template <int V, int N, int LVL>
struct TransposeReduce {
    static __device__ __forceinline__ void run(double (&v)[V], int lane) {
        constexpr int off = 16 >> LVL;
        constexpr int H = (N + 1) / 2;
        const bool hi = (lane & off) != 0;
#pragma unroll
        for (int j = 0; j < H; ++j) {
            const double upper = (H + j < N) ? v[(H + j < N) ? H + j : 0] : 0.0;
            const double send = hi ? v[j] : upper;
            const double keep = hi ? upper : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
        TransposeReduce<V, H, LVL + 1>::run(v, lane);
    }
};
template <int V, int LVL>
struct TransposeReduce<V, 1, LVL> {
    static __device__ __forceinline__ void run(double (&v)[V], int) {
#pragma unroll
        for (int l = LVL; l < 5; ++l) v[0] += __shfl_xor_sync(0xffffffffu, v[0], 16 >> l);
    }
};
template <int V, int N>
struct TransposeReduce<V, N, 5> {   // more than 32 values: not used (V <= 11)
    static __device__ __forceinline__ void run(double (&)[V], int) {}
};
template <int V>
struct TransposeReduce<V, 1, 5> {
    static __device__ __forceinline__ void run(double (&)[V], int) {}
};

template <int V>
__device__ __forceinline__ void warp_transpose_reduce(double (&v)[V], int lane) {
    TransposeReduce<V, V, 0>::run(v, lane);
}

template <int V>
__device__ __forceinline__ int reduce_index(int lane) {
    // position in the original list; V (= padding) when the lane's final slot is a pad
    // entry of a shorter upper half
    int idx = 0, real = V, n = V;
#pragma unroll
    for (int lvl = 0; lvl < 5; ++lvl) {
        if (n <= 1) break;
        const int h = (n + 1) / 2;
        if (lane & (16 >> lvl)) { idx += h; real -= h; }
        else if (real > h) real = h;
        n = h;
    }
    return real >= 1 ? idx : V;
}

}  // namespace pbe
