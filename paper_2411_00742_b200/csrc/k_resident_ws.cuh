// =====================================================================================
//  k_resident_ws — resident march for simulations WITH tangent lanes (rows a1-a8; the C5
//  ensemble regime: one CTA per simulation, N <= NT K bins), with the per-step scalar chain
//  taken off the critical path.
//
//  Why: in k_resident every warp runs the sweep and then the serial scalar chain (moment sums
//  -> mass balance -> kinetics -> time step) in lockstep, so
//  the FP64 pipe idles for the whole chain (35% of a C5 step, round 1).  But the chain of step
//  n+1 needs only the PRIMAL state after step n, and the tangent sweep of step n needs only the
//  chain of step n.  So one step is split into
//
//    A  primal sweep (all warps): n^{n+1} from C^n in flux form, plus the face weights the
//       tangent lanes need (w_lo, w_hi per face, dg = g_{k+1/2} - g_{k-1/2} per bin, with
//       g = n_up + beta psi), kept in thread-private shared memory; mu3 (+mu0..mu2 on samples)
//    --- barrier ---
//    B  warp 0: the scalar chain of step n+1 (sums, mass balance, records, kinetics + time step
//       in lane-parallel dual numbers seeded with the JACOBIAN directions: lane 0 d/dc, lane 1
//       d/dt, lane 2+p tangent seed p), published as numbers; then its tangent sweep.
//       warps 1..: the tangent sweep of step n (overlapping warp 0's chain):
//           ndot_k <- ndot_k - (Ft_{k+1/2} - Ft_{k-1/2}) - Cdot dg_k,
//           Ft = w_hi ndot_hi + w_mid ndot_mid + w_lo ndot_lo,   w_mid = C - (w_lo + w_hi)
//       (k_resident.cuh's lane flux Fdot = Cdot g + Ft, regrouped so the lane-specific Cdot
//       enters through dg only), then the tangent moments
//    --- barrier ---
//    D  every warp: the linear tangent scalars in lane-parallel form (lane p: tangent p):
//       cdot <- cdot - rho_c k_v (mu3dot' - mu3dot), tdot <- landing ? 0 : tdot + dtdot,
//       Cdot = J_C . (cdot, tdot, e_p), dtdot = J_dt . (cdot, tdot, e_p); tangent halo.
//
//  Records, status, loss and gradient follow k_resident (R-23, R-26); the loss and its
//  gradient are accumulated at the end from the sample records, in sample order.
// =====================================================================================
#pragma once
#include <type_traits>

#include "pbe_device.cuh"

namespace pbe {

constexpr int WS_NJ = 2 + MAXP;          // Jacobian directions: c, t, P seeds
#ifndef WS_LAG
#define WS_LAG 2                         // face-weight loads wait for the update WS_LAG bins back
#endif

struct WsMsg {                 // scalar chain (warp 0) -> every warp, once per step
    double C;                  // Courant number
    double kap2, beta2;        // 2 kappa, 2 beta (kapdot = beta Cdot)
    double JC[WS_NJ];          // dC / d(c, t, seed_p)
    double Jdt[WS_NJ];         // d dt / d(c, t, seed_p)
    int go;                    // 0: the march ended before this step
    int sample;                // the step ends on record m
    int landing;               // t^{n+1} := t_samples[m] (tdot := 0)
    int m;
    int last_ok;               // the previous step completed (no NEG / INFEAS): its record is valid
};

// ---------------------------------------------------------------------------------------
// Step A: one primal sweep of KP bins (flux form, R-3/R-6), publishing the face weights.
// x: this thread's bins, hp: primal halo [4][NTP + 2] of the previous step, u: P thread.
// Face f (local, between bins f-1 and f):  C >= 0: a = d_{f-1}, b = d_f, n_up = n_{f-1};
// C < 0: a = d_{f+1}, b = d_f, n_up = n_f.  Returns the clip mask words through `mask`.
// ---------------------------------------------------------------------------------------
template <int KT, int R, bool NEG, int LIMT>
__device__ __forceinline__ bool ws_primal_sweep(double (&x)[KT * R], const double* __restrict__ hp, int NTP, int u,
                                                double C, double kap2, double beta2, int lim, double* __restrict__ W,
                                                int NTT, int i0, int N, double clip_thr, unsigned (&mask)[R]) {
    constexpr int KP = KT * R;
    const int HS = NTP + 2;
    double* wlo = W;
    double* whi = W + (KT + 1) * NTT;
    double* dgp = W + 2 * (KT + 1) * NTT;
    auto X = [&](int j) -> double {
        if (j >= 0 && j < KP) return x[j];
        if (j == -1) return hp[3 * HS + u];
        if (j == -2) return hp[2 * HS + u];
        if (j == KP) return hp[0 * HS + u + 2];
        return hp[1 * HS + u + 2];                                   // KP + 1
    };
    struct Face { double F, g; };
    auto face = [&](int f) -> Face {
        const int ja = NEG ? f + 1 : f - 1;
        const double a = X(ja) - X(ja - 1), b = X(f) - X(f - 1);
        double h = 0.0, qa = 0.0, qb = 0.0;                          // psi = 2h, d psi/da = 2qa, d psi/db = 2qb
        if (LIMT == 2) psi_half_other(lim, a, b, h, qa, qb);     // minmod / superbee / MC (R-31)
        else if (LIMT == 1) psi_half_d_bf(a, b, h, qa, qb);     // van Leer: no branch per face
        const double nup = X(NEG ? f : f - 1);
        const double pak = kap2 * qa, pbk = kap2 * qb;
        const double w_hi = NEG ? pak : pbk, w_lo = NEG ? -pbk : -pak;
        // T layout: face f of this thread = slot [f % KT][R u + f / KT] (+ [KT][prev] at multiples)
        const int q = f / KT, j = f - q * KT;
        if (q < R) { wlo[j * NTT + R * u + q] = w_lo; whi[j * NTT + R * u + q] = w_hi; }
        if (j == 0 && q > 0) { wlo[KT * NTT + R * u + q - 1] = w_lo; whi[KT * NTT + R * u + q - 1] = w_hi; }
        return Face{fma(C, nup, kap2 * h), fma(beta2, h, nup)};
    };
    bool neg = false;
    auto bin = [&](int k, const Face& L, const Face& Rf) {
        const double nn = x[k] - (Rf.F - L.F);
        neg |= (nn < 0.0);
        x[k] = nn;
        dgp[(k % KT) * NTT + R * u + k / KT] = Rf.g - L.g;
    };
    if (!NEG) {                          // right to left: faces read old values on their left
        Face Rf = face(KP);
#pragma unroll
        for (int k = KP - 1; k >= 0; --k) {
            const Face L = face(k);
            bin(k, L, Rf);
            Rf = L;
        }
    } else {                             // left to right
        Face L = face(0);
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            const Face Rf = face(k + 1);
            bin(k, L, Rf);
            L = Rf;
        }
    }
    // round-off clip (R-17) and padding bins i >= N: zeroed, and their tangents with them (mask)
    bool bad = false;
#pragma unroll
    for (int q = 0; q < R; ++q) mask[q] = 0u;
    if (__any_sync(0xffffffffu, neg || (i0 + KP > N))) {
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            const int i = i0 + k;
            const double nn = x[k];
            const bool zero = (i >= N) || (nn < 0.0 && nn >= -clip_thr);
            bad |= (nn < -clip_thr) && (i < N);
            x[k] = zero ? 0.0 : nn;
            if (zero) mask[k / KT] |= 1u << (k % KT);
        }
    }
    return bad;
}

// ---------------------------------------------------------------------------------------
// Step B: the Cdot-free part of the tangent sweep (in place, same sweep order as the primal).
// th: tangent halo [4][P][NTT + 2]; W: face weights of the step; C: the step's Courant number.
// ---------------------------------------------------------------------------------------
// 0 for any non-NaN v (1 for NaN, whose results are NaN anyway): an index offset the compiler
// cannot fold, so a face's weight loads wait for an earlier bin's update.  Without it ptxas
// evaluates every face flux of the thread at once (all are independent of each other) and the
// 9 x P temporaries spill next to the P x KT resident tangents.
__device__ __forceinline__ int ws_order(double v) { return v != v; }

template <int P, int PG, int KT, bool NEG, int LAG = WS_LAG, int P0 = 0, int P1 = PG>
__device__ __forceinline__ void ws_tangent_sweep(double (&x)[PG][KT], const double* __restrict__ th,
                                                 const double* __restrict__ W, int NTG, int tt, int p0, double C) {
    const int HS = NTG + 2;
    const double* wlo = W;
    const double* whi = W + (KT + 1) * NTG;
    // o: ws_order offset (0) that ties a halo load to an earlier update (see ws_order)
    auto X = [&](int p, int j, int o) -> double {
        if (j >= 0 && j < KT) return x[p][j];
        if (j == -1) return th[(3 * P + p0 + p) * HS + tt + o];
        if (j == -2) return th[(2 * P + p0 + p) * HS + tt + o];
        if (j == KT) return th[(0 * P + p0 + p) * HS + tt + 2 + o];
        return th[(1 * P + p0 + p) * HS + tt + 2 + o];                  // KT + 1
    };
    // lane flux of face f: C >= 0 touches (f-2, f-1, f), C < 0 touches (f-1, f, f+1)
    auto Ft = [&](int f, int p, double wl, double wm, double wh, int o = 0) -> double {
        const int lo = NEG ? f - 1 : f - 2;
        return fma(wh, X(p, lo + 2, o), fma(wm, X(p, lo + 1, o), wl * X(p, lo, o)));
    };
    // Stencil form of the flux update (per lane 1 DMUL + 3 DFMA instead of the flux form's
    // 3 + 2): with F_f = wl_f y_lo + wm_f y_mid + wh_f y_hi, bin k's update y_k - (F_{k+1} - F_k)
    // regroups into four per-bin coefficients shared by all lanes.  The sweep runs in place in
    // the primal's order, so the neighbour already updated is carried as its old value (yo).
#if PBE_WS_FLUXFORM
    double Fc[PG > 0 ? PG : 1];
    if (!NEG) {
        {
            const double wl = wlo[KT * NTG + tt], wh = whi[KT * NTG + tt], wm = C - (wl + wh);
#pragma unroll
            for (int p = P0; p < P1; ++p) Fc[p] = Ft(KT, p, wl, wm, wh);
        }
#pragma unroll
        for (int k = KT - 1; k >= 0; --k) {
            const int o = (LAG > 0 && k + LAG < KT) ? ws_order(x[P0][k + LAG < KT ? k + LAG : 0]) : 0;   // updated LAG bins ago
            const double wl = wlo[k * NTG + tt + o], wh = whi[k * NTG + tt + o], wm = C - (wl + wh);
#pragma unroll
            for (int p = P0; p < P1; ++p) {
                const double fl = Ft(k, p, wl, wm, wh, o);         // reads bins < k and k (old)
                x[p][k] = x[p][k] - (Fc[p] - fl);
                Fc[p] = fl;
            }
        }
    } else {
        {
            const double wl = wlo[tt], wh = whi[tt], wm = C - (wl + wh);
#pragma unroll
            for (int p = P0; p < P1; ++p) Fc[p] = Ft(0, p, wl, wm, wh);
        }
#pragma unroll
        for (int k = 0; k < KT; ++k) {
            const int o = (LAG > 0 && k >= LAG) ? ws_order(x[P0][k >= LAG ? k - LAG : 0]) : 0;
            const double wl = wlo[(k + 1) * NTG + tt + o], wh = whi[(k + 1) * NTG + tt + o], wm = C - (wl + wh);
#pragma unroll
            for (int p = P0; p < P1; ++p) {
                const double fr = Ft(k + 1, p, wl, wm, wh, o);     // reads bins > k and k (old)
                x[p][k] = x[p][k] - (fr - Fc[p]);
                Fc[p] = fr;
            }
        }
    }
#else
    (void)Ft;
    double yo[PG > 0 ? PG : 1];
    if (!NEG) {
        // C >= 0, right to left: F_f touches (f-2, f-1, f);
        // y_k' = (1 - wm_{k+1} + wh_k) y_k + (wm_k - wl_{k+1}) y_{k-1} + wl_k y_{k-2} - wh_{k+1} y_{k+1}
        double wlR = wlo[KT * NTG + tt], whR = whi[KT * NTG + tt];
        double wmR = C - (wlR + whR);
#pragma unroll
        for (int p = P0; p < P1; ++p) yo[p] = X(p, KT, 0);         // old y_{k+1} (halo)
#pragma unroll
        for (int k = KT - 1; k >= 0; --k) {
            const int o = (LAG > 0 && k + LAG < KT) ? ws_order(x[P0][k + LAG < KT ? k + LAG : 0]) : 0;
            const double wl = wlo[k * NTG + tt + o], wh = whi[k * NTG + tt + o], wm = C - (wl + wh);
            const double c0 = (1.0 - wmR) + wh, c1 = wm - wlR;
#pragma unroll
            for (int p = P0; p < P1; ++p) {
                const double y = x[p][k];
                x[p][k] = fma(c0, y, fma(c1, X(p, k - 1, o), fma(wl, X(p, k - 2, o), -whR * yo[p])));
                yo[p] = y;
            }
            wlR = wl; whR = wh; wmR = wm;
        }
    } else {
        // C < 0, left to right: F_f touches (f-1, f, f+1);
        // y_k' = (1 - wl_{k+1} + wm_k) y_k + (wh_k - wm_{k+1}) y_{k+1} - wh_{k+1} y_{k+2} + wl_k y_{k-1}
        double wlL = wlo[tt], whL = whi[tt];
        double wmL = C - (wlL + whL);
#pragma unroll
        for (int p = P0; p < P1; ++p) yo[p] = X(p, -1, 0);         // old y_{k-1} (halo)
#pragma unroll
        for (int k = 0; k < KT; ++k) {
            const int o = (LAG > 0 && k >= LAG) ? ws_order(x[P0][k >= LAG ? k - LAG : 0]) : 0;
            const double wl = wlo[(k + 1) * NTG + tt + o], wh = whi[(k + 1) * NTG + tt + o], wm = C - (wl + wh);
            const double c0 = (1.0 - wl) + wmL, c1 = whL - wm;
#pragma unroll
            for (int p = P0; p < P1; ++p) {
                const double y = x[p][k];
                x[p][k] = fma(c0, y, fma(c1, X(p, k + 1, o), fma(wlL, yo[p], -wh * X(p, k + 2, o))));
                yo[p] = y;
            }
            wlL = wl; whL = wh; wmL = wm;
        }
    }
#endif
}

#if PBE_TIMING
// diagnostics build: cycle sums of CTA 0 — [0..4] warp 1: A, barrier 1, B, barrier 2, D;
// [5] warp 0: scalar chain, [6] warp 0: its B after the chain, [7] steps
__device__ unsigned long long g_ws_cycles[8];
#define WS_T(v) const long long v = clock64()
#define WS_ACC(i, a, b) if (blockIdx.x == 0 && (tid == 0 || tid == 32)) ws_acc[i] += (unsigned long long)((b) - (a))
#else
#define WS_T(v)
#define WS_ACC(i, a, b)
#endif

// Grid: one CTA per simulation.  Block: exactly NT threads: warp 0 = the scalar warp (no
// bins), warps 1..NT/32-1 = bin warps, bin-thread b = tid - 32 owns bins [b K, b K + K) with
// (NT - 32) K >= N.  P = tangent lanes (kp.P <= P in use; the others stay 0).  Dynamic smem:
// ws_smem_doubles(P, K, NT - 32) doubles (face weights, halos, mu3 weights).
// Tuning knobs (A/B via PBE_WS_VARIANT): XS keeps the primal bins in shared memory between the
// A phases (frees their registers during the tangent sweep), HALF sweeps the tangent lanes in
// two halves (half the live face temporaries), LAG is ws_order's lag (0: none).
template <int P, int K, int NT, bool XS = false, bool HALF = false, int LAG = WS_LAG>
__global__ void __launch_bounds__(NT, 1) k_resident_ws(const KParams kp) {
    static_assert(P >= 1 && P <= MAXP && 2 + P <= 32, "1..10 tangent lanes");
    static_assert(NT % 32 == 0 && NT >= 64, "a scalar warp and at least one bin warp");
    constexpr int NB = NT - 32;              // bin threads
    constexpr int NWB = NB / 32;             // bin warps
    constexpr int HS = NB + 2;               // halo row: ghost, NB bin threads, ghost
    constexpr int WSZ = (2 * (K + 1) + K) * NB;
    extern __shared__ double smem[];
    // layout (doubles): W = wlo[K+1][NB] whi[K+1][NB] dg[K][NB] | ph [2][4][HS] | th [4][P][HS] | w3 [K][NB]
    double* W = smem;
    double* phalo = W + WSZ;
    double* thalo = phalo + 8 * HS;
    double* tw3 = thalo + 4 * P * HS;
    double* sx = tw3 + K * NB;                       // XS: primal bins [K][NB] between steps
    __shared__ double s_red[NWB][4];                 // primal moment partials (bin warps)
    __shared__ double s_tred[NWB][4][P];             // tangent moment partials
    __shared__ WsMsg s_step2[2];                     // scalar chain -> every warp, parity (n + 1) & 1
    __shared__ long long s_bad;
    __shared__ double2 s_poly[MAXTH][32];            // POLY fast path: lane l's dual coefficient
    __shared__ double s_th[MAXTH], s_sol[3], s_seed[MAXP * (MAXTH + 3)];

    // lane groups (kp.G CTAs per simulation, e.g. the last partial wave of a batch split in two):
    // CTA b marches simulation kp.sim0 + b / G with tangent lanes [lane0, lane0 + nl) of kp.P;
    // every group recomputes the primal march bitwise identically and group 0 writes its outputs
    const int s = kp.sim0 + (int)blockIdx.x / kp.G;
    const int grp = (int)blockIdx.x % kp.G;
    const int lane0 = grp * P;
    const int nl = max(0, min(P, kp.P - lane0));             // lanes of this CTA in use
    const bool primal_out = grp == 0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool scal = warp == 0;             // the scalar warp
    const int bt = tid - 32, bw = warp - 1;  // bin thread / bin warp (bin warps only)
    const int N = kp.N;
    const double L_half = kp.L_lo + 0.5 * kp.dL;
    const bool steps_mode = kp.n_steps > 0;
    const int i0 = bt * K;
#if PBE_TIMING
    unsigned long long ws_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif

    // ---- set-up --------------------------------------------------------------------------
    for (int j = tid; j < 8; j += NT) { phalo[j * HS] = 0.0; phalo[j * HS + NB + 1] = 0.0; }
    for (int j = tid; j < 4 * P * HS; j += NT) thalo[j] = 0.0;          // ndot^0 = 0 (R-20)
    if (tid == 0) s_bad = -1;
    const int nsd = kp.n_params + kp.n_sol;
    const bool kin_smem = kp.n_params <= MAXTH;
    if (kin_smem) {
        const double* th = kp.theta + (size_t)s * kp.n_params;
        for (int j = tid; j < kp.n_params; j += NT) s_th[j] = th[j];
        for (int j = tid; j < kp.n_sol; j += NT) s_sol[j] = kp.sol[j];
        for (int j = tid; j < nl * nsd; j += NT) s_seed[j] = kp.seed[(size_t)lane0 * nsd + j];
        for (int e = tid; e < MAXTH * 32; e += NT) {     // lane l seeds direction l - 2 (lanes 0/1: c, t)
            const int j = e >> 5, l = e & 31;
            const bool on = j < kp.n_params;
            const bool seeded = on && l >= 2 && l - 2 < nl;
            s_poly[j][l] = make_double2(on ? th[j] : 0.0, seeded ? kp.seed[(size_t)(lane0 + l - 2) * nsd + j] : 0.0);
        }
    }
    double x[K];                             // primal bins (bin warps)
    double y[P][K];                          // tangent lanes
    const double* n0 = kp.n0 + (size_t)s * kp.n0_stride;
    double lmax = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int i = i0 + k;
        x[k] = (!scal && i < N) ? __ldg(n0 + i) : 0.0;
        if (!scal) {
            const double Lc = fma((double)i, kp.dL, L_half);
            tw3[k * NB + bt] = ((kp.dL * Lc) * Lc) * Lc;       // mu3 weights: same formula as every kernel
        }
        lmax = fmax(lmax, x[k]);
#pragma unroll
        for (int p = 0; p < P; ++p) y[p][k] = 0.0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, off));
    if (!scal && lane == 0) s_red[bw][0] = lmax;
    __syncthreads();
    double nsc = 0.0;
    for (int w = 0; w < NWB; ++w) nsc = fmax(nsc, s_red[w][0]);
    const double clip_thr = 1e-12 * nsc;
    __syncthreads();
    auto publish_primal = [&](int q) {
        double* h = phalo + q * 4 * HS;
        h[0 * HS + bt + 1] = x[0];
        h[1 * HS + bt + 1] = x[1];
        h[2 * HS + bt + 1] = x[K - 2];
        h[3 * HS + bt + 1] = x[K - 1];
    };
    // mu3 every step (butterfly), mu0..mu2 on sample steps (transpose-reduce); fixed orders
    auto partials = [&](bool all) {
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) v = fma(tw3[k * NB + bt], x[k], v);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) s_red[bw][3] = v;
        if (all) {
            double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const double Lc = fma((double)(i0 + k), kp.dL, L_half);
                double w = kp.dL;
                acc[0] = fma(w, x[k], acc[0]); w *= Lc;
                acc[1] = fma(w, x[k], acc[1]); w *= Lc;
                acc[2] = fma(w, x[k], acc[2]);
            }
            warp_transpose_reduce<3>(acc, lane);
            const int ri = reduce_index<3>(lane);
            if (ri < 3) s_red[bw][ri] = acc[0];
        }
    };
    auto total = [&](int km) -> double { return sum4u<NWB>(&s_red[0][km], 4, NWB); };
    if (!scal) {
        partials(false);                     // mu3(n0)
        publish_primal(0);
        if (XS) {
#pragma unroll
            for (int k = 0; k < K; ++k) sx[k * NB + bt] = x[k];
        }
    }
    __syncthreads();

    // ---- scalar chain (the scalar warp; identical in its lanes).  Its state lives in shared
    //      memory between steps, so none of it holds registers in the bin warps' sweeps -----
    struct Chain { double c, t, mu3p, dt, tn; long long nstep; int m, status, landing, go, last_ok, sample; };
    __shared__ Chain s_ch;
    if (tid == 0)
        s_ch = Chain{kp.c0[s], 0.0, total(3), 0.0, steps_mode ? 0.0 : kp.t_samples[0], 0, 0,
                     kp.max_steps <= 0 ? ST_MAXSTEPS : ST_OK, 0, kp.max_steps > 0, 1, 0};
    __syncwarp();
    double c, t, mu3p, dt, tn;
    long long nstep;
    int m, status, landing;
    bool go, last_ok, sample;
    const double* kT = kp.knot_T + (size_t)s * kp.knotT_stride;
    const int seedl = (lane >= 2 && lane - 2 < nl) ? lane - 2 : -1;   // lanes >= nl carry 0
    const KinLoaderS KLS{s_th, s_sol, s_seed, seedl, kp.n_params, nsd};
    const KinLoader KL{kp.theta + (size_t)s * kp.n_params, kp.sol, kp.seed, seedl >= 0 ? lane0 + seedl : -1,
                       kp.n_params, nsd};
    const KinCache KC = kin_smem ? kin_cache(kp, KLS, kT) : kin_cache(kp, KL, kT);
    const bool poly_fast = kin_smem && kp.law == LAW_POLY && KC.const_T;
    // kinetics + time step of the next step, Jacobian-seeded duals (rows a1, a2) -> s_step
    WsMsg* s_step = &s_step2[0];             // the chain's output slot (set per call)
    auto kinetics = [&](const auto& LDR) __attribute__((always_inline)) -> bool {
        const D1 cD = mk(c, lane == 0 ? 1.0 : 0.0), tD = mk(t, lane == 1 ? 1.0 : 0.0);
        D1 T, G;
        if (poly_fast) {
            const D1 S = cD * KC.ics;
            G = mk(0.0);
            if (S.v > 1.0) {
                const D1 xx = S - 1.0;
#pragma unroll
                for (int j = MAXTH - 1; j >= 0; --j) {
                    const double2 a = s_poly[j][lane];
                    G = G * xx + mk(a.x, a.y);
                }
                G = G * xx;
            }
        } else if (kp.law == LAW_POLY && kp.n_params > MAXTH) {
            const D1 S = supersaturation(kp, LDR, kT, KC, tD, cD, T);
            G = poly_long_warp_seeded<P>(kp.theta + (size_t)s * kp.n_params, kp.seed, nsd, lane0, nl, kp.n_params, S,
                                         seedl);
        } else {
            const D1 S = supersaturation(kp, LDR, kT, KC, tD, cD, T);
            G = growth_rate(kp, LDR, S, T);
        }
        const StepScalars sc = time_step(kp, G, tD, steps_mode ? 0.0 : tn, steps_mode);
        if (sc.err != ST_OK) { status = sc.err; return false; }
        dt = sc.dt.v;
        landing = sc.landing;
        const double Cv = sc.C.v;
        if (lane < 2 + P) { s_step->JC[lane] = sc.C.d; s_step->Jdt[lane] = sc.dt.d; }
        if (lane == 0) {
            s_step->C = Cv;
            s_step->kap2 = 2.0 * sc.kap.v;
            s_step->beta2 = Cv > 0.0 ? (1.0 - 2.0 * Cv) : (Cv < 0.0 ? -(1.0 + 2.0 * Cv) : 0.0);  // kapdot = beta Cdot
        }
        return true;
    };
    // finish step n (n >= 0) and prepare step n + 1; n = -1: prepare step 0
    auto chain = [&](long long n) __attribute__((always_inline)) {
        s_step = &s_step2[(int)((n + 1) & 1)];
        {
            const Chain h = s_ch;
            c = h.c; t = h.t; mu3p = h.mu3p; dt = h.dt; tn = h.tn; nstep = h.nstep; m = h.m; status = h.status;
            landing = h.landing; go = h.go; last_ok = h.last_ok; sample = h.sample;
        }
        bool need_kin = go;
        if (n >= 0) {
            const double mu3n = total(3);
            const double cn = __dsub_rn(c, __dmul_rn(kp.rho_kv, __dsub_rn(mu3n, mu3p)));   // eq-discrete_mass_balance
            need_kin = false;
            if (s_bad == n) { status = ST_NEG; go = false; last_ok = false; }
            else if (cn < 0.0) { status = ST_INFEAS; go = false; last_ok = false; }
            else {
                c = cn; mu3p = mu3n;
                t = landing ? kp.t_samples[m] : t + dt;
                ++nstep;
                if (sample && lane == 0 && primal_out) {
                    const int mr = steps_mode ? 0 : m;
                    double* r = kp.rec + ((size_t)s * kp.M + mr) * 6;
                    r[0] = t; r[1] = c; r[2] = total(0); r[3] = total(1); r[4] = total(2); r[5] = mu3n;
                }
                if (landing) { ++m; if (m < kp.M) tn = kp.t_samples[m]; }
                if (steps_mode ? (nstep >= kp.n_steps) : (m >= kp.M)) go = false;
                else if (nstep >= kp.max_steps) { status = ST_MAXSTEPS; go = false; }
                else need_kin = true;
            }
        }
        if (need_kin) go = kin_smem ? kinetics(KLS) : kinetics(KL);
        sample = go && (landing || (steps_mode && nstep + 1 == kp.n_steps));
        if (lane == 0) {
            s_step->go = go; s_step->sample = sample; s_step->landing = landing;
            s_step->m = steps_mode ? 0 : m; s_step->last_ok = last_ok;
        }
        __syncwarp();
        if (lane == 0) s_ch = Chain{c, t, mu3p, dt, tn, nstep, m, status, landing, go, last_ok, sample};
        __syncwarp();
    };
    if (scal) chain(-1);
    __syncthreads();

    // ---- the march ---------------------------------------------------------------------------
    // Per step n (bin warps; the scalar warp joins at the barriers):
    //   A  primal sweep of step n (C^n) + face weights; primal partials; primal halo;
    //      moments and halo of the tangents y^n (the state after step n-1)
    //   --- barrier 1 ---
    //   B  every warp: the tangent scalars of step n (cdot^n from mu3dot^n, tdot^n, Cdot^n = J^n .)
    //      scalar warp: tangent record of step n-1, then the scalar chain of step n + 1
    //      bin warps: tangent sweep of step n, Cdot part, clip mask
    //   --- barrier 2 ---
    // s_step2[n & 1] holds step n's scalars (written by the chain of step n-1).
    const int pl = lane < P ? lane : 0;      // lane p carries tangent p
    double C = s_step2[0].C, kap2 = s_step2[0].kap2, beta2 = s_step2[0].beta2;
    bool g_go = s_step2[0].go, smp = s_step2[0].sample;
    bool smp_prev = false, lnd_prev = false;                         // sample / landing of step n - 1
    int m_prev = 0;
    double cdl = 0.0, tdl = 0.0, mu3d = 0.0, dtdl = 0.0;             // cdot, tdot, mu3dot, dtdot
    const int vl = kp.limiter;
    const bool gen = vl != LIM_VANLEER && vl != LIM_UPWIND;
    long long n = 0;
    // tangent moments of the current y (mu3dot every step, all four after a sample step)
    auto tangent_moments = [&](bool all) __attribute__((always_inline)) {
        double acc[P];
#pragma unroll
        for (int p = 0; p < P; ++p) acc[p] = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double w = tw3[k * NB + bt];
#pragma unroll
            for (int p = 0; p < P; ++p) acc[p] = fma(w, y[p][k], acc[p]);
        }
        warp_transpose_reduce<P>(acc, lane);
        const int ri = reduce_index<P>(lane);
        if (ri < P) s_tred[bw][3][ri] = acc[0];
        if (all) {
#pragma unroll
            for (int km = 0; km < 3; ++km) {
#pragma unroll
                for (int p = 0; p < P; ++p) acc[p] = 0.0;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const double Lc = fma((double)(i0 + k), kp.dL, L_half);
                    double w = kp.dL;
#pragma unroll
                    for (int e = 0; e < 2; ++e) if (e < km) w *= Lc;
#pragma unroll
                    for (int p = 0; p < P; ++p) acc[p] = fma(w, y[p][k], acc[p]);
                }
                warp_transpose_reduce<P>(acc, lane);
                if (ri < P) s_tred[bw][km][ri] = acc[0];
            }
        }
    };
    auto tsum = [&](int km) -> double { return sum4u<NWB>(&s_tred[0][km][pl], 4 * P, NWB); };
    // lane-parallel tangent scalars at the start of step n (after barrier 1): cdot^n, tdot^n
    auto tangent_scalars = [&]() __attribute__((always_inline)) {
        const double m3 = tsum(3);
        cdl = __dsub_rn(cdl, __dmul_rn(kp.rho_kv, __dsub_rn(m3, mu3d)));   // tangent of the mass balance
        mu3d = m3;
        tdl = lnd_prev ? 0.0 : tdl + dtdl;                             // t := t_m exactly on landing
    };
    // tangent record of sample step n - 1 (scalar warp, after tangent_scalars)
    auto tangent_record = [&](const WsMsg& Mp) __attribute__((always_inline)) {
        if (smp_prev && Mp.last_ok && lane < nl) {
            double* rt = kp.trec + (((size_t)s * kp.M + m_prev) * kp.P + lane0 + lane) * 5;
            rt[0] = cdl; rt[1] = tsum(0); rt[2] = tsum(1); rt[3] = tsum(2); rt[4] = mu3d;
        }
    };
    // One step for a fixed sign of C (NEG: C < 0).  Each sign runs in its own loop (below), so
    // the register allocator never merges the two sweep directions inside one loop body.
    auto step = [&](auto negc) -> bool {
        constexpr bool NEG = decltype(negc)::value;
        const int q = (int)(n & 1);
        WS_T(t0);
        unsigned mask[1] = {0u};
        if (!scal) {
            // ---- A: primal sweep of step n and the face weights of its tangent sweep -------
            bool bad;
            const double* hin = phalo + q * 4 * HS;
            if (XS) {
#pragma unroll
                for (int k = 0; k < K; ++k) x[k] = sx[k * NB + bt];
            }
            if (vl == LIM_VANLEER) bad = ws_primal_sweep<K, 1, NEG, 1>(x, hin, NB, bt, C, kap2, beta2, vl, W, NB, i0, N, clip_thr, mask);
            else if (!gen)         bad = ws_primal_sweep<K, 1, NEG, 0>(x, hin, NB, bt, C, kap2, beta2, vl, W, NB, i0, N, clip_thr, mask);
            else                   bad = ws_primal_sweep<K, 1, NEG, 2>(x, hin, NB, bt, C, kap2, beta2, vl, W, NB, i0, N, clip_thr, mask);
            if (bad) s_bad = n;
            partials(smp);
            publish_primal(q ^ 1);
            if (XS) {
#pragma unroll
                for (int k = 0; k < K; ++k) sx[k * NB + bt] = x[k];
            }
            // ---- the tangents y^n: moments (for cdot^n) and halo (for the sweep below) -----
            tangent_moments(smp_prev);
            // only the three sides this step's sweep direction reads (C >= 0: the left
            // neighbour's last two bins and the right neighbour's first; C < 0: mirrored)
#pragma unroll
            for (int p = 0; p < P; ++p) {
                thalo[(0 * P + p) * HS + bt + 1] = y[p][0];
                if (NEG) thalo[(1 * P + p) * HS + bt + 1] = y[p][1];
                if (!NEG) thalo[(2 * P + p) * HS + bt + 1] = y[p][K - 2];
                thalo[(3 * P + p) * HS + bt + 1] = y[p][K - 1];
            }
        }
        WS_T(t1);
        __syncthreads();                                               // barrier 1
        WS_T(t2);
        const WsMsg& Mq = s_step2[q];                                  // step n's scalars
        tangent_scalars();
        if (scal) {
            // ---- B (scalar warp): tangent record of step n - 1, scalar chain of step n + 1 -----
            tangent_record(s_step2[q]);
            chain(n);
        } else {
            // ---- B (bin warps): the tangent sweep of step n -----------------------------------
            const double Cd_l = fma(Mq.JC[0], cdl, fma(Mq.JC[1], tdl, Mq.JC[2 + pl]));   // J^n . (cdot, tdot, e_p)
            if (HALF) {
                ws_tangent_sweep<P, P, K, NEG, LAG, 0, P / 2>(y, thalo, W, NB, bt, 0, C);
                ws_tangent_sweep<P, P, K, NEG, LAG, P / 2, P>(y, thalo, W, NB, bt, 0, C);
            } else {
                ws_tangent_sweep<P, P, K, NEG, LAG>(y, thalo, W, NB, bt, 0, C);
            }
            {   // Cdot part: ndot_k -= Cdot (g_{k+1/2} - g_{k-1/2})
                const double* dg = W + 2 * (K + 1) * NB;
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const double cd = __shfl_sync(0xffffffffu, Cd_l, p);
#pragma unroll
                    for (int k = 0; k < K; ++k) y[p][k] = fma(-cd, dg[k * NB + bt], y[p][k]);
                }
            }
            if (mask[0]) {                                             // clipped / padding bins
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (mask[0] & (1u << k)) {
#pragma unroll
                        for (int p = 0; p < P; ++p) y[p][k] = 0.0;
                    }
            }
        }
        dtdl = fma(Mq.Jdt[0], cdl, fma(Mq.Jdt[1], tdl, Mq.Jdt[2 + pl]));
        smp_prev = smp; lnd_prev = Mq.landing; m_prev = Mq.m;
        WS_T(t3);
        __syncthreads();                                               // barrier 2
        WS_T(t4);
        const WsMsg& Mn = s_step2[q ^ 1];                              // step n + 1's scalars
        g_go = Mn.go;
        ++n;
        WS_T(t5);
        if (tid == 32) { WS_ACC(0, t0, t1); WS_ACC(1, t1, t2); WS_ACC(2, t2, t3); WS_ACC(3, t3, t4); WS_ACC(4, t4, t5); }
        if (tid == 0) { WS_ACC(5, t2, t3); WS_ACC(6, t3, t4); WS_ACC(7, 0, 1); }
        if (!g_go) return false;
        C = Mn.C; kap2 = Mn.kap2; beta2 = Mn.beta2; smp = Mn.sample;
        return true;
    };
    while (g_go) {
        if (C >= 0.0) { while (step(std::false_type{}) && C >= 0.0) {} }
        else          { while (step(std::true_type{}) && C < 0.0) {} }
    }
    // the record of the last sample step (its tangent moments were not taken yet)
    if (smp_prev) {
        if (!scal) tangent_moments(true);
        __syncthreads();
        tangent_scalars();
        if (scal) tangent_record(s_step2[(int)(n & 1)]);
    }

    // ---- epilogue --------------------------------------------------------------------------
#if PBE_TIMING
    if (blockIdx.x == 0 && tid == 32) for (int i = 0; i < 5; ++i) g_ws_cycles[i] = ws_acc[i];
    if (blockIdx.x == 0 && tid == 0) for (int i = 5; i < 8; ++i) g_ws_cycles[i] = ws_acc[i];
#endif
    if (XS && !scal) {
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = sx[k * NB + bt];
    }
    if (!scal && kp.n_final && primal_out) {
#pragma unroll
        for (int k = 0; k < K; ++k) { const int i = i0 + k; if (i < N) kp.n_final[(size_t)s * N + i] = x[k]; }
    }
    if (!scal && kp.ndot_final) {
#pragma unroll
        for (int p = 0; p < P; ++p)
            if (p < nl) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int i = i0 + k;
                    if (i < N) kp.ndot_final[((size_t)s * kp.P + lane0 + p) * N + i] = y[p][k];
                }
            }
    }
    if (tid == 0 && primal_out) { kp.status[s] = s_ch.status; kp.steps[s] = s_ch.nstep; }
    // ---- loss and gradient from the sample records (R-23), in sample order ------------------
    __syncthreads();                       // records are complete and visible
    if (scal) {
        const bool ok = s_ch.status == ST_OK;
        const bool has_target = kp.target != nullptr;
        const double qnan = __longlong_as_double(0x7ff8000000000000ll);
        double loss = 0.0, gacc = 0.0;
        if (has_target && ok) {
            const double* tgt = kp.target + (size_t)s * kp.M * 2;
            double sc2 = 0.0, sl2 = 0.0;
            for (int j = lane; j < kp.M; j += 32) { sc2 += tgt[2 * j] * tgt[2 * j]; sl2 += tgt[2 * j + 1] * tgt[2 * j + 1]; }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                sc2 += __shfl_xor_sync(0xffffffffu, sc2, off);
                sl2 += __shfl_xor_sync(0xffffffffu, sl2, off);
            }
            const double rms_c = sqrt(sc2 / kp.M), rms_L = sqrt(sl2 / kp.M);
            const int Mr = steps_mode ? 1 : kp.M;
            const int pg = lane0 + (lane < nl ? lane : 0);
            for (int mr = 0; mr < Mr; ++mr) {
                const double* r = kp.rec + ((size_t)s * kp.M + mr) * 6;
                const double* rt = kp.trec + (((size_t)s * kp.M + mr) * kp.P + pg) * 5;
                const double Lb = r[3] / r[2];
                const double Lbd = (rt[2] * r[2] - r[3] * rt[1]) / (r[2] * r[2]);
                const double rc = (r[1] - tgt[2 * mr]) / rms_c, rL = (Lb - tgt[2 * mr + 1]) / rms_L;
                loss += rc * rc + rL * rL;
                gacc += 2.0 * (rc / rms_c) * rt[0] + 2.0 * (rL / rms_L) * Lbd;
            }
        }
        if (lane == 0 && kp.loss && primal_out) kp.loss[s] = (has_target && ok) ? loss : qnan;
        if (lane < nl && kp.grad) kp.grad[(size_t)s * kp.P + lane0 + lane] = (has_target && ok) ? gacc : qnan;
    }
}

// dynamic shared memory of k_resident_ws<P, K, NT> (NB = NT - 32 bin threads), in doubles
constexpr size_t ws_smem_doubles(int P, int K, int NB, bool XS = false) {
    return (size_t)(2 * (K + 1) + K) * NB + 8 * (size_t)(NB + 2) + (size_t)4 * P * (NB + 2) + (size_t)K * NB +
           (XS ? (size_t)K * NB : 0);
}

}  // namespace pbe
