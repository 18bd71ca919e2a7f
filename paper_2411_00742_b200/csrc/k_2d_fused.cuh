// =====================================================================================
//  k_2d_fused — NEXT-1 (2D model, Godunov splitting) with both sweeps of a
//  split step fused per HBM pass, barrier-free inside the march.
//
//  A warp owns a strip of F2_W = 28 columns i_s .. i_s+27 and F2_H rows j0 .. j0+H-1 of one
//  simulation; lane l holds column i = i_s - 2 + l (lanes 0,1 and 30,31 are the column halo).
//  The warp marches down the rows r = j0-2 .. j0+H+1, one coalesced 256-byte row load each:
//    sweep 1 (along L1, C1): the face flux F_{i-1/2} of a lane needs n_{i-2..i+1} of its row
//           -> two warp shuffles; F_{i+1/2} is the next lane's flux -> one more shuffle;
//           g = n - (F_{i+1/2} - F_{i-1/2}) for lanes 2..29 (exact for the owned columns);
//           rows outside [0, N2) are ghosts: g = 0.
//    sweep 2 (along L2, C2) runs down the lane's own column in registers: with g of rows
//           r-3 .. r it forms the face between rows r-2 and r-1 (either sign of C2) and
//           emits f^{n+1} of row r-2 = g_{r-2} - (F_{(r-2)+1/2} - F_{(r-3)+1/2}).
//  One face per cell and sweep (no redundant faces); the 2 halo rows above/below a strip and
//  the 4 halo lanes are the only recomputation.  Fused with the cross moments (SI
//  eq-moment2D), the round-off clip, and the store.  Eight strips side by side form a tile (one
//  CTA); per-tile partials are summed in tile order by the CTA that completes the last tile of
//  the simulation, so results never depend on the batch or on the tile-to-CTA assignment.
//  Then one grid barrier and the per-simulation scalar phase (kinetics, dt, mass balance).
//  Algorithmic traffic per cell and step: 8 B read + 8 B write (+ halo re-reads, mostly L2).
// =====================================================================================
#pragma once
#include "k_2d.cuh"

namespace pbe {

#ifndef PBE_F2_H
#define PBE_F2_H 32
#endif
#ifndef PBE_F2_RB
#define PBE_F2_RB 4
#endif
#ifndef PBE_F2_MINB
#define PBE_F2_MINB 3
#endif
constexpr int F2_W = 28;                       // owned columns per warp strip
constexpr int F2_H = PBE_F2_H;                 // owned rows per strip
constexpr int F2_WARPS = 8;                    // strips per tile (CTA)
constexpr int F2_NT = 32 * F2_WARPS;
constexpr int F2_TXC = F2_W * F2_WARPS;        // tile width (columns)
constexpr int F2_RB = PBE_F2_RB;               // rows per load batch (ping-pong prefetch)

struct Params2DF {
    KParams kp;
    int N2;
    double L2_lo, dL2, inv_dL2;
    double* A;            // [S][R2][P1] (bin (j, i) at row j + 2, column i + 2)
    double* B;
    long long P1, R2;
    int NTX, NTY;         // tiles along L1 / L2
    double* part;         // [S][NTX NTY][7]
    unsigned* bar;
    const unsigned long long* nscale_bits;
    int* final_buf;       // [S] 0: final state in A, 1: in B (zeroed by the host)
    unsigned* cnt;        // [S] tiles completed this step (zeroed by the host, reset by the last)
    double* tot;          // [S][8] step totals (mu00, mu10, mu01, mu11, mu02, mu12, negative flag)
    unsigned* work;       // [2] tile counters of alternate steps (zeroed by the host)
};

// Limited flux term kap psi(a, b) = k2 ab/(a+b) (0 unless ab > 0), k2 = |C|(1-|C|) = 2 kap
// (psi = 2ab/(a+b) is the van Leer limited slope), in the select-free
// form psi = (a|b| + |a|b) / (|a| + |b|): the numerator is 2 round(ab) when ab > 0 and exactly 0
// otherwise; the denominator is |a+b| when ab > 0 (+1e-300 keeps 0/0 out; it changes no
// quotient with |a+b| > 1e-284).  Upwind passes k2 = 0 (exactly 0 term).
__device__ __forceinline__ double limited(double a, double b, double k2h) {   // k2h = k2 / 2
    // separately rounded products: exact cancellation for ab < 0 (see psi_half_vl_sf)
    const double num = __dadd_rn(__dmul_rn(fabs(a), b), __dmul_rn(a, fabs(b)));
    const double den = (fabs(a) + fabs(b)) + 1e-300;
    return (k2h * num) * rcp_nr(den);
}

// Limited term of a face: van Leer / upwind use the select-free form above (k = k2/2 or 0);
// GEN (minmod, superbee, MC; NEXT-4) goes through psi_half with k = k2 = 2 kap.
template <bool GEN>
__device__ __forceinline__ double lim_term(double a, double b, double k, int lim) {
    if (GEN) return k * psi_half(lim, a, b);
    return limited(a, b, k);
}

// Sliding state of one lane's column for sweep 2.
struct ColState {
    double gm3, gm2, gm1, Fprev;     // g of rows r-3, r-2, r-1; face below row r-3
    double S0, S1, S2;               // sum v, sum v L2, sum v L2^2 over emitted rows
    double L2;                       // L2 centre of the next emitted row
    bool bad;
};

// One input row of a strip: sweep 1 across lanes, then the sweep-2 face between rows r-2 and
// r-1; if EMIT, the finished cell of row r-2 is clipped, stored and added to the moments.
template <bool NEG1, bool NEG2, bool EMIT, bool GEN>
__device__ __forceinline__ void strip_row(double w, ColState& cs, double C1, double k1, double C2, double k2,
                                          double clip, double dL2, bool own, bool ok, bool sample, double* dst,
                                          int lim) {
    const double wm1 = __shfl_up_sync(0xffffffffu, w, 1);
    double F;
    if (!NEG1) {
        const double wm2 = __shfl_up_sync(0xffffffffu, w, 2);
        F = fma(C1, wm1, lim_term<GEN>(wm1 - wm2, w - wm1, k1, lim));
    } else {
        const double wp1 = __shfl_down_sync(0xffffffffu, w, 1);
        F = fma(C1, w, lim_term<GEN>(wp1 - w, w - wm1, k1, lim));
    }
    const double Fp = __shfl_down_sync(0xffffffffu, F, 1);
    const double g = w - (Fp - F);                 // ghost rows: w = 0 in all lanes -> g = 0
    double F2;
    if (!NEG2) F2 = fma(C2, cs.gm2, lim_term<GEN>(cs.gm2 - cs.gm3, cs.gm1 - cs.gm2, k2, lim));
    else       F2 = fma(C2, cs.gm1, lim_term<GEN>(g - cs.gm1, cs.gm1 - cs.gm2, k2, lim));
    if (EMIT) {                                    // ok: row r-2 < N2 (no branch: keeps the warp converged)
        const bool keep = own && ok;
        double v = cs.gm2 - (F2 - cs.Fprev);
        cs.bad |= keep && v < -clip;               // status NEG; the stored state is then moot
        v = keep ? fmax(v, 0.0) : 0.0;             // round-off clip (R-17); dropped cells add nothing
        if (keep) *dst = v;
        const double vl2 = v * cs.L2;
        cs.S2 = fma(vl2, cs.L2, cs.S2);            // mu12 every step
        cs.S0 += v; cs.S1 += vl2;                  // used on sample steps only
        cs.L2 += dL2;
    }
    cs.Fprev = F2;
    cs.gm3 = cs.gm2; cs.gm2 = cs.gm1; cs.gm1 = g;
}

// One warp strip: march rows j0-2 .. j0+H+1 of fin (RB-row load batches, ping-pong prefetch),
// write the owned cells of rows j0 .. j0+H-1 to fout.  Per-lane moment sums in cs (the caller
// applies the column weights and drops the halo lanes).
template <bool NEG1, bool NEG2, bool GEN>
__device__ __forceinline__ void strip_march(const double* __restrict__ fin, double* __restrict__ fout, long long P1,
                                            int N1, int N2, int is, int j0, double C1, double k1, double C2, double k2,
                                            double clip, bool sample, double dL2, double L2_lo, ColState& cs, int lim) {
    constexpr int RB = F2_RB, NB = (F2_H + 4) / F2_RB;
    static_assert((F2_H + 4) % F2_RB == 0 && NB % 2 == 1 && RB >= 4, "batch layout");
    const int lane = threadIdx.x & 31;
    const int i = is - 2 + lane;
    const bool own = lane >= 2 && lane < 2 + F2_W && i < N1;
    const double* src = fin + (size_t)j0 * P1 + (is + lane);       // padded row j0 = real row j0-2
    double* dst = fout + (size_t)(j0 + 2) * P1 + (is + lane);      // padded row of real row j0
    const int nrow = N2 - j0;                                      // emitted rows < nrow
    cs.gm3 = cs.gm2 = cs.gm1 = cs.Fprev = 0.0;
    cs.L2 = fma((double)j0, dL2, L2_lo + 0.5 * dL2);
    double A[RB], B[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) A[q] = src[(size_t)q * P1];
#pragma unroll
    for (int q = 0; q < RB; ++q) B[q] = src[(size_t)(RB + q) * P1];
    // batch 0: rows 0..3 fill the window, rows 4..RB-1 emit rows j0 .. j0+RB-5
#pragma unroll
    for (int q = 0; q < 4; ++q) strip_row<NEG1, NEG2, false, GEN>(A[q], cs, C1, k1, C2, k2, clip, dL2, own, true, sample, dst, lim);
#pragma unroll
    for (int q = 4; q < RB; ++q) {
        strip_row<NEG1, NEG2, true, GEN>(A[q], cs, C1, k1, C2, k2, clip, dL2, own, q - 4 < nrow, sample, dst, lim);
        dst += P1;
    }
#pragma unroll
    for (int q = 0; q < RB; ++q) A[q] = src[(size_t)(2 * RB + q) * P1];
    int e = RB - 4;                                                // emitted rows so far
#pragma unroll 1
    for (int k = 1; k < NB; k += 2) {
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            strip_row<NEG1, NEG2, true, GEN>(B[q], cs, C1, k1, C2, k2, clip, dL2, own, e + q < nrow, sample, dst, lim);
            dst += P1;
        }
        if (k + 2 < NB) {
#pragma unroll
            for (int q = 0; q < RB; ++q) B[q] = src[(size_t)((k + 2) * RB + q) * P1];
        }
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            strip_row<NEG1, NEG2, true, GEN>(A[q], cs, C1, k1, C2, k2, clip, dL2, own, e + RB + q < nrow, sample, dst, lim);
            dst += P1;
        }
        if (k + 3 < NB) {
#pragma unroll
            for (int q = 0; q < RB; ++q) A[q] = src[(size_t)((k + 3) * RB + q) * P1];
        }
        e += 2 * RB;
    }
}

__global__ void __launch_bounds__(F2_NT, PBE_F2_MINB) k_2d_fused(const Params2DF p) {
    const KParams& kp = p.kp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = F2_WARPS;
    const unsigned G = gridDim.x;
    const int S = kp.n_sims, N1 = kp.N, N2 = p.N2;
    const long long P1 = p.P1, PL = p.R2 * P1;
    const bool steps_mode = kp.n_steps > 0;
    const int lim = kp.limiter;
    const int H = kp.n_params / 2;
    const int T2 = p.NTX * p.NTY;

    __shared__ double s_C1[K2D_MAXS], s_k1[K2D_MAXS], s_C2[K2D_MAXS], s_k2[K2D_MAXS];
    __shared__ int s_active[K2D_MAXS], s_sample[K2D_MAXS];
    struct SimState { double c, t, mu12p, dt, clip; long long nstep; int m, status, landing; };
    __shared__ SimState s_ss[K2D_MAXS];
    __shared__ double s_red[NW][7];
    __shared__ int s_last;
    __shared__ unsigned s_u;

    auto kinetics = [&](int s, SimState& W) -> bool {
        const double* th = kp.theta + (size_t)s * kp.n_params;
        const KinLoader K1{th, kp.sol, kp.seed, -1, H, kp.n_params + kp.n_sol};
        const KinLoader K2{th + H, kp.sol, kp.seed, -1, H, kp.n_params + kp.n_sol};
        KParams kh = kp;
        kh.n_params = H;
        const double* kT = kp.knot_T + (size_t)s * kp.knotT_stride;
        const KinCache KC = kin_cache(kh, K1, kT);
        D1 T;
        const D1 Sat = supersaturation(kh, K1, kT, KC, mk(W.t), mk(W.c), T);
        const double G1 = growth_rate(kh, K1, Sat, T).v, G2 = growth_rate(kh, K2, Sat, T).v;
        double dt;
        if (kp.dt_fixed > 0.0) dt = kp.dt_fixed;
        else {
            double dtc = INFINITY;
            if (fabs(G1) > 1e-300) dtc = fmin(dtc, kp.courant * kp.dL * rcp_nr(fabs(G1)));
            if (fabs(G2) > 1e-300) dtc = fmin(dtc, kp.courant * p.dL2 * rcp_nr(fabs(G2)));
            dt = fmin(dtc, kp.dt_max);
        }
        bool landing = false;
        if (!steps_mode) {
            const double tn = kp.t_samples[W.m];
            if (W.t + dt >= tn - 1e-9 * dt) { dt = tn - W.t; landing = true; }
        } else if (isinf(dt)) {
            dt = 0.0;
        }
        const double C1 = G1 * dt * kp.inv_dL, C2 = G2 * dt * p.inv_dL2;
        if (fabs(C1) > 1.0 || fabs(C2) > 1.0) { W.status = ST_CFL; return false; }
        W.dt = dt;
        W.landing = landing;
        if (lane == 0) {
            s_C1[s] = C1; s_k1[s] = fabs(C1) * (1.0 - fabs(C1));     // 2 kap
            s_C2[s] = C2; s_k2[s] = fabs(C2) * (1.0 - fabs(C2));
        }
        return true;
    };

    // ---- initial state: per-tile mu12(f0) partials written by the load kernel --------------------
    unsigned gen = 0;
    for (int s = warp; s < S; s += NW) {
        const double* pt = p.part + (size_t)s * T2 * 7;
        double a5 = 0.0;
        for (int b = lane; b < T2; b += 32) a5 += pt[(size_t)b * 7 + 5];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) a5 += __shfl_xor_sync(0xffffffffu, a5, off);
        SimState W{};
        W.c = kp.c0[s]; W.t = 0.0; W.mu12p = a5; W.dt = 0.0; W.nstep = 0; W.m = 0; W.status = ST_OK;
        W.landing = 0;
        W.clip = 1e-12 * __longlong_as_double((long long)p.nscale_bits[s]);
        bool go = kp.max_steps > 0;
        if (!go) W.status = ST_MAXSTEPS;
        if (go) go = kinetics(s, W);
        if (lane == 0) {
            s_active[s] = go;
            s_sample[s] = go && (W.landing || (steps_mode && kp.n_steps == 1));
            s_ss[s] = W;
        }
    }
    grid_sync(p.bar, G, gen);

    const double wa = kp.dL * p.dL2;
    int src = 0;
    unsigned step = 0;
    while (true) {
        int any = 0;
        for (int s = 0; s < S; ++s) any |= s_active[s];
        if (!any) break;
        const double* fin = src ? p.B : p.A;
        double* fout = src ? p.A : p.B;
        const unsigned total = (unsigned)S * (unsigned)T2;
        // dynamic tile scheduling: counter work[step & 1]; the other one (last used a step ago,
        // before the grid barrier) is reset here for the next step
        unsigned* work = p.work + (step & 1);
        if (blockIdx.x == 0 && tid == 0) p.work[(step + 1) & 1] = 0u;
        ++step;
        while (true) {
            if (tid == 0) s_u = atomicAdd(work, 1u);
            __syncthreads();
            const unsigned u = s_u;
            if (u >= total) break;
            const int s = (int)(u / (unsigned)T2), tl = (int)(u - (unsigned)s * (unsigned)T2);
            if (!s_active[s]) { __syncthreads(); continue; }        // uniform over the CTA
            const int ty = tl / p.NTX, tx = tl - ty * p.NTX;
            const int is = tx * F2_TXC + warp * F2_W, j0 = ty * F2_H;
            double acc[6] = {0, 0, 0, 0, 0, 0};
            bool bad = false;
            {   // strips past N1 march the zero padding (inside P1) and emit nothing
                const double C1 = s_C1[s], k1 = s_k1[s], C2 = s_C2[s], k2 = s_k2[s];
                const double clip = s_ss[s].clip;
                const bool sample = s_sample[s] != 0;
                const double* fi = fin + (size_t)s * PL;
                double* fo = fout + (size_t)s * PL;
                ColState cs;
                cs.S0 = cs.S1 = cs.S2 = 0.0;
                cs.bad = false;
                // van Leer: k2/2 into the select-free form; upwind: no limited term; other
                // limiters (NEXT-4): the generic path with the full k2
                const bool gen = lim != LIM_VANLEER && lim != LIM_UPWIND;
                const double k1v = gen ? k1 : (lim == LIM_VANLEER ? 0.5 * k1 : 0.0);
                const double k2v = gen ? k2 : (lim == LIM_VANLEER ? 0.5 * k2 : 0.0);
                const int sel = (gen ? 4 : 0) + (C1 < 0.0 ? 2 : 0) + (C2 < 0.0 ? 1 : 0);
#define PBE_STRIP(A, B, GG) strip_march<A, B, GG>(fi, fo, P1, N1, N2, is, j0, C1, k1v, C2, k2v, clip, sample, p.dL2, \
                                                  p.L2_lo, cs, lim)
                switch (sel) {
                    case 0: PBE_STRIP(false, false, false); break;
                    case 1: PBE_STRIP(false, true, false); break;
                    case 2: PBE_STRIP(true, false, false); break;
                    case 3: PBE_STRIP(true, true, false); break;
                    case 4: PBE_STRIP(false, false, true); break;
                    case 5: PBE_STRIP(false, true, true); break;
                    case 6: PBE_STRIP(true, false, true); break;
                    default: PBE_STRIP(true, true, true); break;
                }
#undef PBE_STRIP
                bad = cs.bad;
                const bool own = lane >= 2 && lane < 2 + F2_W && is - 2 + lane < N1;
                const double Sm[3] = {own ? cs.S0 : 0.0, own ? cs.S1 : 0.0, own ? cs.S2 : 0.0};
                // column weights: mu_pq = dL1 dL2 sum L1^p L2^q n
                const double L1 = fma((double)(is - 2 + lane), kp.dL, kp.L_lo + 0.5 * kp.dL);
                acc[5] = L1 * (wa * Sm[2]);
                if (sample) {
                    acc[0] = wa * Sm[0]; acc[1] = L1 * acc[0]; acc[2] = wa * Sm[1];
                    acc[3] = L1 * acc[2]; acc[4] = wa * Sm[2];
                }
            }
            // ---- tile partials (fixed order: lanes, then warps) -> part[s][tl] -------------------
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                for (int k = 0; k < 6; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
            const int anybad = __syncthreads_or(bad);
            if (lane == 0)
#pragma unroll
                for (int k = 0; k < 6; ++k) s_red[warp][k] = acc[k];
            __syncthreads();
            if (tid < 7) {
                double t = 0.0;
                if (tid < 6) for (int w2 = 0; w2 < NW; ++w2) t += s_red[w2][tid];
                else t = anybad ? 1.0 : 0.0;
                p.part[((size_t)s * T2 + tl) * 7 + tid] = t;
                __threadfence();
            }
            __syncthreads();
            // the CTA completing the last tile of simulation s sums its tile partials in tile order
            // (the same order whoever does it) -> tot[s]; the scalar phase then reads 7 numbers
            if (tid == 0) s_last = atomicAdd(p.cnt + s, 1u) == (unsigned)(T2 - 1);
            __syncthreads();
            if (s_last) {
                __threadfence();
                double a[7] = {0, 0, 0, 0, 0, 0, 0};
                const double* pt = p.part + (size_t)s * T2 * 7;
                // UB tiles' partials in flight per L2 round trip; per-thread addition order unchanged
                constexpr int UB = 4;
                int b = tid;
                for (; b + F2_NT * (UB - 1) < T2; b += F2_NT * UB) {
                    double x[UB][7];
#pragma unroll
                    for (int u = 0; u < UB; ++u)
#pragma unroll
                        for (int k = 0; k < 7; ++k) x[u][k] = __ldcg(pt + (size_t)(b + F2_NT * u) * 7 + k);
#pragma unroll
                    for (int u = 0; u < UB; ++u)
#pragma unroll
                        for (int k = 0; k < 7; ++k) a[k] += x[u][k];
                }
                for (; b < T2; b += F2_NT)
#pragma unroll
                    for (int k = 0; k < 7; ++k) a[k] += __ldcg(pt + (size_t)b * 7 + k);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                    for (int k = 0; k < 7; ++k) a[k] += __shfl_xor_sync(0xffffffffu, a[k], off);
                if (lane == 0)
#pragma unroll
                    for (int k = 0; k < 7; ++k) s_red[warp][k] = a[k];
                __syncthreads();
                if (tid < 7) {
                    double t = 0.0;
                    for (int w2 = 0; w2 < NW; ++w2) t += s_red[w2][tid];
                    p.tot[(size_t)s * 8 + tid] = t;
                }
                if (tid == 0) p.cnt[s] = 0u;
            }
            __syncthreads();
        }
        grid_sync(p.bar, G, gen);
        // ---- scalar phase (every CTA, all simulations; warp per simulation) ----------------------
        for (int s = warp; s < S; s += NW) {
            if (!s_active[s]) continue;
            SimState W = s_ss[s];
            double mu[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) mu[k] = __ldcg(p.tot + (size_t)s * 8 + k);
            const double badf = __ldcg(p.tot + (size_t)s * 8 + 6);
            const bool sample = s_sample[s] != 0;
            bool go = true;
            const double cn = W.c - kp.rho_kv * (mu[5] - W.mu12p);
            if (badf > 0.0) { W.status = ST_NEG; go = false; }
            else if (cn < 0.0) { W.status = ST_INFEAS; go = false; }
            else {
                W.c = cn; W.mu12p = mu[5];
                W.t = W.landing ? kp.t_samples[W.m] : W.t + W.dt;
                ++W.nstep;
                if (sample && blockIdx.x == 0 && lane == 0) {
                    const int mr = steps_mode ? 0 : W.m;
                    double* r = kp.rec + ((size_t)s * kp.M + mr) * 8;
                    r[0] = W.t; r[1] = W.c;
                    for (int k = 0; k < 6; ++k) r[2 + k] = mu[k];
                }
                if (W.landing) ++W.m;
                if (steps_mode ? (W.nstep >= kp.n_steps) : (W.m >= kp.M)) go = false;
                else if (W.nstep >= kp.max_steps) { W.status = ST_MAXSTEPS; go = false; }
                else go = kinetics(s, W);
            }
            __syncwarp();
            if (lane == 0) {
                s_active[s] = go;
                s_sample[s] = go && (W.landing || (steps_mode && W.nstep + 1 == kp.n_steps));
                s_ss[s] = W;
                if (!go && blockIdx.x == 0) p.final_buf[s] = src ^ 1;    // its last state is in fout
            }
        }
        __syncthreads();
        src ^= 1;
    }
    if (blockIdx.x == 0 && tid < S) {
        kp.status[tid] = s_ss[tid].status;
        kp.steps[tid] = s_ss[tid].nstep;
    }
}

// initial load: f0 -> A interior, per-tile mu12 partials (tile = F2_TXC columns x F2_H rows,
// summed lanes-then-warps like k_2d_fused), max(f0) bits.  Grid (T2, S), F2_NT threads.
__global__ void __launch_bounds__(F2_NT) k_2d_fused_load(const double* __restrict__ f0, long long f0_stride, int N1,
                                                         int N2, double* A, long long P1, long long R2, int NTX,
                                                         double* part, unsigned long long* nscale_bits, double L_lo,
                                                         double dL, double L2_lo, double dL2) {
    const int s = blockIdx.y, tl = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ty = tl / NTX, tx = tl - ty * NTX;
    const int i = tx * F2_TXC + warp * F2_W + lane, j0 = ty * F2_H;
    const long long PL = R2 * P1;
    double acc = 0.0, m = 0.0;
    if (lane < F2_W && i < N1) {
        const double L1 = fma((double)i, dL, L_lo + 0.5 * dL);
        for (int j = j0; j < j0 + F2_H && j < N2; ++j) {
            const double v = f0[(size_t)s * f0_stride + (size_t)j * N1 + i];
            A[(size_t)s * PL + (size_t)(j + 2) * P1 + i + 2] = v;
            m = fmax(m, v);
            const double L2 = fma((double)j, dL2, L2_lo + 0.5 * dL2);
            acc = fma(L1, dL * dL2 * v * L2 * L2, acc);
        }
    }
    __shared__ double s_a[F2_WARPS], s_m[F2_WARPS];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, off);
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    }
    if (lane == 0) { s_a[warp] = acc; s_m[warp] = m; }
    __syncthreads();
    if (tid == 0) {
        double t = 0.0, mm = 0.0;
        for (int w = 0; w < F2_WARPS; ++w) { t += s_a[w]; mm = fmax(mm, s_m[w]); }
        double* pt = part + ((size_t)s * gridDim.x + tl) * 7;
        for (int k = 0; k < 7; ++k) pt[k] = 0.0;
        pt[5] = t;
        atomicMax(nscale_bits + s, (unsigned long long)__double_as_longlong(mm));
    }
}

// final state per simulation (A or B, per final_buf) -> f_final [S][N2][N1]
__global__ void k_2d_fused_store(const double* __restrict__ A, const double* __restrict__ B, const int* __restrict__ which,
                                 int S, int N1, int N2, long long P1, long long R2, double* f_final) {
    const long long PL = R2 * P1;
    const long long n = (long long)S * N2 * N1;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int s = (int)(e / ((long long)N2 * N1));
        const long long r = e - (long long)s * N2 * N1;
        const int j = (int)(r / N1), i = (int)(r - (long long)j * N1);
        const double* b = which[s] ? B : A;
        f_final[e] = b[(size_t)s * PL + (size_t)(j + 2) * P1 + i + 2];
    }
}

}  // namespace pbe
