// =====================================================================================
//  k_stream_tb — NEXT-4: temporal blocking of uncapped CFL steps in the HBM-streaming march
//  (steps mode, dt_max = inf, no fixed dt, primal only; BASELINE config C4).
//
//  In an uncapped CFL step the Courant number is C = nu sgn(G) EXACTLY (R-9), so the sweep
//  depends on the kinetics only through the sign of G.  While that sign is unchanged, KB
//  consecutive steps are the same geometric update and can be fused per HBM pass:
//
//    per tile: one TMA bulk load of tile + GH = 2 KB ghost-width halo cells per side, d <= KB
//      sub-steps in shared memory (the halo's garbage front moves 2 cells per sub-step and
//      never reaches the owned cells), per-sub-step mu3 partials of the owned cells, one
//      16-byte store of the owned cells after the last sub-step
//    grid barrier
//    scalar phase (one warp per simulation, fixed order): replay the d sub-steps: mass
//      balance c^{n+1} = c^n - rho_c k_v (mu3^{n+1} - mu3^n) (L304-312), S, G, the clock
//      t += nu dL/|G| (SI L859); if sgn G changes inside the block the block is valid only up
//      to that sub-step: the simulation keeps its buffer and redoes that prefix (bitwise the
//      same sub-steps), then continues with the new sign.  Each simulation owns its buffer
//      parity and block depth, so no global consensus is needed.
//
//  Algorithmic traffic per bin-update: 16 B / d (one read + one write per d steps).
// =====================================================================================
#pragma once
#include "k_2d.cuh"      // line_update<NEG> (K = 4 cells from an 8-cell window)
#include "k_stream.cuh"

namespace pbe {

#ifndef PBE_TB_MINB
#define PBE_TB_MINB 2      // 2 CTAs/SM (measured best: 3.34e11 vs 2.50e11 at 3, 2.49e11 at 1)
#endif
constexpr int TB_KB = 8;                 // max fused steps per block
constexpr int TB_GH = 2 * TB_KB;         // ghost / halo width (cells)
constexpr int TB_STAGES = 2;
constexpr int TB_NWC = 8;
constexpr int TB_NT = 32 * (TB_NWC + 1);
// tile size of the temporal-blocking kernel (a function of N only: batch-independent sums)
__host__ __device__ inline int stream_tb_tile(int N) { return N >= 2048 * 64 ? 2048 : (N >= 1024 * 64 ? 1024 : 512); }

struct StreamTBParams {
    KParams kp;
    double* buf0;            // [S][pitch], bin i at index i + TB_GH
    double* buf1;
    long long pitch;
    int TB, T_sim;
    long long n_tiles;
    double* part;            // [S][T_sim][NWC][KB][5]  (mu0..mu3, negative flag) per sub-step
    unsigned* bar;
    int* active;
    int* final_buf;          // [S]
    const unsigned long long* nscale_bits;
};

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// One consumer warp's share of a tile (v2: warp-independent sub-steps).  Warp w owns the
// SEG = TB/8 cells [GH + w SEG, GH + (w+1) SEG) of the window and keeps the region
// [w SEG, w SEG + SEG + 2 GH) = 32 KW cells in registers, KW contiguous cells per lane.  A
// sub-step exchanges 2 cells with each neighbour lane by shuffles and updates the lane's KW
// cells (eq-highRes_growth, flux form); the outermost 2 cells of the region go stale per
// sub-step (lanes 0 / 31 see no neighbour), which the 2 KB-cell halo absorbs.  No shared-
// memory round trips, no CTA barriers inside the tile.
struct TBTile {
    const double* win;           // smem stage: window cells [b0 - GH, b0 + TB + GH)
    double* dst;                 // output row at bin b0 (owned cells)
    double* part;                // [KB][5] this warp's partials of the tile
    int b0, nb, N, TB, d;
    bool sample_last;
    double C, clip, dL, L_half;
    int lim;
    unsigned long long* empty;   // stage's empty barrier
    double* w3s;                 // smem [NWC][KW][32]: mu3 weights of the lanes' cells
};

template <int KW, bool NEG, int LK, bool INT>      // INT: the warp's region lies inside [0, N)
__device__ __forceinline__ void tb_tile_warp(const TBTile& T) {
    constexpr int KB = TB_KB, GH = TB_GH, NWC = TB_NWC;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int SEG = T.TB / NWC;
    const int x0 = warp * SEG + lane * KW;                      // window index of the lane's first cell
    const double C = T.C, aC = fabs(C), kap2 = aC * (1.0 - aC), kh = 0.5 * kap2;
    double c[KW];
    double* w3 = T.w3s + (size_t)warp * KW * 32 + lane;         // [k][lane]: conflict-free
    unsigned dom = 0, own = 0;
#pragma unroll
    for (int k = 0; k < KW; ++k) {
        const int x = x0 + k, i = T.b0 - GH + x;
        c[k] = T.win[x];
        const bool in = i >= 0 && i < T.N;
        const bool ow = x >= GH + warp * SEG && x < GH + (warp + 1) * SEG && x - GH < T.nb;
        dom |= (in ? 1u : 0u) << k;
        own |= (ow ? 1u : 0u) << k;
        const double Lc = fma((double)i, T.dL, T.L_half);
        w3[k * 32] = ow ? T.dL * Lc * Lc * Lc : 0.0;            // mu3 weight (0 off the owned cells)
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(T.empty);                        // this warp is done with the stage
    double am[3] = {0.0, 0.0, 0.0};
#pragma unroll 1
    for (int q = 0; q < T.d; ++q) {
        // neighbours' boundary cells
        const double L1 = __shfl_up_sync(0xffffffffu, c[KW - 1], 1), L2 = __shfl_up_sync(0xffffffffu, c[KW - 2], 1);
        const double R1 = __shfl_down_sync(0xffffffffu, c[0], 1), R2 = __shfl_down_sync(0xffffffffu, c[1], 1);
        double w[KW + 4];
        w[0] = L2; w[1] = L1; w[KW + 2] = R1; w[KW + 3] = R2;
#pragma unroll
        for (int k = 0; k < KW; ++k) w[k + 2] = c[k];
        double F[KW + 1];
#pragma unroll
        for (int f = 2; f <= KW + 2; ++f) {                     // face between window cells f-1 | f
            const int u = NEG ? f : f - 1;
            const int ja = NEG ? f + 1 : f - 1;
            const double a = w[ja] - w[ja - 1], b = w[f] - w[f - 1];
            if (LK == 1) {                                      // select-free van Leer, 1/2 folded into kap
                const double num = __dadd_rn(__dmul_rn(fabs(a), b), __dmul_rn(a, fabs(b)));
                F[f - 2] = fma(C, w[u], (kh * num) * rcp_nr((fabs(a) + fabs(b)) + 1e-300));
            } else {
                const double h = LK == 2 ? psi_half(T.lim, a, b) : 0.0;
                F[f - 2] = fma(C, w[u], kap2 * h);
            }
        }
        const bool last = q == T.d - 1;
        bool bad = false;
        double a3 = 0.0;
#pragma unroll
        for (int k = 0; k < KW; ++k) {
            double v = w[k + 2] - (F[k + 1] - F[k]);
            if (!INT) v = ((dom >> k) & 1u) ? v : 0.0;          // ghost cells outside [0, N) stay 0
            const bool o = (own >> k) & 1u;
            bad |= o && v < -T.clip;                            // status NEG: the stored value is moot
            v = fmax(v, 0.0);                                   // round-off clip (R-17)
            c[k] = v;
            a3 = fma(w3[k * 32], v, a3);
        }
        // this sub-step's warp partial (fixed-order xor tree); lane 0 writes [mu3, bad]
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) a3 += __shfl_xor_sync(0xffffffffu, a3, off);
        const bool bq = __any_sync(0xffffffffu, bad);
        if (lane == 0) { T.part[q * 5 + 3] = a3; T.part[q * 5 + 4] = bq ? 1.0 : 0.0; }
        if (last) {
#pragma unroll
            for (int k = 0; k < KW; ++k) {
                if ((own >> k) & 1u) {
                    T.dst[x0 + k - GH] = c[k];                  // owned cells after d sub-steps
                    if (T.sample_last) {
                        const double Lc = fma((double)(T.b0 - GH + x0 + k), T.dL, T.L_half);
                        const double w0 = T.dL * c[k], w1 = w0 * Lc;
                        am[0] += w0; am[1] += w1; am[2] = fma(w1, Lc, am[2]);
                    }
                }
            }
        }
    }
    if (T.sample_last) {
#pragma unroll
        for (int km = 0; km < 3; ++km) {
            double r = am[km];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
            if (lane == 0) T.part[(T.d - 1) * 5 + km] = r;
        }
    }
}

#if PBE_TB_MAXNREG
__global__ void __maxnreg__(PBE_TB_MAXNREG) k_stream_tb(const StreamTBParams sp) {
#else
__global__ void __launch_bounds__(TB_NT, PBE_TB_MINB) k_stream_tb(const StreamTBParams sp) {
#endif
    constexpr int KB = TB_KB, GH = TB_GH, NWC = TB_NWC, K = 4;
    const KParams& kp = sp.kp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = (warp == NWC);
    const int N = kp.N, TB = sp.TB;
    const int WL = TB + 2 * GH;                       // window length (cells)
    const unsigned G = gridDim.x;
    const int vl = kp.limiter;
    const double L_half = kp.L_lo + 0.5 * kp.dL;

    const long long t_lo = (sp.n_tiles * blockIdx.x) / G;
    const long long t_hi = (sp.n_tiles * (blockIdx.x + 1)) / G;
    const int s_lo = (int)(t_lo / sp.T_sim);
    const int ns = (t_hi > t_lo) ? (int)((t_hi - 1) / sp.T_sim) - s_lo + 1 : 0;

    extern __shared__ __align__(128) double smem[];   // [STAGES][WL] stage, [2][WL] work
    double* work0 = smem + (size_t)TB_STAGES * WL;
    double* work1 = work0 + WL;
    __shared__ __align__(8) unsigned long long s_full[TB_STAGES], s_empty[TB_STAGES];

    struct SimS {
        double c, t, mu3p, clip, G;     // G: growth rate at the start of the next block
        long long nstep;
        int status, cur, depth, sign, active, sample;
    };
    __shared__ SimS s_sim[STREAM_MAXS];

    if (tid == 0)
        for (int i = 0; i < TB_STAGES; ++i) { mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], NWC); }
    for (int x = tid; x < 2 * WL; x += TB_NT) work0[x] = 0.0;      // edge cells are read, never used
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    // growth rate at concentration c (primal; T constant or profile at time t)
    auto growth = [&](int s, double c, double t) -> double {
        const KinLoader KL{kp.theta + (size_t)s * kp.n_params, kp.sol, kp.seed, -1, kp.n_params, kp.n_params + kp.n_sol};
        const double* kT = kp.knot_T + (size_t)s * kp.knotT_stride;
        const KinCache KC = kin_cache(kp, KL, kT);
        D1 T;
        const D1 S = supersaturation(kp, KL, kT, KC, mk(t), mk(c), T);
        const double g = growth_rate(kp, KL, S, T).v;
        return fabs(g) > 1e-300 ? g : 0.0;
    };
    auto sgn = [](double g) { return g > 0.0 ? 1 : (g < 0.0 ? -1 : 0); };

    // ---- init: mu3(n0) from the load kernel's per-tile partials (sub-step 0 slot) --------------
    auto sum_sub = [&](int s, int q, int km) -> double {    // fixed order: lanes, then xor tree
        const double* pt = sp.part + (size_t)s * sp.T_sim * NWC * KB * 5;
        const int ne = sp.T_sim * NWC;
        double a = 0.0;
        constexpr int UB = 8;                                // 8 L2 round trips in flight, same order
        int e = lane;
        for (; e + 32 * (UB - 1) < ne; e += 32 * UB) {
            double x[UB];
#pragma unroll
            for (int u = 0; u < UB; ++u) x[u] = pt[((size_t)(e + 32 * u) * KB + q) * 5 + km];
#pragma unroll
            for (int u = 0; u < UB; ++u) a += x[u];
        }
        for (; e < ne; e += 32) a += pt[((size_t)e * KB + q) * 5 + km];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
        return a;
    };
    if (warp < ns) {
        const int s = s_lo + warp;
        SimS W{};
        W.c = kp.c0[s]; W.t = 0.0; W.mu3p = sum_sub(s, 0, 3); W.nstep = 0; W.status = ST_OK; W.cur = 0;
        W.clip = 1e-12 * __longlong_as_double((long long)sp.nscale_bits[s]);
        W.G = growth(s, W.c, W.t);
        W.sign = sgn(W.G);
        W.active = kp.n_steps > 0 && kp.max_steps > 0;
        if (kp.max_steps <= 0) W.status = ST_MAXSTEPS;
        W.depth = (int)min(min((long long)KB, kp.n_steps), max(kp.max_steps, 1LL));   // never past max_steps
        W.sample = W.depth == kp.n_steps;
        if (lane == 0) s_sim[warp] = W;
    }
    __syncthreads();

    unsigned gen = 0;
    long long n = 0;
    unsigned long long qq = 0;
    auto tile_active = [&](long long t) { return s_sim[(int)(t / sp.T_sim) - s_lo].active != 0; };
    auto next_active = [&](long long t) { while (t < t_hi && !tile_active(t)) ++t; return t; };
    while (true) {
        if (producer) {
            if (lane == 0) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
                unsigned long long q = qq;
                for (long long t = next_active(t_lo); t < t_hi; t = next_active(t + 1), ++q) {
                    const int st = (int)(q % TB_STAGES);
                    if (q >= TB_STAGES) mbar_wait(&s_empty[st], (unsigned)(((q / TB_STAGES) - 1) & 1));
                    const int s = (int)(t / sp.T_sim), j = (int)(t - (long long)s * sp.T_sim);
                    const int b0 = j * TB;
                    const double* src = s_sim[s - s_lo].cur ? sp.buf1 : sp.buf0;
                    const unsigned bytes = (unsigned)WL * 8u;               // [b0 - GH, b0 + TB + GH)
                    mbar_expect_tx(&s_full[st], bytes);
                    bulk_g2s(smem + (size_t)st * WL, src + (size_t)s * sp.pitch + b0, bytes, &s_full[st]);
                }
            }
            for (long long t = next_active(t_lo); t < t_hi; t = next_active(t + 1)) ++qq;
        } else {
            for (long long t = next_active(t_lo); t < t_hi; t = next_active(t + 1), ++qq) {
                const int st = (int)(qq % TB_STAGES);
                mbar_wait(&s_full[st], (unsigned)((qq / TB_STAGES) & 1));
                const int s = (int)(t / sp.T_sim), j = (int)(t - (long long)s * sp.T_sim);
                const int b0 = j * TB, nb = min(TB, N - b0);
                const SimS& W = s_sim[s - s_lo];
                const int lk = vl == LIM_VANLEER ? 1 : (vl == LIM_UPWIND ? 0 : 2);
                TBTile tile{smem + (size_t)st * WL, (W.cur ? sp.buf0 : sp.buf1) + (size_t)s * sp.pitch + b0 + GH,
                            sp.part + (((size_t)s * sp.T_sim + j) * NWC + warp) * KB * 5, b0, nb, N, TB, W.depth,
                            W.sample != 0, W.sign * kp.courant, W.clip, kp.dL, L_half, vl, &s_empty[st], work0};
                const bool neg_c = W.sign < 0;
                // this warp's register region [b0 - GH + w SEG, + SEG + 2 GH) inside the domain?
                const int rg0 = b0 - GH + warp * (TB / NWC);
                const bool inside = rg0 >= 0 && rg0 + TB / NWC + 2 * GH <= N;
#define PBE_TBW(KWV)                                                                                        \
    do {                                                                                                    \
        if (lk == 1) {                                                                                      \
            if (inside) { if (!neg_c) tb_tile_warp<KWV, false, 1, true>(tile); else tb_tile_warp<KWV, true, 1, true>(tile); } \
            else        { if (!neg_c) tb_tile_warp<KWV, false, 1, false>(tile); else tb_tile_warp<KWV, true, 1, false>(tile); } \
        } else if (lk == 0) {                                                                               \
            if (!neg_c) tb_tile_warp<KWV, false, 0, false>(tile); else tb_tile_warp<KWV, true, 0, false>(tile); \
        } else {                                                                                            \
            if (!neg_c) tb_tile_warp<KWV, false, 2, false>(tile); else tb_tile_warp<KWV, true, 2, false>(tile); \
        }                                                                                                   \
    } while (0)
#if PBE_TB_ONLY_VL9
                if (!neg_c) tb_tile_warp<9, false, 1, false>(tile); else tb_tile_warp<9, true, 1, false>(tile);   // A/B only
#else
                if (TB == 2048) PBE_TBW(9); else if (TB == 1024) PBE_TBW(5); else PBE_TBW(3);
#endif
#undef PBE_TBW
            }
        }

        // ---- grid barrier + active count ------------------------------------------------------
        if (tid == 0) {
            int mine = 0;
            for (int slot = 0; slot < ns; ++slot)
                if ((long long)(s_lo + slot) * sp.T_sim >= t_lo && s_sim[slot].active) ++mine;
            if (mine) atomicAdd(&sp.active[n % 3], mine);
        }
        grid_sync(sp.bar, G, gen);
        const int still = *((volatile int*)&sp.active[n % 3]);
        if (blockIdx.x == 0 && tid == 0) sp.active[(n + 2) % 3] = 0;
        if (still == 0) break;

        // ---- scalar phase: replay the block's sub-steps (one warp per simulation) --------------
        if (warp < ns && s_sim[warp].active) {
            const int slot = warp, s = s_lo + slot;
            const bool owner = (long long)s * sp.T_sim >= t_lo;
            const SimS W0 = s_sim[slot];
            SimS W = W0;
            const int d = W.depth;
            int valid = d;
            double mu[4] = {0.0, 0.0, 0.0, 0.0};
            bool fail = false;
            for (int q = 0; q < d; ++q) {
                const double mu3n = sum_sub(s, q, 3);
                const double badf = sum_sub(s, q, 4);
                const double cn = W.c - kp.rho_kv * (mu3n - W.mu3p);
                // clock of this sub-step: uncapped CFL dt = nu dL / |G| (0 when G = 0, steps mode)
                const double dt = W.G != 0.0 ? (kp.courant * kp.dL) * rcp_nr(fabs(W.G)) : 0.0;
                if (badf > 0.0) { W.status = ST_NEG; fail = true; valid = q + 1; break; }
                if (cn < 0.0) { W.status = ST_INFEAS; fail = true; valid = q + 1; break; }
                W.c = cn; W.mu3p = mu3n; W.t += dt; ++W.nstep;
                W.G = growth(s, W.c, W.t);
                if (q + 1 < d && sgn(W.G) != W.sign) { valid = q + 1; break; }   // sign change inside
            }
            if (valid < d) {
                // redo the valid prefix from the unchanged buffer (bitwise the same sub-steps).  On a
                // failure (NEG / INFEAS at sub-step valid - 1) the redo ends exactly at the failing step,
                // which fails again there, so n_final holds the failing step's state like every other
                // kernel (R-26) instead of the state after the whole block
                W = W0;
                W.depth = valid;
                W.sample = W0.sample && false;
            } else {
                if (W.sample && owner && !fail) {
                    for (int km = 0; km < 4; ++km) mu[km] = sum_sub(s, d - 1, km);
                    if (lane == 0) {
                        double* r = kp.rec + (size_t)s * kp.M * 6;
                        r[0] = W.t; r[1] = W.c; r[2] = mu[0]; r[3] = mu[1]; r[4] = mu[2]; r[5] = mu[3];
                    }
                }
                W.cur ^= 1;                                  // the block's result is the current state
                if (fail || W.nstep >= kp.n_steps) W.active = 0;
                else if (W.nstep >= kp.max_steps) { W.status = ST_MAXSTEPS; W.active = 0; }
                else {
                    W.sign = sgn(W.G);
                    W.depth = (int)min(min((long long)KB, kp.n_steps - W.nstep), kp.max_steps - W.nstep);
                    W.sample = (W.nstep + W.depth == kp.n_steps);
                }
                if (!W.active && owner && lane == 0) sp.final_buf[s] = W.cur;
            }
            __syncwarp();
            if (lane == 0) s_sim[slot] = W;
        }
        __syncthreads();
        ++n;
    }
    if (warp < ns) {
        const int s = s_lo + warp;
        if ((long long)s * sp.T_sim >= t_lo && lane == 0) {
            const SimS W = s_sim[warp];
            kp.status[s] = W.status;
            kp.steps[s] = W.nstep;
            if (kp.loss) kp.loss[s] = __longlong_as_double(0x7ff8000000000000ll);
            // never marched (inactive from the start): n_final = n0.  A failure in the very first
            // step also has nstep = 0 but its buffer was set to the failing step's state (R-26)
            if (W.nstep == 0 && W.status != ST_NEG && W.status != ST_INFEAS) sp.final_buf[s] = 0;
        }
    }
}

// n0 -> buffer 0 (index i + GH), mu3(n0) partials per tile in sub-step slot 0, max(n0) bits
__global__ void __launch_bounds__(256) k_stream_tb_load(const double* __restrict__ n0, long long n0_stride, int N,
                                                        double* __restrict__ buf, long long pitch, unsigned long long* nscale_bits,
                                                        int TB, int T_sim, double* __restrict__ part, double L_lo, double dL) {
    const int s = blockIdx.y, j = blockIdx.x;
    const int b0 = j * TB, nb = min(TB, N - b0);
    double m = 0.0, a3 = 0.0;
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        const int i = b0 + k;
        const double v = n0[(size_t)s * n0_stride + i];
        buf[(size_t)s * pitch + TB_GH + i] = v;
        m = fmax(m, v);
        const double Lc = fma((double)i, dL, L_lo + 0.5 * dL);
        a3 = fma(dL * Lc * Lc * Lc, v, a3);
    }
    __shared__ double s_a[8], s_m[8];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
        a3 += __shfl_xor_sync(0xffffffffu, a3, off);
    }
    if ((threadIdx.x & 31) == 0) { s_a[threadIdx.x >> 5] = a3; s_m[threadIdx.x >> 5] = m; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0, mm = 0.0;
        for (int w = 0; w < 8; ++w) { t += s_a[w]; mm = fmax(mm, s_m[w]); }
        double* pt = part + ((size_t)s * T_sim + j) * TB_NWC * TB_KB * 5;
        for (int e = 0; e < TB_NWC * TB_KB * 5; ++e) pt[e] = 0.0;
        pt[3] = t;                                   // warp 0, sub-step 0, mu3
        atomicMax(nscale_bits + s, (unsigned long long)__double_as_longlong(mm));
    }
}

__global__ void k_stream_tb_store(const double* __restrict__ buf0, const double* __restrict__ buf1,
                                  const int* __restrict__ final_buf, int N, long long pitch, double* __restrict__ n_final) {
    const int s = blockIdx.y;
    const double* b = final_buf[s] ? buf1 : buf0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
        n_final[(size_t)s * N + i] = b[(size_t)s * pitch + TB_GH + i];
}

}  // namespace pbe
