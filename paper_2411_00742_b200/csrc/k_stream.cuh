// =====================================================================================
//  k_stream — grid-wide persistent HBM-streaming march for large meshes (10^5 - 10^6+ bins,
//  single simulations or batches).  Rows a1-a8.
//
//  State lives in HBM in two ping-pong buffers, padded rows [S][V][pitch] (bin i at row
//  index i + 2; two zero ghost cells on each side never written: the boundary conditions
//  n(0) = n(inf) = 0 of PAPER.md L278-280).  One cooperative launch runs every time step:
//
//    for each of this CTA's tiles (contiguous static range, <= MAXS simulations per CTA)
//        TMA bulk copy (cp.async.bulk, mbarrier completion) of the tile + 2-bin halos of
//        every variable into a double-buffered smem stage (the next tile streams in while
//        this one is computed)
//        K = 4 bins per thread: limited fluxes of 5 faces, update, round-off clip,
//        moment partials; coalesced 16-byte stores to the other buffer
//        block reduction of the tile partials -> global part[s][tile][5][V]
//    grid barrier (atomic arrive + acquire spin)
//    scalar phase: one warp per simulation of this CTA sums the tile partials of its
//        simulation in a fixed order (deterministic, bitwise identical in every CTA that
//        touches the simulation), mass balance, clock, records, kinetics of the next step
//        in lane-parallel dual numbers
//
//  Algorithmic traffic: 8 B read + 8 B write per bin-update and variable (16 (1 + P) B).
// =====================================================================================
#pragma once
#include <cooperative_groups.h>
#include <type_traits>

#include "pbe_device.cuh"

namespace pbe {

#if PBE_TIMING
// per CTA: own tile work (loop top -> CTA arrives at the grid barrier), grid-barrier wait,
// scalar phase, steps, warp-tiles that took the round-off clip path (diagnostics builds only;
// tools/stream_cycles.py)
__device__ unsigned long long g_stream_cycles[1024][5];
#endif

constexpr int STREAM_MAXS = 8;      // simulations one CTA may touch
constexpr int STREAM_NWC = 8;       // compute warps per CTA
constexpr int STREAM_NT = 32 * (STREAM_NWC + 1);   // + 1 producer (TMA) warp
#ifndef PBE_STREAM_MINB1
#define PBE_STREAM_MINB1 2                              // primal: CTAs per SM
#endif
#ifndef PBE_STREAM_STG1
#define PBE_STREAM_STG1 3                               // primal: smem pipeline depth
#endif
template <int V> struct StreamCfg {
    static constexpr int K = V <= 3 ? 4 : 2;         // consecutive bins per thread per pass
    static constexpr int MINB = V == 1 ? PBE_STREAM_MINB1 : 1;   // CTAs per SM (register budget)
    static constexpr int STAGES = V == 1 ? PBE_STREAM_STG1 : 2;  // smem pipeline depth
};
// Tile size: a function of N and V only, so a simulation's partial-sum order (and hence
// its result, bitwise) never depends on the batch it runs in.
__host__ __device__ inline int stream_tile(int N, int V) {
    int tb = 256;
    const int cap = V == 1 ? 4096 : 1024;
    while (tb < cap && tb * 256 < N) tb <<= 1;
    return tb;
}

struct StreamParams {
    KParams kp;
    double* buf0;           // [S][V][pitch]
    double* buf1;
    long long pitch;        // doubles per (sim, variable) row, >= N + 4, multiple of 4
    int TB;                 // bins per tile (stream_tile(N, V))
    int T_sim;              // tiles per simulation
    long long n_tiles;      // S * T_sim
    double* part;           // [S][T_sim][NWC][5][V] per-warp tile partials (slot 4: negative flag)
    unsigned* bar;          // [2]: arrive count, generation
    int* active;            // [3] rotating counters of simulations still marching
    int* final_buf;         // [S] buffer (0/1) holding each simulation's final state
    const unsigned long long* nscale_bits;  // [S] max(n0_s) as uint64 bits (non-negative)
    // dynamic tile scheduling (k_stream<P, true>): per-step tile counters, per-simulation step
    // coefficients published by the simulation's owner warp, and the step they are valid for
    unsigned* tile_ctr;     // [3] rotating per-step counters
    void* coef;             // [S] SimCoef<P>
    unsigned* coef_step;    // [S] step index of coef[s] (0xffffffff before the first publication)
};

// ---- PTX helpers ----------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// 1D bulk copy global -> shared, completion counted on `bar` (TMA, SASS UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid-wide barrier for a cooperative launch (all CTAs co-resident).
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks, unsigned& gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned target = gen + 1;
        __threadfence();
        const unsigned arrived = atomicAdd(&bar[0], 1u) + 1u;
        if (arrived == nblocks) {
            bar[0] = 0u;
            __threadfence();
            atomicExch(&bar[1], target);
        } else {
            while (ld_acquire(&bar[1]) < target) __nanosleep(32);
        }
        __threadfence();
    }
    ++gen;
    __syncthreads();
}

// Per-simulation coefficients of the current step, read by every thread of the CTA.
template <int P>
struct SimCoef {
    double C, kap2, beta2;      // Courant, 2 kap, 2 beta (kapdot = beta Cdot)
    double Cd[P > 0 ? P : 1];   // Cdot of every tangent lane
    int active, sample;         // march this step / sample step (all moments)
};

// One thread's K bins of a tile: fluxes of K+1 faces from the smem window, update, moment
// partials, 16-byte stores.  NEG = (C < 0) (direction is uniform per tile).
// LK: limiter kind (0 upwind, 1 van Leer, 2 minmod/superbee/MC via psi_half_dl)
template <int P, int K, bool NEG, int LK>
__device__ __forceinline__ void stream_bins(const double* __restrict__ sb, int RS, int g0, int nb, int i_base,
                                            const SimCoef<P>& cf, int lim, bool sample, double L_half, double dL,
                                            double* __restrict__ drow, long long pitch,
                                            double (&acc)[4][1 + P], bool& neg) {
    constexpr int V = 1 + P;
    constexpr int PP = P > 0 ? P : 1;
    const double C = cf.C, kap2 = cf.kap2, beta2 = cf.beta2;
    // window x[v][0..K+3] = bins g0-2 .. g0+K+1 of the tile (smem row index g0 .. g0+K+3)
    double x[V][K + 4];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const double2* w2 = reinterpret_cast<const double2*>(sb + (size_t)v * RS + g0);
#pragma unroll
        for (int q = 0; q < (K + 4) / 2; ++q) { const double2 d = w2[q]; x[v][2 * q] = d.x; x[v][2 * q + 1] = d.y; }
    }
    double F[K + 1], Fd[K + 1][PP];
#pragma unroll
    for (int f = 2; f <= K + 2; ++f) {       // face between window cells f-1 | f
        const int u = NEG ? f : f - 1;
        const int ja = NEG ? f + 1 : f - 1;
        const double a = x[0][ja] - x[0][ja - 1], b = x[0][f] - x[0][f - 1];
        double h = 0.0, qa = 0.0, qb = 0.0;
        if (LK == 2) psi_half_dl(lim, a, b, h, qa, qb);
        else if (LK == 1) {
            if (P == 0) h = psi_half_vl_sf(a, b);            // primal only: select-free
            else psi_half_d_bf(a, b, h, qa, qb);
        }
        const double nup = x[0][u];
        F[f - 2] = fma(C, nup, kap2 * h);
        if (P > 0) {
            // lane flux regrouped over the three cells it touches (see k_resident.cuh face_lane)
            const double gq = fma(beta2, h, nup), pak = kap2 * qa, pbk = kap2 * qb;
            const int lo = NEG ? f - 1 : f - 2;
            const double w_hi = NEG ? pak : pbk;
            const double w_mid = NEG ? C - (pak - pbk) : C + (pak - pbk);
            const double w_lo = NEG ? -pbk : -pak;
#pragma unroll
            for (int p = 0; p < P; ++p)
                Fd[f - 2][p] = fma(cf.Cd[p], gq, fma(w_hi, x[1 + p][lo + 2], fma(w_mid, x[1 + p][lo + 1], w_lo * x[1 + p][lo])));
        }
    }
    double y[V][K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double nn = x[0][k + 2] - (F[k + 1] - F[k]);
        neg |= (nn < 0.0);
        y[0][k] = nn;
#pragma unroll
        for (int p = 0; p < P; ++p) y[1 + p][k] = x[1 + p][k + 2] - (Fd[k + 1][p] - Fd[k][p]);
    }
    // moment partials (mu3 every step; all moments on sample steps); bins >= nb excluded
    const bool full = g0 + K <= nb;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double Lc = fma((double)(i_base + g0 + k), dL, L_half);
        const double w1 = dL * Lc, w2 = w1 * Lc, w3 = w2 * Lc;
        const bool in = full || (g0 + k < nb);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const double yv = in ? y[v][k] : 0.0;
            acc[3][v] = fma(w3, yv, acc[3][v]);
            if (sample) {
                acc[0][v] = fma(dL, yv, acc[0][v]);
                acc[1][v] = fma(w1, yv, acc[1][v]);
                acc[2][v] = fma(w2, yv, acc[2][v]);
            }
        }
    }
    // 16-byte stores (row index of tile bin g0 is i_base + g0 + 2: 16-byte aligned)
#pragma unroll
    for (int v = 0; v < V; ++v) {
        double* d1 = drow + (size_t)v * pitch + g0;
        if (full) {
            double2* d2 = reinterpret_cast<double2*>(d1);
#pragma unroll
            for (int q = 0; q < K / 2; ++q) d2[q] = make_double2(y[v][2 * q], y[v][2 * q + 1]);
        } else {
            for (int k = 0; k < K && g0 + k < nb; ++k) d1[k] = y[v][k];
        }
    }
}

// DYN = false: every CTA streams a static contiguous tile range and replicates the scalar phase of
// the <= STREAM_MAXS simulations it touches.  DYN = true (default): tiles are handed out by a per-
// step atomic counter (a CTA that finishes early takes more: no imbalance wait at the grid barrier);
// simulation s is owned by CTA s % G (slot s / G), whose warp publishes the step coefficients to
// global memory with a release flag that the producers acquire before streaming s's tiles.  Tile
// partials keep their [s][tile][warp] slots, so every sum keeps its fixed order (bitwise the same
// results as the static schedule).
template <int P, bool DYN>
__global__ void __launch_bounds__(STREAM_NT, StreamCfg<1 + P>::MINB) k_stream(const StreamParams sp) {
    constexpr int V = 1 + P;
    constexpr int K = StreamCfg<V>::K;
    constexpr int STG = StreamCfg<V>::STAGES;
    constexpr int NWC = STREAM_NWC;
    const KParams& kp = sp.kp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = (warp == NWC);
    const int N = kp.N, TB = sp.TB;
    const int RS = TB + 4;                          // smem row (tile + halos), doubles
    const bool steps_mode = kp.n_steps > 0;
    const unsigned G = gridDim.x;
    const double L_half = kp.L_lo + 0.5 * kp.dL;

    // static tile range of this CTA (DYN: only the owned simulations s = blockIdx + slot G)
    const long long t_lo = DYN ? 0 : (sp.n_tiles * blockIdx.x) / G;
    const long long t_hi = DYN ? 0 : (sp.n_tiles * (blockIdx.x + 1)) / G;
    const int s_lo = DYN ? 0 : (int)(t_lo / sp.T_sim);
    const int ns = DYN ? (kp.n_sims > (int)blockIdx.x ? (kp.n_sims - (int)blockIdx.x + (int)G - 1) / (int)G : 0)
                       : ((t_hi > t_lo) ? (int)((t_hi - 1) / sp.T_sim) - s_lo + 1 : 0);
    auto sim_of_slot = [&](int slot) { return DYN ? (int)blockIdx.x + slot * (int)G : s_lo + slot; };
    auto is_owner = [&](int slot) { return DYN || (long long)(s_lo + slot) * sp.T_sim >= t_lo; };

    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) unsigned long long s_full[STG], s_empty[STG];
    __shared__ SimCoef<P> s_coef[STREAM_MAXS];
    __shared__ double s_clip[STREAM_MAXS];
    __shared__ SimCoef<P> s_cfs[DYN ? STG : 1];      // DYN: coefficients of the tile in each stage
    __shared__ long long s_tile[DYN ? STG : 1];      // DYN: tile id in each stage (-1: end of step)
    SimCoef<P>* gcoef = reinterpret_cast<SimCoef<P>*>(sp.coef);
    // DYN: the owner publishes slot's coefficients of step `step` (every lane has them in s_coef)
    auto publish = [&](int slot, unsigned step) {
        if (!DYN) return;
        __syncwarp();
        const int s = sim_of_slot(slot);
        if (lane == 0) {
            gcoef[s] = s_coef[slot];
            __threadfence();
            st_release(&sp.coef_step[s], step);
        }
    };

    // per-simulation scalar state: primal per slot (lane 0 copy), tangent per (slot, lane)
    struct SimPrimal { double c, t, mu3p, dt, loss, rms_c, rms_L; long long nstep; int m, status, landing, go; };
    struct SimTan { double c, t, mu3p, dt, gacc; };
    __shared__ SimPrimal s_sp[STREAM_MAXS];
    __shared__ SimTan s_st[STREAM_MAXS][32];

    if (tid == 0) {
        for (int i = 0; i < STG; ++i) { mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], NWC); }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    const int pl = lane < kp.P ? lane : -1;
    auto kinetics = [&](int slot, int s, SimPrimal& W, SimTan& T) -> bool {
        const KinLoader KL{kp.theta + (size_t)s * kp.n_params, kp.sol, kp.seed, pl, kp.n_params, kp.n_params + kp.n_sol};
        const double* kT = kp.knot_T + (size_t)s * kp.knotT_stride;
        const D1 t = mk(W.t, T.t), c = mk(W.c, T.c);
        const KinCache KC = kin_cache(kp, KL, kT);
        D1 Tk;
        const D1 S = supersaturation(kp, KL, kT, KC, t, c, Tk);
        const D1 Gr = growth_rate(kp, KL, S, Tk);
        const double tn = steps_mode ? 0.0 : kp.t_samples[W.m];
        const StepScalars sc = time_step(kp, Gr, t, tn, steps_mode);
        if (sc.err != ST_OK) { W.status = sc.err; return false; }
        W.dt = sc.dt.v; T.dt = sc.dt.d;
        W.landing = sc.landing;
        const double C = sc.C.v;
        if (lane == 0) {
            s_coef[slot].C = C;
            s_coef[slot].kap2 = 2.0 * sc.kap.v;
            s_coef[slot].beta2 = C > 0.0 ? (1.0 - 2.0 * C) : (C < 0.0 ? -(1.0 + 2.0 * C) : 0.0);
        }
        // every lane slot < P is written (unused lanes >= kp.P carry 0, never uninitialised smem)
        if (lane < P) s_coef[slot].Cd[lane] = (pl >= 0) ? sc.C.d : 0.0;
        return true;
    };
    auto set_inactive = [&](int slot) {
        if (lane == 0) { s_coef[slot].active = 0; s_coef[slot].sample = 0; }
    };
    // totals of simulation s from the per-(tile, warp) partials, fixed order (deterministic):
    // lane l sums entries e = l, l + 32, ...; then a fixed xor tree per value.
    auto sim_totals = [&](int s, bool sample, double (&tot)[4], double (&totd)[4], double& badf) {
        const double* pt = sp.part + (size_t)s * sp.T_sim * NWC * 5 * V;
        const int ne = sp.T_sim * NWC;
        double a[4][V];
#pragma unroll
        for (int km = 0; km < 4; ++km)
#pragma unroll
            for (int v = 0; v < V; ++v) a[km][v] = 0.0;
        double bf = 0.0;
        // The entries are L2 round trips (written by other SMs this step): load UB entries into
        // registers before adding, so one round trip serves UB entries.  The per-lane addition
        // order is unchanged (bitwise identical totals).
        auto accum = [&](auto SAMPLE) {
            constexpr bool SM = decltype(SAMPLE)::value;
            constexpr int NKM = SM ? 4 : 1;                  // moments summed: all, or mu3 only
            constexpr int NX = NKM * V + 1;                  // + negative flag
            constexpr int UB = 16 / NX > 2 ? 16 / NX : 2;
            int e = lane;
            for (; e + 32 * (UB - 1) < ne; e += 32 * UB) {
                double x[UB][NX];
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                    const double* q = pt + (size_t)(e + 32 * u) * 5 * V;
#pragma unroll
                    for (int j = 0; j < NKM; ++j)
#pragma unroll
                        for (int v = 0; v < V; ++v) x[u][j * V + v] = q[(SM ? j : 3) * V + v];
                    x[u][NKM * V] = q[4 * V];
                }
#pragma unroll
                for (int u = 0; u < UB; ++u) {
#pragma unroll
                    for (int j = 0; j < NKM; ++j)
#pragma unroll
                        for (int v = 0; v < V; ++v) a[SM ? j : 3][v] += x[u][j * V + v];
                    bf += x[u][NKM * V];
                }
            }
            for (; e < ne; e += 32) {
                const double* q = pt + (size_t)e * 5 * V;
#pragma unroll
                for (int j = 0; j < NKM; ++j)
#pragma unroll
                    for (int v = 0; v < V; ++v) a[SM ? j : 3][v] += q[(SM ? j : 3) * V + v];
                bf += q[4 * V];
            }
        };
        if (sample) accum(std::true_type{}); else accum(std::false_type{});
#pragma unroll
        for (int km = 0; km < 4; ++km) {
            tot[km] = 0.0; totd[km] = 0.0;
            if (km == 3 || sample) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                    for (int v = 0; v < V; ++v) a[km][v] += __shfl_xor_sync(0xffffffffu, a[km][v], off);
                tot[km] = a[km][0];
#pragma unroll
                for (int p = 0; p < P; ++p) if (p == pl) totd[km] = a[km][1 + p];
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) bf += __shfl_xor_sync(0xffffffffu, bf, off);
        badf = bf;
    };

    // DYN: the totals of every owned simulation summed by all NWC consumer warps of the CTA (the
    // sum is on the step's critical path: the other CTAs' producers wait for the coefficients).
    // Warp w takes entries e with (e / 32) % NWC == w, lane l entries e % 32 == l, in increasing
    // order; lanes combine by a fixed xor tree, warps in warp order: deterministic.
    constexpr int NXV = 4 * V + 1;
    __shared__ double s_wtot[DYN ? STREAM_MAXS : 1][DYN ? NWC : 1][DYN ? NXV : 1];
    auto cta_partials = [&](int slot, bool sample) {
        const int s = sim_of_slot(slot);
        const double* pt = sp.part + (size_t)s * sp.T_sim * NWC * 5 * V;
        const int ne = sp.T_sim * NWC;
        double a[NXV];
#pragma unroll
        for (int x = 0; x < NXV; ++x) a[x] = 0.0;
#pragma unroll 4
        for (int e = warp * 32 + lane; e < ne; e += NWC * 32) {             // independent L2 loads
            const double* q = pt + (size_t)e * 5 * V;
            if (sample) {
#pragma unroll
                for (int x = 0; x < 4 * V; ++x) a[x] += q[x];
            } else {
#pragma unroll
                for (int v = 0; v < V; ++v) a[3 * V + v] += q[3 * V + v];
            }
            a[4 * V] += q[4 * V];
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
            for (int x = 0; x < NXV; ++x) a[x] += __shfl_xor_sync(0xffffffffu, a[x], off);
        if (lane < NXV) {
            double mine = 0.0;
#pragma unroll
            for (int x = 0; x < NXV; ++x) if (x == lane) mine = a[x];
            s_wtot[slot][warp][lane] = mine;
        }
    };
    auto cta_totals = [&](int slot, bool sample, double (&tot)[4], double (&totd)[4], double& badf) {
        double a[NXV];
#pragma unroll
        for (int x = 0; x < NXV; ++x) a[x] = 0.0;
        for (int w = 0; w < NWC; ++w)
#pragma unroll
            for (int x = 0; x < NXV; ++x) a[x] += s_wtot[slot][w][x];
#pragma unroll
        for (int km = 0; km < 4; ++km) {
            const bool on = km == 3 || sample;
            tot[km] = on ? a[km * V] : 0.0;
            totd[km] = 0.0;
#pragma unroll
            for (int p = 0; p < P; ++p) if (p == pl && on) totd[km] = a[km * V + 1 + p];
        }
        badf = a[4 * V];
    };

    // ---- scalar state init (one warp per simulation slot); mu3(n0) from the load kernel's
    //      per-tile partials (same layout and order as a step) ----------------------------
    if (warp < ns) {
        const int slot = warp, s = sim_of_slot(slot);
        double tot[4], totd[4], badf;
        sim_totals(s, false, tot, totd, badf);
        SimPrimal W{};
        SimTan T{};
        W.c = kp.c0[s]; W.t = 0.0; W.mu3p = tot[3]; W.dt = 0.0; W.loss = 0.0; W.rms_c = 1.0; W.rms_L = 1.0;
        W.nstep = 0; W.m = 0; W.status = ST_OK; W.landing = 0; W.go = 1;
        T.c = T.t = T.mu3p = T.dt = T.gacc = 0.0;
        if (kp.target) {
            const double* tg = kp.target + (size_t)s * kp.M * 2;
            double sc2 = 0.0, sl2 = 0.0;
            for (int j = lane; j < kp.M; j += 32) { sc2 += tg[2 * j] * tg[2 * j]; sl2 += tg[2 * j + 1] * tg[2 * j + 1]; }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                sc2 += __shfl_xor_sync(0xffffffffu, sc2, off);
                sl2 += __shfl_xor_sync(0xffffffffu, sl2, off);
            }
            W.rms_c = sqrt(sc2 / kp.M); W.rms_L = sqrt(sl2 / kp.M);
        }
        if (lane == 0) s_clip[slot] = 1e-12 * __longlong_as_double((long long)sp.nscale_bits[s]);
        if (kp.max_steps <= 0) { W.status = ST_MAXSTEPS; W.go = 0; }
        if (W.go && !kinetics(slot, s, W, T)) W.go = 0;
        if (W.go) {
            if (lane == 0) { s_coef[slot].active = 1; s_coef[slot].sample = W.landing || (steps_mode && kp.n_steps == 1); }
        } else {
            set_inactive(slot);
        }
        publish(slot, 0u);
        __syncwarp();
        if (lane == 0) s_sp[slot] = W;
        s_st[slot][lane] = T;
    }
    __syncthreads();

    unsigned gen = 0;
    long long n = 0;
#if PBE_TIMING
    unsigned long long tc_work = 0, tc_wait = 0, tc_scal = 0, tc_steps = 0, tc_top = clock64(), tc_arr = 0;
#endif
    int src_sel = 0;
    unsigned long long qq = 0;          // running tile counter (stage = qq % STG, phase = (qq / STG) & 1)
    const int vl = kp.limiter;
    auto tile_active = [&](long long t) { return s_coef[(int)(t / sp.T_sim) - s_lo].active != 0; };
    auto next_active = [&](long long t) { while (t < t_hi && !tile_active(t)) ++t; return t; };
    while (true) {
        const double* src = src_sel ? sp.buf1 : sp.buf0;
        double* dst = src_sel ? sp.buf0 : sp.buf1;
        const unsigned long long q0 = qq;
        if (DYN) {
            if (producer) {
                // ---- TMA producer: tiles from the step's atomic counter, in counter order ----------
                if (lane == 0) {
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    unsigned long long q = q0;
                    while (true) {
                        long long t = (long long)atomicAdd(&sp.tile_ctr[n % 3], 1u);
                        int s = 0;
                        bool live = false;
                        while (t < sp.n_tiles) {
                            s = (int)(t / sp.T_sim);
                            while (ld_acquire(&sp.coef_step[s]) != (unsigned)n) __nanosleep(20);
                            if (gcoef[s].active) { live = true; break; }
                            // inactive simulation: skip the rest of its tiles in one step
                            atomicMax(&sp.tile_ctr[n % 3], (unsigned)((long long)(s + 1) * sp.T_sim));
                            t = (long long)atomicAdd(&sp.tile_ctr[n % 3], 1u);
                        }
                        const int st = (int)(q % STG);
                        if (q >= STG) mbar_wait(&s_empty[st], (unsigned)(((q / STG) - 1) & 1));
                        ++q;
                        if (!live) {                       // end of the step for this CTA
                            s_tile[st] = -1;
                            mbar_arrive(&s_full[st]);
                            break;
                        }
                        s_cfs[st] = gcoef[s];
                        s_tile[st] = t;
                        const int j = (int)(t - (long long)s * sp.T_sim);
                        const int b0 = j * TB, nb = min(TB, N - b0);
                        const unsigned n_el = (unsigned)((nb + 4 + 1) & ~1);   // even -> 16-byte multiple
                        mbar_expect_tx(&s_full[st], n_el * 8u * V);
#pragma unroll
                        for (int v = 0; v < V; ++v)
                            bulk_g2s(smem + ((size_t)st * V + v) * RS, src + ((size_t)s * V + v) * sp.pitch + b0,
                                     n_el * 8u, &s_full[st]);
                    }
                    qq = q;
                }
                qq = __shfl_sync(0xffffffffu, qq, 0);
            } else {
                // ---- consumers: whatever tile each stage holds, until the end marker ----------------
                while (true) {
                    const int st = (int)(qq % STG);
                    mbar_wait(&s_full[st], (unsigned)((qq / STG) & 1));
                    ++qq;
                    const long long t = s_tile[st];
                    if (t < 0) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&s_empty[st]);
                        break;
                    }
                    const int s = (int)(t / sp.T_sim), j = (int)(t - (long long)s * sp.T_sim);
                    const int b0 = j * TB, nb = min(TB, N - b0);
                    const SimCoef<P> cf = s_cfs[st];
                    const bool sample = cf.sample != 0;
                    const double* sb = smem + (size_t)st * V * RS;
                    double* drow = dst + (size_t)s * V * sp.pitch + b0 + 2;
                    double acc[4][V];
#pragma unroll
                    for (int km = 0; km < 4; ++km)
#pragma unroll
                        for (int v = 0; v < V; ++v) acc[km][v] = 0.0;
                    bool neg = false;
#define PBE_SB(NEGV, LKV)                                                                                  \
    for (int g0 = (warp * 32 + lane) * K; g0 < nb; g0 += NWC * 32 * K)                                     \
        stream_bins<P, K, NEGV, LKV>(sb, RS, g0, nb, b0, cf, vl, sample, L_half, kp.dL, drow, sp.pitch, acc, neg)
                    const int lk = vl == LIM_VANLEER ? 1 : (vl == LIM_UPWIND ? 0 : 2);
                    if (cf.C >= 0.0) {
                        if (lk == 1) PBE_SB(false, 1); else if (lk == 0) PBE_SB(false, 0); else PBE_SB(false, 2);
                    } else {
                        if (lk == 1) PBE_SB(true, 1); else if (lk == 0) PBE_SB(true, 0); else PBE_SB(true, 2);
                    }
#undef PBE_SB
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&s_empty[st]);           // stage free for the producer
                    bool bad = false;
                    if (__any_sync(0xffffffffu, neg)) {
                        const double thr = 1e-12 * __longlong_as_double((long long)sp.nscale_bits[s]);
                        for (int g0 = (warp * 32 + lane) * K; g0 < nb; g0 += NWC * 32 * K)
                            for (int k = 0; k < K && g0 + k < nb; ++k) {
                                const double nn = drow[g0 + k];
                                if (nn < 0.0) {
                                    if (nn >= -thr) {
                                        const double Lc = fma((double)(b0 + g0 + k), kp.dL, L_half);
                                        const double w1 = kp.dL * Lc, w2 = w1 * Lc, w3 = w2 * Lc;
#pragma unroll
                                        for (int v = 0; v < V; ++v) {
                                            const double yv = drow[(size_t)v * sp.pitch + g0 + k];
                                            acc[3][v] -= w3 * yv;
                                            if (sample) { acc[0][v] -= kp.dL * yv; acc[1][v] -= w1 * yv; acc[2][v] -= w2 * yv; }
                                            drow[(size_t)v * sp.pitch + g0 + k] = 0.0;
                                        }
                                    } else {
                                        bad = true;
                                    }
                                }
                            }
                    }
                    double* pt = sp.part + (((size_t)s * sp.T_sim + j) * NWC + warp) * 5 * V;
#pragma unroll
                    for (int km = 0; km < 4; ++km) {
                        if (km == 3 || sample) {
                            double r[V];
#pragma unroll
                            for (int v = 0; v < V; ++v) r[v] = acc[km][v];
                            warp_transpose_reduce<V>(r, lane);
                            const int idx = reduce_index<V>(lane);
                            if (idx < V) pt[km * V + idx] = r[0];
                        }
                    }
                    const bool bad_any = __any_sync(0xffffffffu, bad);
                    if (lane == 0) pt[4 * V] = bad_any ? 1.0 : 0.0;
                }
            }
        } else {
        if (producer) {
            // ---- TMA producer: one elected lane streams the active tiles through the stages ----
            if (lane == 0) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
                unsigned long long q = q0;
                for (long long t = next_active(t_lo); t < t_hi; t = next_active(t + 1), ++q) {
                    const int st = (int)(q % STG);
                    if (q >= STG) mbar_wait(&s_empty[st], (unsigned)(((q / STG) - 1) & 1));
                    const int s = (int)(t / sp.T_sim), j = (int)(t - (long long)s * sp.T_sim);
                    const int b0 = j * TB, nb = min(TB, N - b0);
                    const unsigned n_el = (unsigned)((nb + 4 + 1) & ~1);   // even -> 16-byte multiple
                    mbar_expect_tx(&s_full[st], n_el * 8u * V);
#pragma unroll
                    for (int v = 0; v < V; ++v)
                        bulk_g2s(smem + ((size_t)st * V + v) * RS, src + ((size_t)s * V + v) * sp.pitch + b0,
                                 n_el * 8u, &s_full[st]);
                }
            }
            // the producer warp counts the same tiles as the consumers
            for (long long t = next_active(t_lo); t < t_hi; t = next_active(t + 1)) ++qq;
        } else {
            // ---- consumers --------------------------------------------------------------------
            for (long long t = next_active(t_lo); t < t_hi; t = next_active(t + 1), ++qq) {
                const int st = (int)(qq % STG);
                mbar_wait(&s_full[st], (unsigned)((qq / STG) & 1));
                const int s = (int)(t / sp.T_sim), j = (int)(t - (long long)s * sp.T_sim);
                const int b0 = j * TB, nb = min(TB, N - b0);
                const int slot = s - s_lo;
                const SimCoef<P>& cf = s_coef[slot];
                const bool sample = cf.sample != 0;
                const double* sb = smem + (size_t)st * V * RS;
                double* drow = dst + (size_t)s * V * sp.pitch + b0 + 2;
                double acc[4][V];
#pragma unroll
                for (int km = 0; km < 4; ++km)
#pragma unroll
                    for (int v = 0; v < V; ++v) acc[km][v] = 0.0;
                bool neg = false;
#define PBE_SB(NEGV, LKV)                                                                                  \
    for (int g0 = (warp * 32 + lane) * K; g0 < nb; g0 += NWC * 32 * K)                                     \
        stream_bins<P, K, NEGV, LKV>(sb, RS, g0, nb, b0, cf, vl, sample, L_half, kp.dL, drow, sp.pitch, acc, neg)
                const int lk = vl == LIM_VANLEER ? 1 : (vl == LIM_UPWIND ? 0 : 2);
                if (cf.C >= 0.0) {
                    if (lk == 1) PBE_SB(false, 1); else if (lk == 0) PBE_SB(false, 0); else PBE_SB(false, 2);
                } else {
                    if (lk == 1) PBE_SB(true, 1); else if (lk == 0) PBE_SB(true, 0); else PBE_SB(true, 2);
                }
#undef PBE_SB
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_empty[st]);           // stage free for the producer
                // round-off clip (R-17), rare: fix the stored values of this warp's bins
                bool bad = false;
                if (__any_sync(0xffffffffu, neg)) {
#if PBE_TIMING
                    if (lane == 0 && blockIdx.x < 1024) atomicAdd(&g_stream_cycles[blockIdx.x][4], 1ull);
#endif
                    const double thr = s_clip[slot];
                    for (int g0 = (warp * 32 + lane) * K; g0 < nb; g0 += NWC * 32 * K)
                        for (int k = 0; k < K && g0 + k < nb; ++k) {
                            const double nn = drow[g0 + k];
                            if (nn < 0.0) {
                                if (nn >= -thr) {
                                    // zero the bin and its tangents; remove it from the partials
                                    const double Lc = fma((double)(b0 + g0 + k), kp.dL, L_half);
                                    const double w1 = kp.dL * Lc, w2 = w1 * Lc, w3 = w2 * Lc;
#pragma unroll
                                    for (int v = 0; v < V; ++v) {
                                        const double yv = drow[(size_t)v * sp.pitch + g0 + k];
                                        acc[3][v] -= w3 * yv;
                                        if (sample) { acc[0][v] -= kp.dL * yv; acc[1][v] -= w1 * yv; acc[2][v] -= w2 * yv; }
                                        drow[(size_t)v * sp.pitch + g0 + k] = 0.0;
                                    }
                                } else {
                                    bad = true;
                                }
                            }
                        }
                }
                // per-warp tile partials
                double* pt = sp.part + (((size_t)s * sp.T_sim + j) * NWC + warp) * 5 * V;
#pragma unroll
                for (int km = 0; km < 4; ++km) {
                    if (km == 3 || sample) {
                        double r[V];
#pragma unroll
                        for (int v = 0; v < V; ++v) r[v] = acc[km][v];
                        warp_transpose_reduce<V>(r, lane);
                        const int idx = reduce_index<V>(lane);
                        if (idx < V) pt[km * V + idx] = r[0];
                    }
                }
                const bool bad_any = __any_sync(0xffffffffu, bad);
                if (lane == 0) pt[4 * V] = bad_any ? 1.0 : 0.0;
            }
        }

        }

        // ---- grid barrier + active count ------------------------------------------------------
        if (tid == 0) {
            int mine = 0;
            for (int slot = 0; slot < ns; ++slot)
                if (is_owner(slot) && s_coef[slot].active) ++mine;                       // owner CTA counts
            if (mine) atomicAdd(&sp.active[n % 3], mine);
        }
#if PBE_TIMING
        __syncthreads();
        tc_arr = clock64();
        tc_work += tc_arr - tc_top;
#endif
        grid_sync(sp.bar, G, gen);
#if PBE_TIMING
        const unsigned long long tc_rel = clock64();
        tc_wait += tc_rel - tc_arr;
        ++tc_steps;
#endif
        const int still = *((volatile int*)&sp.active[n % 3]);
        if (blockIdx.x == 0 && tid == 0) {
            sp.active[(n + 2) % 3] = 0;                                   // read by all before barrier n
            if (DYN) sp.tile_ctr[(n + 2) % 3] = 0u;                       // used by all before barrier n
        }
        if (still == 0) break;

        // ---- scalar phase: one warp per simulation slot ----------------------------------------
        if (DYN) {
            if (warp < NWC)
                for (int slot = 0; slot < ns; ++slot)
                    if (s_coef[slot].active) cta_partials(slot, s_coef[slot].sample != 0);
            __syncthreads();
        }
        if (DYN && warp < ns && !s_coef[warp].active) publish(warp, (unsigned)(n + 1));   // stays inactive
        if (warp < ns && s_coef[warp].active) {
            const int slot = warp, s = sim_of_slot(slot);
            const bool owner = is_owner(slot);
            SimPrimal W = s_sp[slot];
            SimTan T = s_st[slot][lane];
            const bool sample = s_coef[slot].sample != 0;
            double tot[4], totd[4], badf;
            if (DYN) cta_totals(slot, sample, tot, totd, badf);
            else sim_totals(s, sample, tot, totd, badf);
            const D1 mu3n = mk(tot[3], totd[3]);
            const D1 c = mk(W.c, T.c), mu3p = mk(W.mu3p, T.mu3p);
            const D1 cn = c - kp.rho_kv * (mu3n - mu3p);
            bool go = true;
            if (badf > 0.0) { W.status = ST_NEG; go = false; }
            else if (cn.v < 0.0) { W.status = ST_INFEAS; go = false; }
            else {
                W.c = cn.v; T.c = cn.d; W.mu3p = mu3n.v; T.mu3p = mu3n.d;
                if (W.landing) { W.t = kp.t_samples[W.m]; T.t = 0.0; }
                else { W.t = W.t + W.dt; T.t = T.t + T.dt; }
                ++W.nstep;
                if (sample && owner) {
                    const int mr = steps_mode ? 0 : W.m;
                    double* r = kp.rec + ((size_t)s * kp.M + mr) * 6;
                    if (lane == 0) { r[0] = W.t; r[1] = W.c; r[2] = tot[0]; r[3] = tot[1]; r[4] = tot[2]; r[5] = tot[3]; }
                    if (pl >= 0) {
                        double* rt = kp.trec + (((size_t)s * kp.M + mr) * kp.P + pl) * 5;
                        rt[0] = T.c; rt[1] = totd[0]; rt[2] = totd[1]; rt[3] = totd[2]; rt[4] = totd[3];
                    }
                    if (kp.target) {
                        const double* tg = kp.target + (size_t)s * kp.M * 2;
                        const double Lb = tot[1] / tot[0];
                        const double Lbd = (totd[1] * tot[0] - tot[1] * totd[0]) / (tot[0] * tot[0]);
                        const double rc = (W.c - tg[2 * mr]) / W.rms_c, rL = (Lb - tg[2 * mr + 1]) / W.rms_L;
                        W.loss += rc * rc + rL * rL;
                        T.gacc += 2.0 * (rc / W.rms_c) * T.c + 2.0 * (rL / W.rms_L) * Lbd;
                    }
                }
                if (W.landing) ++W.m;
                if (steps_mode ? (W.nstep >= kp.n_steps) : (W.m >= kp.M)) go = false;
                else if (W.nstep >= kp.max_steps) { W.status = ST_MAXSTEPS; go = false; }
                else go = kinetics(slot, s, W, T);
            }
            W.go = go;
            if (go) {
                if (lane == 0) s_coef[slot].sample = W.landing || (steps_mode && W.nstep + 1 == kp.n_steps);
            } else {
                set_inactive(slot);
                if (owner && lane == 0) sp.final_buf[s] = src_sel ^ 1;   // state of this step is in dst
            }
            publish(slot, (unsigned)(n + 1));
            __syncwarp();
            if (lane == 0) s_sp[slot] = W;
            s_st[slot][lane] = T;
        }
        __syncthreads();
#if PBE_TIMING
        tc_top = clock64();
        tc_scal += tc_top - tc_rel;
#endif
        src_sel ^= 1;
        ++n;
    }

#if PBE_TIMING
    if (threadIdx.x == 0 && blockIdx.x < 1024) {
        g_stream_cycles[blockIdx.x][0] = tc_work; g_stream_cycles[blockIdx.x][1] = tc_wait;
        g_stream_cycles[blockIdx.x][2] = tc_scal; g_stream_cycles[blockIdx.x][3] = tc_steps;
    }
#endif
    // ---- epilogue: per-simulation status / loss / gradient (owner CTA) --------------------------
    if (warp < ns) {
        const int slot = warp, s = sim_of_slot(slot);
        if (is_owner(slot)) {
            const SimPrimal W = s_sp[slot];
            const SimTan T = s_st[slot][lane];
            const bool ok = W.status == ST_OK;
            const double qnan = __longlong_as_double(0x7ff8000000000000ll);
            if (lane == 0) {
                kp.status[s] = W.status;
                kp.steps[s] = W.nstep;
                if (kp.loss) kp.loss[s] = (kp.target && ok) ? W.loss : qnan;
                if (W.nstep == 0) sp.final_buf[s] = 0;
            }
            if (pl >= 0 && kp.grad) kp.grad[(size_t)s * kp.P + pl] = (kp.target && ok) ? T.gacc : qnan;
        }
    }
}

// n0 (caller layout [S or 1][N]) -> padded buffer 0; tangent rows 0; per-sim max(n0) bits;
// mu3(n0) partial of every tile in the step-partial layout (warp slot 0, fixed order).
// Grid (T_sim, S), 256 threads: one CTA per tile.
template <int V>
__global__ void __launch_bounds__(256) k_stream_load(const double* __restrict__ n0, long long n0_stride, int N, int S,
                              double* __restrict__ buf, long long pitch, unsigned long long* nscale_bits,
                              int TB, int T_sim, double* __restrict__ part, double L_lo, double dL) {
    const int s = blockIdx.y, j = blockIdx.x;
    const int b0 = j * TB, nb = min(TB, N - b0);
    double m = 0.0, a3 = 0.0;
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        const int i = b0 + k;
        const double v = n0[(size_t)s * n0_stride + i];
        buf[(size_t)s * V * pitch + 2 + i] = v;
#pragma unroll
        for (int p = 1; p < V; ++p) buf[((size_t)s * V + p) * pitch + 2 + i] = 0.0;
        m = fmax(m, v);
        const double Lc = fma((double)i, dL, L_lo + 0.5 * dL);
        a3 = fma(dL * Lc * Lc * Lc, v, a3);
    }
    __shared__ double s_a[8];
    __shared__ double s_m[8];
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
        double* pt = part + ((size_t)s * T_sim + j) * STREAM_NWC * 5 * V;
        for (int e = 0; e < STREAM_NWC * 5 * V; ++e) pt[e] = 0.0;
        pt[3 * V] = t;
        atomicMax(nscale_bits + s, (unsigned long long)__double_as_longlong(mm));
    }
}

// final state (buffer chosen per simulation) -> caller n_final [S][N] / ndot_final [S][P][N]
template <int V>
__global__ void k_stream_store(const double* __restrict__ buf0, const double* __restrict__ buf1,
                               const int* __restrict__ final_buf, int N, int P, long long pitch,
                               double* __restrict__ n_final, double* __restrict__ ndot_final) {
    const int s = blockIdx.y;
    const double* b = final_buf[s] ? buf1 : buf0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        if (n_final) n_final[(size_t)s * N + i] = b[(size_t)s * V * pitch + 2 + i];
        if (ndot_final)
            for (int p = 0; p < P; ++p)
                ndot_final[((size_t)s * P + p) * N + i] = b[((size_t)s * V + 1 + p) * pitch + 2 + i];
    }
}

}  // namespace pbe
