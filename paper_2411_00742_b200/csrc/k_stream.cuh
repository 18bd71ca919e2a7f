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

#include "pbe_device.cuh"

namespace pbe {

constexpr int STREAM_MAXS = 8;      // simulations one CTA may touch
constexpr int STREAM_NT = 256;      // threads per CTA
template <int V> struct StreamCfg {
    static constexpr int K = V <= 3 ? 4 : 2;        // consecutive bins per thread per pass
    static constexpr int MINB = V == 1 ? 2 : 1;     // CTAs per SM (register budget)
};

struct StreamParams {
    KParams kp;
    double* buf0;           // [S][V][pitch]
    double* buf1;
    long long pitch;        // doubles per (sim, variable) row, >= N + 4, multiple of 4
    int TB;                 // bins per tile (multiple of 4 * STREAM_NT... or of 4)
    int T_sim;              // tiles per simulation
    long long n_tiles;      // S * T_sim
    double* part;           // [S][T_sim][5][V]
    unsigned* bar;          // [2]: arrive count, generation
    int* active;            // [3] rotating counters of simulations still marching
    int* final_buf;         // [S] buffer (0/1) holding each simulation's final state
    const unsigned long long* nscale_bits;  // [S] max(n0_s) as uint64 bits (non-negative)
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

template <int P>
__global__ void __launch_bounds__(STREAM_NT, StreamCfg<1 + P>::MINB) k_stream(const StreamParams sp) {
    constexpr int V = 1 + P;
    constexpr int PP = P > 0 ? P : 1;
    constexpr int K = StreamCfg<V>::K;
    const KParams& kp = sp.kp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = STREAM_NT / 32;
    const int N = kp.N, TB = sp.TB;
    const int RS = TB + 4;                          // smem row (tile + halos), doubles
    const bool steps_mode = kp.n_steps > 0;
    const unsigned G = gridDim.x;

    // static tile range of this CTA
    const long long t_lo = (sp.n_tiles * blockIdx.x) / G;
    const long long t_hi = (sp.n_tiles * (blockIdx.x + 1)) / G;
    const int s_lo = (int)(t_lo / sp.T_sim);
    const int ns = (t_hi > t_lo) ? (int)((t_hi - 1) / sp.T_sim) - s_lo + 1 : 0;

    extern __shared__ __align__(128) double smem[];
    double* stage[2] = {smem, smem + (size_t)V * RS};
    __shared__ __align__(8) unsigned long long s_mbar[2];
    __shared__ SimCoef<P> s_coef[STREAM_MAXS];
    __shared__ double s_red[NW][5][V];
    __shared__ double s_clip[STREAM_MAXS];

    // per-simulation scalar state: primal per slot (lane 0 copy), tangent per (slot, lane)
    struct SimPrimal { double c, t, mu3p, dt, loss, rms_c, rms_L; long long nstep; int m, status, landing, go; };
    struct SimTan { double c, t, mu3p, dt, gacc; };
    __shared__ SimPrimal s_sp[STREAM_MAXS];
    __shared__ SimTan s_st[STREAM_MAXS][32];

    if (tid == 0) { mbar_init(&s_mbar[0], 1); mbar_init(&s_mbar[1], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    // ---- tile bookkeeping ---------------------------------------------------------------
    auto tile_src = [&](long long t, int step_parity, int& s, int& j, int& b0, int& nb) {
        s = (int)(t / sp.T_sim);
        j = (int)(t - (long long)s * sp.T_sim);
        b0 = j * TB;
        nb = min(TB, N - b0);
        (void)step_parity;
    };
    // issue the bulk loads of tile t (all V rows) into stage st
    auto issue = [&](long long t, int st, const double* src) {
        int s, j, b0, nb;
        tile_src(t, 0, s, j, b0, nb);
        const unsigned n_el = (unsigned)((nb + 4 + 1) & ~1);        // even -> 16-byte multiple
        mbar_expect_tx(&s_mbar[st], n_el * 8u * V);
#pragma unroll
        for (int v = 0; v < V; ++v)
            bulk_g2s(stage[st] + (size_t)v * RS, src + ((size_t)s * V + v) * sp.pitch + b0, n_el * 8u, &s_mbar[st]);
    };

    // ---- scalar state init (one warp per simulation slot) ------------------------------
    const int pl = lane < kp.P ? lane : -1;
    auto kinetics = [&](int slot, int s, SimPrimal& W, SimTan& T) -> bool {
        const KinLoader KL{kp.theta + (size_t)s * kp.n_params, kp.sol, kp.seed, pl, kp.n_params, kp.n_params + kp.n_sol};
        const double* kT = kp.knot_T + (size_t)s * kp.knotT_stride;
        const D1 t = mk(W.t, T.t), c = mk(W.c, T.c);
        const D1 Tk = temperature(kp, kT, t);
        const D1 cs = solubility(kp, KL, Tk);
        const D1 S = c / cs;
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
        if (pl >= 0 && pl < P) s_coef[slot].Cd[pl] = sc.C.d;
        return true;
    };
    auto set_inactive = [&](int slot) {
        if (lane == 0) { s_coef[slot].active = 0; s_coef[slot].sample = 0; s_coef[slot].C = 0.0;
                         s_coef[slot].kap2 = 0.0; s_coef[slot].beta2 = 0.0; }
    };

    // mu3(n0) of every simulation of this CTA: partials of step "-1" are not available, so
    // sum the initial buffer directly (each slot warp, fixed order over bins).
    if (warp < ns) {
        const int slot = warp, s = s_lo + slot;
        const double* row = sp.buf0 + (size_t)s * V * sp.pitch + 2;
        double a = 0.0;
        for (int i = lane; i < N; i += 32) {
            const double Lc = fma((double)i, kp.dL, kp.L_lo + 0.5 * kp.dL);
            a = fma(kp.dL * Lc * Lc * Lc, row[i], a);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);   // fixed tree
        SimPrimal W{};
        SimTan T{};
        W.c = kp.c0[s]; W.t = 0.0; W.mu3p = a; W.dt = 0.0; W.loss = 0.0; W.rms_c = 1.0; W.rms_L = 1.0;
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
            if (lane == 0) {
                s_coef[slot].active = 1;
                s_coef[slot].sample = W.landing || (steps_mode && kp.n_steps == 1);
            }
        } else {
            set_inactive(slot);
        }
        __syncwarp();
        if (lane == 0) s_sp[slot] = W;
        s_st[slot][lane] = T;
    }
    __syncthreads();

    unsigned gen = 0;
    long long n = 0;
    int src_sel = 0;
    unsigned phase[2] = {0u, 0u};
    while (true) {
        const double* src = src_sel ? sp.buf1 : sp.buf0;
        double* dst = src_sel ? sp.buf0 : sp.buf1;
        // ---- tiles ----------------------------------------------------------------------
        // skip leading/trailing tiles of inactive simulations
        bool first_issued = false;
        auto tile_active = [&](long long t) { return s_coef[(int)(t / sp.T_sim) - s_lo].active != 0; };
        long long t_next = t_lo;
        while (t_next < t_hi && !tile_active(t_next)) ++t_next;
        if (tid == 0 && t_next < t_hi) { asm volatile("fence.proxy.async.global;" ::: "memory"); issue(t_next, 0, src); }
        first_issued = t_next < t_hi;
        int st = 0;
        for (long long t = t_next; first_issued && t < t_hi;) {
            // find the next active tile to prefetch
            long long tn = t + 1;
            while (tn < t_hi && !tile_active(tn)) ++tn;
            if (tid == 0 && tn < t_hi) issue(tn, st ^ 1, src);
            mbar_wait(&s_mbar[st], phase[st]);
            phase[st] ^= 1u;

            int s, j, b0, nb;
            tile_src(t, 0, s, j, b0, nb);
            const int slot = s - s_lo;
            const SimCoef<P>& cf = s_coef[slot];
            const double C = cf.C, kap2 = cf.kap2, beta2 = cf.beta2;
            const bool sample = cf.sample != 0;
            const double clip_thr = s_clip[slot];
            double Cd[PP];
#pragma unroll
            for (int p = 0; p < PP; ++p) Cd[p] = (p < P) ? cf.Cd[p] : 0.0;
            const double* sb = stage[st];

            double acc[4][V];
#pragma unroll
            for (int km = 0; km < 4; ++km)
#pragma unroll
                for (int v = 0; v < V; ++v) acc[km][v] = 0.0;
            bool bad = false;
            const bool vl = kp.limiter == LIM_VANLEER;

            for (int g0 = tid * K; g0 < nb; g0 += STREAM_NT * K) {
                // window x[v][0..K+3] = bins b0+g0-2 .. b0+g0+K+1 (smem row index g0 .. g0+K+3)
                double x[V][K + 4];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const double2* w2 = reinterpret_cast<const double2*>(sb + (size_t)v * RS + g0);
#pragma unroll
                    for (int q = 0; q < (K + 4) / 2; ++q) { const double2 d = w2[q]; x[v][2 * q] = d.x; x[v][2 * q + 1] = d.y; }
                }
                // face between window cells (f-1, f), f = 2..K+2  (bins b0+g0+f-3 | b0+g0+f-2)
                double F[K + 1], Fd[K + 1][PP];
#pragma unroll
                for (int f = 2; f <= K + 2; ++f) {
                    const int u = C >= 0.0 ? f - 1 : f;
                    const int ja = C >= 0.0 ? f - 1 : f + 1;
                    const double a = x[0][ja] - x[0][ja - 1], b = x[0][f] - x[0][f - 1];
                    double h = 0.0, qa = 0.0, qb = 0.0;
                    if (vl) psi_half_d(a, b, h, qa, qb);
                    const double nup = x[0][u];
                    F[f - 2] = fma(C, nup, kap2 * h);
                    const double gq = fma(beta2, h, nup), pak = kap2 * qa, pbk = kap2 * qb;
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        const double ad = x[1 + p][ja] - x[1 + p][ja - 1], bd = x[1 + p][f] - x[1 + p][f - 1];
                        Fd[f - 2][p] = fma(Cd[p], gq, fma(C, x[1 + p][u], fma(pak, ad, pbk * bd)));
                    }
                }
                // update bins k = 0..K-1 (window cell k + 2)
                double y[V][K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int i = b0 + g0 + k;
                    const double nn = x[0][k + 2] - (F[k + 1] - F[k]);
                    const bool zero = (i >= N) || (nn < 0.0 && nn >= -clip_thr);
                    bad |= (nn < -clip_thr) && (i < N);
                    y[0][k] = zero ? 0.0 : nn;
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        const double nd = x[1 + p][k + 2] - (Fd[k + 1][p] - Fd[k][p]);
                        y[1 + p][k] = zero ? 0.0 : nd;
                    }
                    const double Lc = fma((double)i, kp.dL, kp.L_lo + 0.5 * kp.dL);
                    double w = kp.dL;
#pragma unroll
                    for (int km = 0; km < 4; ++km) {
                        if (km == 3 || sample) {
#pragma unroll
                            for (int v = 0; v < V; ++v) acc[km][v] = fma(w, y[v][k], acc[km][v]);
                        }
                        w *= Lc;
                    }
                }
                // coalesced 16-byte stores (row index of bin b0+g0 is b0+g0+2: 16-byte aligned)
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    double2* d2 = reinterpret_cast<double2*>(dst + ((size_t)s * V + v) * sp.pitch + b0 + g0 + 2);
                    if (g0 + K <= nb) {
#pragma unroll
                        for (int q = 0; q < K / 2; ++q) d2[q] = make_double2(y[v][2 * q], y[v][2 * q + 1]);
                    } else {
                        double* d1 = dst + ((size_t)s * V + v) * sp.pitch + b0 + g0 + 2;
                        for (int k = 0; k < K && g0 + k < nb; ++k) d1[k] = y[v][k];
                    }
                }
            }
            // ---- tile partials: warp transpose-reduce, then warp 0 sums the warps ------------
#pragma unroll
            for (int km = 0; km < 4; ++km) {
                if (km == 3 || sample) {
                    double r[V];
#pragma unroll
                    for (int v = 0; v < V; ++v) r[v] = acc[km][v];
                    warp_transpose_reduce<V>(r, lane);
                    const int idx = reduce_index<V>(lane);
                    if (idx < V) s_red[warp][km][idx] = r[0];
                }
            }
            const int bad_any = __syncthreads_or(bad);
            if (warp == 0) {
                double* pt = sp.part + (((size_t)s * sp.T_sim + j) * 5) * V;
                for (int e = lane; e < 4 * V; e += 32) {
                    const int km = e / V, v = e - km * V;
                    if (km == 3 || sample) {
                        double a = 0.0;
                        for (int w = 0; w < NW; ++w) a += s_red[w][km][v];
                        pt[km * V + v] = a;
                    }
                }
                if (lane == 0) pt[4 * V] = bad_any ? 1.0 : 0.0;
            }
            __syncthreads();       // stage st and s_red free for reuse
            st ^= 1;
            t = tn;
        }

        // ---- grid barrier + active count ------------------------------------------------------
        if (tid == 0) {
            int mine = 0;
            for (int slot = 0; slot < ns; ++slot) {
                const int s = s_lo + slot;
                if ((long long)s * sp.T_sim >= t_lo && s_coef[slot].active) ++mine;   // owner CTA counts
            }
            if (mine) atomicAdd(&sp.active[n % 3], mine);
        }
        grid_sync(sp.bar, G, gen);
        const int still = *((volatile int*)&sp.active[n % 3]);
        if (blockIdx.x == 0 && tid == 0) sp.active[(n + 2) % 3] = 0;      // read by all before barrier n
        if (still == 0) break;

        // ---- scalar phase: one warp per simulation slot ----------------------------------------
        if (warp < ns && s_coef[warp].active) {
            const int slot = warp, s = s_lo + slot;
            const bool owner = (long long)s * sp.T_sim >= t_lo;
            SimPrimal W = s_sp[slot];
            SimTan T = s_st[slot][lane];
            const bool sample = s_coef[slot].sample != 0;
            double tot[4] = {0.0, 0.0, 0.0, 0.0}, totd[4] = {0.0, 0.0, 0.0, 0.0};
            double badf = 0.0;
            const double* pt = sp.part + ((size_t)s * sp.T_sim * 5) * V;
            for (int jt = 0; jt < sp.T_sim; ++jt) {
                const double* q = pt + (size_t)jt * 5 * V;
#pragma unroll
                for (int km = 0; km < 4; ++km) {
                    if (km == 3 || sample) {
                        tot[km] += q[km * V];
                        if (pl >= 0) totd[km] += q[km * V + 1 + pl];
                    }
                }
                badf += q[4 * V];
            }
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
            __syncwarp();
            if (lane == 0) s_sp[slot] = W;
            s_st[slot][lane] = T;
        }
        __syncthreads();
        src_sel ^= 1;
        ++n;
    }

    // ---- epilogue: per-simulation status / loss / gradient (owner CTA) --------------------------
    if (warp < ns) {
        const int slot = warp, s = s_lo + slot;
        if ((long long)s * sp.T_sim >= t_lo) {
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

// n0 (caller layout [S or 1][N]) -> padded buffer 0; tangent rows 0; per-sim max(n0) bits.
template <int V>
__global__ void k_stream_load(const double* __restrict__ n0, long long n0_stride, int N, int S,
                              double* __restrict__ buf, long long pitch, unsigned long long* nscale_bits) {
    const int s = blockIdx.y;
    double m = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const double v = n0[(size_t)s * n0_stride + i];
        buf[(size_t)s * V * pitch + 2 + i] = v;
#pragma unroll
        for (int p = 1; p < V; ++p) buf[((size_t)s * V + p) * pitch + 2 + i] = 0.0;
        m = fmax(m, v);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(nscale_bits + s, (unsigned long long)__double_as_longlong(m));
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
