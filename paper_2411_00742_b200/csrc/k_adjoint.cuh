// =====================================================================================
//  k_adjoint — NEXT-3: reverse-mode (discrete adjoint) gradient of the RSS loss with
//  respect to every kinetic parameter, with trajectory checkpointing.  This is the regime
//  the paper reaches with jax.grad + checkpointing ("for
//  1000 parameters specifically, jax-AD is 40x faster than jax-ND").  The cost of one
//  gradient is a fixed number of passes over the march, independent of the parameter count.
//
//  Step k of the forward march (the same discrete map as the other kernels; rows a1-a7):
//     G^k   = law(S(c^k, T(t^k)); theta)                       (row a1)
//     C^k, dt^k, landing = time_step(G^k, t^k)                 (row a2, R-7..R-9)
//     n^{k+1} = Phi(n^k; C^k)  (flux form, clip R-17)          (rows a3, a4)
//     c^{k+1} = c^k - rho_c k_v (mu3(n^{k+1}) - mu3p^k),  mu3p^{k+1} = mu3(n^{k+1})
//     t^{k+1} = landing ? t_m : t^k + dt^k
//     loss   += ((c - c^)/rms_c)^2 + ((mu1/mu0 - L^)/rms_L)^2 at samples  (row a7, R-23)
//  theta enters ONLY through the scalar G^k, so
//     dL/dtheta_j = sum_k lambda_G^k dG^k/dtheta_j
//  with lambda_G^k the adjoint of G^k.  The vector part is the transposed flux update
//     Lambda_f = lambda_f - lambda_{f-1}   (face f between bins f-1 and f)
//     lambda^k_j = lambda^{k+1}_j + sum_{faces f touching j} Lambda_f dF_f/dn_j
//     lambda_C^k = sum_f Lambda_f dF_f/dC,     dF/dC = n_up + beta psi  (kapdot = beta Cdot)
//  using the same face partials as the tangent lanes (k_resident.cuh: w_lo, w_mid, w_hi, g).
//  The scalar chain (c, t, G) -> (C, t') is linearised once in the forward pass with 3 lanes of
//  dual numbers (seeds dc, dt, dG) and stored in a per-step trace; the reverse pass only needs
//  that trace, the face partials at n^k and the clip marks of n^{k+1}.
//
//  Checkpointing: the forward pass stores n^k every Kseg steps; the reverse pass walks the
//  segments backwards, re-marches each one from its checkpoint (kinetics not re-evaluated: C^k
//  comes from the trace, so the recomputed states are bitwise the forward ones) into a segment
//  buffer, then runs the adjoint steps of the segment.  Memory per simulation: trace
//  16 doubles x steps, checkpoints N x steps/Kseg, segment N x (Kseg + 1).
//
//  Clip marks: a bin zeroed by the round-off clip (R-17) is stored as -0.0 (an exact zero for
//  all arithmetic); every other zero is canonicalised to +0.0.  The adjoint of a clipped bin is
//  0, exactly as the tangent lanes zero a clipped bin's tangents.
//
//  One CTA per simulation, K bins per thread (contiguous), state and adjoint in shared memory
//  double-buffered by step parity; warp 0 runs the scalar phases (two barriers per step).
// =====================================================================================
#pragma once
#include <cooperative_groups.h>
#include <type_traits>

#include "pbe_device.cuh"

namespace pbe {

#if PBE_TIMING
__device__ unsigned long long g_adj_cycles[16];    // forward, recompute, backward-vector, backward-scalar
#define PBE_ATS(v) long long v = clock64()
#define PBE_ATA(i, a, b) t_acc[i] += (unsigned long long)((b) - (a))
#else
#define PBE_ATS(v)
#define PBE_ATA(i, a, b)
#endif

constexpr int ADJ_TR = 16;        // doubles per step in the scalar trace
// physical length (doubles, even) of one padded state row of an NT-thread CTA with K bins per
// thread: logical index x = bin + 2 in [0, NT K + 4) stored at x + x / K (host and device)
__host__ __device__ constexpr int adj_row(int NT, int K) { return ((NT * K + 4) + (NT * K + 4) / K + 2) & ~1; }
enum AdjTrace {
    TR_C = 0, TR_KAP2, TR_BETA2,          // Courant number, 2 kap, 2 beta (kapdot = beta Cdot)
    TR_CC, TR_CT, TR_CG,                  // dC/dc, dC/dt (total, through G), dC/dG
    TR_TC, TR_TT, TR_TG,                  // dt'/dc, dt'/dt, dt'/dG   (t' = t^{k+1})
    TR_S, TR_T,                           // supersaturation and temperature of the step
    TR_LC, TR_L0, TR_L1,                  // d loss / d(c, mu0, mu1)(n^{k+1}) if step k lands on a sample
    TR_LG                                 // lambda_G^k, the adjoint of G^k (written by the reverse pass)
};

struct AdjParams {
    KParams kp;           // 1D, P = 0, sample mode, target set
    double* ck;           // [S][n_ck][N] checkpoints n^{j Kseg}
    double* seg;          // [S][Kseg + 1][N] states n^{k0} .. n^{k1} of the current segment
    double* tr;           // [S][max_steps][ADJ_TR]
    double* gtheta;       // [S][n_params]
    long long n_ck;       // checkpoint slots per simulation
    int Kseg;
    int seg_smem;         // 1: the segment states live in shared memory (seg unused)
    int traj;             // 1: every state n^0..n^K is kept (ck holds K + 1 rows): no re-march, the
                          //    reverse pass prefetches n^{k-1} with cp.async while it works on k
};

// 16-byte global -> shared copy that bypasses registers (LDGSTS), and its completion wait
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// cluster mode: remote shared-memory stores that complete bytes on the RECEIVER's mbarrier
// (st.async), so each CTA waits only for the data it needs instead of a cluster-wide barrier
__device__ __forceinline__ unsigned adj_mapa(const void* p, int rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void adj_st_async2(unsigned raddr, double a, double b, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                 ::"r"(raddr), "d"(a), "d"(b), "r"(rbar) : "memory");
}
__device__ __forceinline__ void adj_st_async1(unsigned raddr, double a, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];"
                 ::"r"(raddr), "d"(a), "r"(rbar) : "memory");
}
__device__ __forceinline__ void adj_mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void adj_mbar_arrive(unsigned long long* bar, unsigned tx) {
    if (tx)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(tx) : "memory");
    else
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void adj_mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(a), "r"(parity) : "memory");
}

// dG/dtheta_j at (S, T) in closed form (the parameters enter the laws of growth_rate as
// below; dpow(x, y) = exp(y log x) there).
__device__ __forceinline__ double dG_dtheta(const KParams& kp, const double* __restrict__ th, double S, double T, int j) {
    if (kp.law == LAW_CONST) return j == 0 ? 1.0 : 0.0;
    if (kp.law == LAW_ARRH) {
        const double Tk = T + 273.15;
        if (S > 1.0) {
            if (j > 2) return 0.0;
            const double lx = log(S - 1.0);
            const double EP = exp(-th[1] / Tk) * exp(th[2] * lx);
            return j == 0 ? EP : (j == 1 ? -th[0] * EP / Tk : th[0] * EP * lx);
        }
        if (S < 1.0 && kp.n_params >= 6) {
            if (j < 3) return 0.0;
            const double lx = log(1.0 - S);
            const double EP = exp(-th[4] / Tk) * exp(th[5] * lx);
            return j == 3 ? -EP : (j == 4 ? th[3] * EP / Tk : -th[3] * EP * lx);
        }
        return 0.0;
    }
    if (S > 1.0) return pow(S - 1.0, (double)(j + 1));           // POLY: G = sum_j a_j (S-1)^(j+1)
    return 0.0;
}

// NTB: the CTA width bound (256; 512 with K = 4 is an A/B variant).
// CL: a thread-block cluster of CS CTAs per simulation (trajectory mode only), CTA r holding bins
// [r NT K, (r + 1) NT K): edge bins and edge adjoints are pushed into the neighbours' ghost cells
// over DSMEM, warp/CTA partial sums are added across the cluster in a fixed order by every CTA
// (so every CTA runs the identical scalar chain and no broadcast is needed), the step barrier
// after the partials is cluster.sync(), and rank 0 alone writes the trace and the records.
// NEXT-3 at N = 2000 on 9 experiments: 16 CTAs each = 144 SMs instead of 9.
template <int K, int NTB = 256, bool CL = false>
__global__ void __launch_bounds__(NTB) k_adjoint(const AdjParams ap) {
    namespace cg = cooperative_groups;
    const KParams& kp = ap.kp;
#if PBE_TIMING
    unsigned long long t_acc[16] = {};
#endif
    const int CS = CL ? (int)cg::this_cluster().num_blocks() : 1;
    const int rank = CL ? (int)cg::this_cluster().block_rank() : 0;
    const int s = blockIdx.x / CS, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NT = blockDim.x, NW = NT >> 5;
    const int N = kp.N, NP = adj_row(NT, K);                 // physical row length (doubles)
    const int NB = NT * K, b0 = rank * NB;                   // this CTA's bins [b0, b0 + NB)
    const int i0 = b0 + tid * K;                             // global index of the thread's first bin
    auto cl_sync = [&]() __attribute__((always_inline)) {
        if constexpr (CL) cg::this_cluster().sync(); else __syncthreads();
    };
    // bank-conflict-free rows: logical index x = bin + 2 lives at x + x / K, so thread t's window
    // x = K t + j (j = 0..K+3, compile-time) sits at (K + 1) t + j + j / K -- an odd stride across
    // the warp (K even) instead of K: 2 wavefronts per 8-byte LDS/STS instead of K (ncu: 11.7)
    const int tb = (K + 1) * tid;
#define PX(j) (tb + (j) + (j) / K)
    const int lim = kp.limiter;
    const double rho = kp.rho_kv;
    const int Kseg = ap.Kseg;
    double* trs = ap.tr + (size_t)s * kp.max_steps * ADJ_TR;
    const int CP = ap.traj ? (N + 1) & ~1 : N;          // checkpoint row pitch (16-B rows for cp.async)
    double* cks = ap.ck + (size_t)s * ap.n_ck * CP;
    extern __shared__ __align__(16) double sm[];
    double* nb = sm;                      // [2][NP] states, bin i at px(i + 2)
    double* lb = sm + 2 * NP;             // [2][NP] adjoints (same layout)
    // segment states n^{k0..k1}: shared memory when they fit (host decides), else global;
    // trajectory mode: a ring of 3 states (n^{k+1}, n^k and n^{k-1} in flight); rows in the
    // padded layout of nb (the global segment buffer too: it is this kernel's scratch)
    double* sgs = (ap.seg_smem || ap.traj) ? sm + 4 * NP : ap.seg + (size_t)s * (Kseg + 1) * NP;
    // the segment's trace rows, staged in shared memory at every segment start
    double* s_trs = sm + 4 * NP + (ap.traj ? (size_t)3 * NP : (ap.seg_smem ? (size_t)(Kseg + 1) * NP : 0));
    // trajectory mode: state k (contiguous in HBM) -> ring slot k % 3 (padded), 8-byte cp.async
    // (local index x = bin - b0 + 2, ghost/halo bins included)
    auto fetch_state = [&](long long k) {
        const double* src = cks + (size_t)k * CP;
        double* dst = sgs + (size_t)(k % 3) * NP;
        for (int x = tid; x < NB + 4; x += NT) {
            const int i = b0 - 2 + x;
            if (i >= 0 && i < N) cp_async8(dst + x + x / K, src + i);
        }
    };
    // warp partials, double-buffered by step parity: [par][m][rank NW + warp] -- in CL mode every
    // warp pushes its partials into EVERY CTA of the cluster (remote stores do not stall), so the
    // reads after the exchange are local; m: mu0..mu3 (or lambda_C, 0, 0, 0), clip-failure flag
    __shared__ __align__(16) double s_red[2][5][32];
    __shared__ unsigned long long s_mbar[2];       // CL: one mbarrier per parity (partials + halos)
    unsigned mph = 0;                              // CL: phase bit of s_mbar[0], s_mbar[1]
    __shared__ double s_sc[12];
    __shared__ double s_pp[32][2];                 // long polynomial: per-warp (G, dG/dx) partials
    __shared__ double s_cm[2];                     // warp 0's c, mu3p (read by every warp)
    __shared__ int s_go, s_sample, s_ok;
    __shared__ long long s_nsteps;
    enum { SC_C = 0, SC_KAP2, SC_BETA2, SC_LM, SC_L0, SC_L1, SC_LG, SC_S, SC_T, SC_CLIP };

    for (int j = tid; j < 4 * NP; j += NT) sm[j] = 0.0;
    for (int j = tid; j < 2 * 5 * 32; j += NT) (&s_red[0][0][0])[j] = 0.0;
    if (CL && tid == 0) {
        adj_mbar_init(&s_mbar[0], NW);             // every local warp arrives once per phase
        adj_mbar_init(&s_mbar[1], NW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl_sync();                                     // CL: the barriers exist before any remote store
    double lmax = 0.0;
    {
        const double* n0 = kp.n0 + (size_t)s * kp.n0_stride;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int i = i0 + k;
            if (i < N) { const double v = n0[i]; nb[PX(k + 2)] = v; lmax = fmax(lmax, v); }
        }
        if (CL && tid < 4) {                       // halo bins b0-2, b0-1, b0+NB, b0+NB+1
            const int x = tid < 2 ? tid : NB + tid;
            const int i = b0 - 2 + x;
            if (i >= 0 && i < N) nb[x + x / K] = n0[i];
        }
    }
    // cluster neighbours' shared memory (DSMEM): the same offset in CTA rank r
    auto remote = [&](auto* p, int r) -> decltype(p) {
        if constexpr (CL) return cg::this_cluster().map_shared_rank(p, r);
        else return p;
    };
    // push this CTA's two edge values of row `row` into the neighbours' ghost cells (CL only),
    // completing 16 bytes on the neighbour's mbarrier of parity par (two 8-byte st.async: the
    // padded ghost pair is not always 16-byte aligned)
    auto push_halo = [&](double* row, int par) __attribute__((always_inline)) {
        if constexpr (CL) {
            if (tid == 0 && rank > 0) {            // local bins 0, 1 -> left neighbour's x = NB+2, NB+3
                const unsigned rb = adj_mapa(&s_mbar[par], rank - 1);
                adj_st_async1(adj_mapa(row + (NB + 2) + (NB + 2) / K, rank - 1), row[2 + 2 / K], rb);
                adj_st_async1(adj_mapa(row + (NB + 3) + (NB + 3) / K, rank - 1), row[3 + 3 / K], rb);
            }
            if (tid == NT - 1 && rank < CS - 1) {  // local bins NB-2, NB-1 -> right neighbour's x = 0, 1
                const unsigned rb = adj_mapa(&s_mbar[par], rank + 1);
                adj_st_async1(adj_mapa(row, rank + 1), row[NB + NB / K], rb);
                adj_st_async1(adj_mapa(row + 1, rank + 1), row[(NB + 1) + (NB + 1) / K], rb);
            }
        }
    };
    // this warp's partials a[0..4] (identical in every lane after a butterfly) -> slot
    // rank NW + warp of every CTA (lane r stores to rank r; remote ones with st.async)
    auto put_partials = [&](int par, const double* a) __attribute__((always_inline)) {
        if constexpr (CL) {
            const int e = rank * NW + warp;
            if (lane == rank) {
#pragma unroll
                for (int m = 0; m < 5; ++m) s_red[par][m][e] = a[m];
            } else if (lane < CS) {
                const unsigned rb = adj_mapa(&s_mbar[par], lane);
#pragma unroll
                for (int m = 0; m < 5; ++m) adj_st_async1(adj_mapa(&s_red[par][m][e], lane), a[m], rb);
            }
        } else if (lane == 0) {
#pragma unroll
            for (int m = 0; m < 5; ++m) s_red[par][m][warp] = a[m];
        }
    };
    // the exchange point of a step: the partials of parity par (and, with halo, the neighbours'
    // edge values) of every CTA are in place.  CL: each warp arrives on the local mbarrier (warp 0
    // also posts the expected remote bytes) and every thread waits for the phase; else a CTA barrier.
    auto exchange = [&](int par, bool halo) __attribute__((always_inline)) {
        if constexpr (CL) {
            __syncwarp();
            if (lane == 0) {
                const unsigned tx = (unsigned)((CS - 1) * NW * 40) +
                                    (halo ? 16u * ((rank > 0) + (rank < CS - 1)) : 0u);
                adj_mbar_arrive(&s_mbar[par], warp == 0 ? tx : 0u);
            }
            adj_mbar_wait(&s_mbar[par], (mph >> par) & 1u);
            mph ^= 1u << par;
        } else {
            __syncthreads();
        }
    };
    // block sums of mu0..mu3 of nb[q] (all four if `all`, else mu3) -> s_red[par] (warp partials)
    auto moment_partials = [&](int q, bool all, int par, const double* slot0 = nullptr, bool bad = false) {
        double a[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        const double* x = nb + q * NP;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int i = i0 + k;
            if (i < N) {
                const double L = fma((double)i, kp.dL, kp.L_lo + 0.5 * kp.dL);
                const double w0 = kp.dL * x[PX(k + 2)], w1 = w0 * L, w2 = w1 * L;
                a[3] = fma(w2, L, a[3]);
                if (all) { a[0] += w0; a[1] += w1; a[2] += w2; }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
            for (int m = 0; m < 4; ++m) a[m] += __shfl_xor_sync(0xffffffffu, a[m], off);
        if (slot0) a[0] = *slot0;
        a[4] = __any_sync(0xffffffffu, bad) ? 1.0 : 0.0;
        put_partials(par, a);
    };
    // CL: the 32 partial slots of a row (unused slots stay 0) summed (or max-ed) by a fixed
    // pairwise tree in registers; every lane loads the row itself (16-byte broadcast loads), so
    // no shuffles: identical in every lane and every CTA
    auto tree32 = [&](const double* row, bool mx) __attribute__((always_inline)) -> double {
        double v[16];
        const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const double2 p2 = r2[i];
            v[i] = mx ? fmax(p2.x, p2.y) : p2.x + p2.y;
        }
#pragma unroll
        for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
            for (int i = 0; i < w; ++i) v[i] = mx ? fmax(v[i], v[i + w]) : v[i] + v[i + w];
        return v[0];
    };
    // total (or max) of slot m of the partials s_red[par] over the CTA (warp order) -- over the
    // cluster in CL mode.  Whole warps, after the exchange that follows the partials.
    auto red_total = [&](int m, int par, bool mx) -> double {
        if constexpr (!CL) {
            double t = 0.0;
            for (int w = 0; w < NW; ++w) t = mx ? fmax(t, s_red[par][m][w]) : t + s_red[par][m][w];
            return t;
        } else {
            return tree32(&s_red[par][m][0], mx);
        }
    };
    // sums of slots m1 and m2
    auto red_total2 = [&](int m1, int m2, int par, double& t1, double& t2) __attribute__((always_inline)) {
        if constexpr (!CL) {
            t1 = 0.0; t2 = 0.0;
            for (int w = 0; w < NW; ++w) { t1 += s_red[par][m1][w]; t2 += s_red[par][m2][w]; }
        } else {
            t1 = tree32(&s_red[par][m1][0], false);
            t2 = tree32(&s_red[par][m2][0], false);
        }
    };
    int rpar = 0;                                   // parity of the partials being read
    auto block_total = [&](int m) -> double { return red_total(m, rpar, false); };
    // forward update nb[q] -> nb[q^1] (eq-highRes_growth, flux form; clip marks as -0.0)
    // limited half slope of kind LIMT (0 upwind, 1 van Leer branch-free, 2 minmod/superbee/MC):
    // the sweep direction and the limiter are resolved once per step, not per face (a branch per
    // face makes every face its own basic block and serialises their latency chains)
    auto half_slope = [&](auto limc, double a, double b, double& h, double& qa, double& qb)
        __attribute__((always_inline)) {
        constexpr int LIMT = decltype(limc)::value;
        h = qa = qb = 0.0;
        if (LIMT == 1) psi_half_d_bf(a, b, h, qa, qb);
        else if (LIMT == 2) psi_half_other(lim, a, b, h, qa, qb);
    };
    auto with_kind = [&](double C, auto&& body) __attribute__((always_inline)) {
        const int lk = lim == LIM_VANLEER ? 1 : (lim == LIM_UPWIND ? 0 : 2);
        if (C >= 0.0) {
            if (lk == 1) return body(std::false_type{}, std::integral_constant<int, 1>{});
            if (lk == 0) return body(std::false_type{}, std::integral_constant<int, 0>{});
            return body(std::false_type{}, std::integral_constant<int, 2>{});
        }
        if (lk == 1) return body(std::true_type{}, std::integral_constant<int, 1>{});
        if (lk == 0) return body(std::true_type{}, std::integral_constant<int, 0>{});
        return body(std::true_type{}, std::integral_constant<int, 2>{});
    };
    auto update = [&](int q, double C, double kap2, double clip) -> bool {
        const double* in = nb + q * NP;                            // in[PX(j)] = bin i0 - 2 + j
        double* out = nb + (q ^ 1) * NP;
        double w[K + 4], F[K + 1];
#pragma unroll
        for (int j = 0; j < K + 4; ++j) w[j] = in[PX(j)];
        with_kind(C, [&](auto negc, auto limc) {
            constexpr bool NEG = decltype(negc)::value;
#pragma unroll
            for (int f = 0; f <= K; ++f) {                         // face between bins i0+f-1 | i0+f
                double h, qa, qb;
                if (!NEG) {
                    half_slope(limc, w[f + 1] - w[f], w[f + 2] - w[f + 1], h, qa, qb);
                    F[f] = fma(C, w[f + 1], kap2 * h);
                } else {
                    half_slope(limc, w[f + 3] - w[f + 2], w[f + 2] - w[f + 1], h, qa, qb);
                    F[f] = fma(C, w[f + 2], kap2 * h);
                }
            }
        });
        bool bad = false;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (i0 + k < N) {
                double v = (w[k + 2] - (F[k + 1] - F[k])) + 0.0;     // +0.0: canonical zero
                if (v < 0.0) { if (v >= -clip) v = -0.0; else bad = true; }   // R-17 (mark)
                out[PX(k + 2)] = v;
            }
        }
        return bad;
    };

#pragma unroll
    for (int off = 16; off > 0; off >>= 1) lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, off));
    moment_partials(0, false, 0, &lmax);           // mu0 slot reused for max(n0) (mu3 in slot 3)
    exchange(0, false);

    // ---- warp-0 scalar state of the forward pass ----------------------------------------------
    const KinLoader KL{kp.theta + (size_t)s * kp.n_params, kp.sol, kp.seed, -1, kp.n_params, kp.n_params + kp.n_sol};
    const double* kT = kp.knot_T + (size_t)s * kp.knotT_stride;
    const double* tgt = kp.target + (size_t)s * kp.M * 2;
    double c = kp.c0[s], t = 0.0, mu3p = 0.0, loss = 0.0, rms_c = 1.0, rms_L = 1.0, dt = 0.0;
    long long nstep = 0;
    int m = 0, status = ST_OK;
    bool landing = false;
    // kinetics of the step from (c, t) + its linearisation (lane 0: dc, lane 1: dt, lane 2: dG)
    const KinCache KC = kin_cache(kp, KL, kT);           // constant: theta, solubility, knots
    double tn_c = kp.t_samples[0];                         // t_samples[m], read once per sample
    // long polynomial at constant T (NEXT-3's 1000-coefficient regime): the terms are split over
    // EVERY thread of the CTA (the other warps would idle at the barrier while warp 0 runs the
    // kinetics): thread t sums terms [t m, t m + m) by Horner with d/dx, scaled by x^(t m + 1);
    // warp butterflies, then warp 0 adds the warp partials in warp order.  Step 0 uses the
    // warp-cooperative form.
    const bool poly_blk = kp.law == LAW_POLY && kp.n_params > MAXTH && KC.const_T;
    bool use_blk = false;                                  // warp 0: the partials of this step are ready
    // coefficients a_j of this thread's terms [tid PM, tid PM + PM) kept in registers for the
    // march when n_params <= NT PM (an L1 miss per term per step otherwise: 4.6k cycles/step
    // at 64 threads x 16 terms)
    constexpr int PM = (1024 + NTB - 1) / NTB;
    const bool poly_reg = poly_blk && kp.n_params <= NT * PM;
    double pc[PM];
#pragma unroll
    for (int i = 0; i < PM; ++i) {
        const int j = tid * PM + i;
        pc[i] = poly_reg && j < kp.n_params ? kp.theta[(size_t)s * kp.n_params + j] : 0.0;
    }
    auto poly_partials = [&](double Sv) {                  // every thread, after the step's barrier
        double tt = 0.0, dtt = 0.0;
        if (Sv > 1.0 && poly_reg) {
            const double x = Sv - 1.0;
            const int j0 = tid * PM;
            double qv = 0.0, dq = 0.0;
#pragma unroll
            for (int i = PM - 1; i >= 0; --i) {
                dq = fma(dq, x, qv);
                qv = fma(qv, x, pc[i]);
            }
            // x^(tid PM) = (x^PM)^tid: the PM-power by squarings (PM a power of two), then the
            // thread-dependent part -- the same products as ipow(x, tid PM), fewer loop trips
            double xl;
            if constexpr ((PM & (PM - 1)) == 0) {
                double xp = x;
#pragma unroll
                for (int m = 1; m < PM; m <<= 1) xp = xp * xp;
                xl = tid > 0 ? ipow(xp, tid) : 1.0;
            } else {
                xl = ipow(x, j0);
            }
            tt = xl * x * qv;
            dtt = xl * fma((double)(j0 + 1), qv, x * dq);
        } else if (Sv > 1.0) {
            const double x = Sv - 1.0;
            const int mm = (kp.n_params + NT - 1) / NT, j0 = tid * mm;
            const double* a = kp.theta + (size_t)s * kp.n_params;
            double qv = 0.0, dq = 0.0;
            for (int i = mm - 1; i >= 0; --i) {
                const int j = j0 + i;
                const double aj = j < kp.n_params ? __ldg(a + j) : 0.0;
                dq = fma(dq, x, qv);
                qv = fma(qv, x, aj);
            }
            const double xl = ipow(x, j0);
            tt = xl * x * qv;
            dtt = xl * fma((double)(j0 + 1), qv, x * dq);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            tt += __shfl_xor_sync(0xffffffffu, tt, off);
            dtt += __shfl_xor_sync(0xffffffffu, dtt, off);
        }
        if (lane == 0) { s_pp[warp][0] = tt; s_pp[warp][1] = dtt; }
    };
    auto kinetics = [&](long long k) -> bool {
        const D1 cD = mk(c, lane == 0 ? 1.0 : 0.0), tD = mk(t, lane == 1 ? 1.0 : 0.0);
        D1 T;
        const D1 S = supersaturation(kp, KL, kT, KC, tD, cD, T);
        D1 G;
        if (use_blk) {                                     // block partials of this S (same value)
            double tt = 0.0, dtt = 0.0;
            for (int w = 0; w < NW; ++w) { tt += s_pp[w][0]; dtt += s_pp[w][1]; }
            G = S.v > 1.0 ? D1{tt, dtt * S.d} : mk(0.0);
        } else {
            G = (kp.law == LAW_POLY && kp.n_params > MAXTH)
                    ? poly_long_warp(kp.theta + (size_t)s * kp.n_params, kp.n_params, S)   // warp-cooperative
                    : growth_rate(kp, KL, S, T);
        }
        if (lane == 2) G = mk(G.v, 1.0);
        const double tn = tn_c;
        const StepScalars sc = time_step(kp, G, tD, tn, false);
        if (sc.err != ST_OK) { status = sc.err; return false; }
        const D1 tp = sc.landing ? mk(tn) : tD + sc.dt;
        const double Cv = sc.C.v;
        const double beta = Cv > 0.0 ? 0.5 * (1.0 - 2.0 * Cv) : (Cv < 0.0 ? -0.5 * (1.0 + 2.0 * Cv) : 0.0);
        const double dC0 = __shfl_sync(0xffffffffu, sc.C.d, 0), dC1 = __shfl_sync(0xffffffffu, sc.C.d, 1);
        const double dC2 = __shfl_sync(0xffffffffu, sc.C.d, 2);
        const double dT0 = __shfl_sync(0xffffffffu, tp.d, 0), dT1 = __shfl_sync(0xffffffffu, tp.d, 1);
        const double dT2 = __shfl_sync(0xffffffffu, tp.d, 2);
        if (lane == 0 && rank == 0) {
            double* r = trs + (size_t)k * ADJ_TR;
            r[TR_C] = Cv; r[TR_KAP2] = 2.0 * sc.kap.v; r[TR_BETA2] = 2.0 * beta;
            r[TR_CC] = dC0; r[TR_CT] = dC1; r[TR_CG] = dC2;
            r[TR_TC] = dT0; r[TR_TT] = dT1; r[TR_TG] = dT2;
            r[TR_S] = S.v; r[TR_T] = T.v;
            r[TR_LC] = 0.0; r[TR_L0] = 0.0; r[TR_L1] = 0.0;
        }
        if (lane == 0) { s_sc[SC_C] = Cv; s_sc[SC_KAP2] = 2.0 * sc.kap.v; }
        dt = sc.dt.v;
        landing = sc.landing;
        return true;
    };
    if (warp == 0) {
        const double nmax = red_total(0, 0, true);
        mu3p = red_total(3, 0, false);
        double sc2 = 0.0, sl2 = 0.0;
        for (int j = lane; j < kp.M; j += 32) { sc2 += tgt[2 * j] * tgt[2 * j]; sl2 += tgt[2 * j + 1] * tgt[2 * j + 1]; }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            sc2 += __shfl_xor_sync(0xffffffffu, sc2, off);
            sl2 += __shfl_xor_sync(0xffffffffu, sl2, off);
        }
        rms_c = sqrt(sc2 / kp.M); rms_L = sqrt(sl2 / kp.M);
        bool go = kp.max_steps > 0;
        if (!go) status = ST_MAXSTEPS;
        if (go) go = kinetics(0);
        if (lane == 0) {
            s_go = go;
            s_sample = go && landing;
            s_sc[SC_CLIP] = 1e-12 * nmax;
            s_cm[0] = c; s_cm[1] = mu3p;
        }
    }
    __syncthreads();
    const double clip = s_sc[SC_CLIP];

    // ---- forward pass: checkpoints + trace -------------------------------------------------------
    int q = 0;
    long long k = 0;
    PBE_ATS(tf0);
    while (s_go) {
        if (ap.traj || k % Kseg == 0) {
            double* ckp = cks + (size_t)(ap.traj ? k : k / Kseg) * CP;
#pragma unroll
            for (int j = 0; j < K; ++j) if (i0 + j < N) ckp[i0 + j] = nb[q * NP + PX(j + 2)];
        }
        PBE_ATS(tq0);
        const bool bad = update(q, s_sc[SC_C], s_sc[SC_KAP2], clip);
        const int par = (int)((k + 1) & 1);
        push_halo(nb + (q ^ 1) * NP, par);
        moment_partials(q ^ 1, s_sample != 0, par, nullptr, bad);
        PBE_ATS(tq1);
        PBE_ATA(5, tq0, tq1);
        exchange(par, true);
        rpar = par;
        PBE_ATS(tqx);
        PBE_ATA(1, tq1, tqx);
        // mu3(n^{k+1}) and the clip-failure flag in one reduction, by every warp (poly) or warp 0
        double mu3_k = 0.0, bad_k = 0.0;
        if (poly_blk || warp == 0) red_total2(3, 4, rpar, mu3_k, bad_k);
        PBE_ATS(tp0);
        PBE_ATA(14, tqx, tp0);
        if (poly_blk) {
            // every warp: c^{k+1} and S of the next step exactly as warp 0 forms them below
            const double cn = __dsub_rn(s_cm[0], __dmul_rn(rho, __dsub_rn(mu3_k, s_cm[1])));
            poly_partials(__dmul_rn(cn, KC.ics.v));
            PBE_ATS(tp1);
            PBE_ATA(15, tp0, tp1);
            __syncthreads();
            use_blk = true;
        }
        PBE_ATS(tq2);
        PBE_ATA(6, tq1, tq2);
        if (warp == 0) {
            const bool sample = s_sample != 0;
            const double mu3 = mu3_k;
            const double cn = __dsub_rn(c, __dmul_rn(rho, __dsub_rn(mu3, mu3p)));   // eq-discrete_mass_balance
            bool go = true;
            if (bad_k > 0.0) { status = ST_NEG; go = false; }
            else if (cn < 0.0) { status = ST_INFEAS; go = false; }
            else {
                c = cn; mu3p = mu3;
                t = landing ? kp.t_samples[m] : t + dt;
                ++nstep;
                if (sample) {
                    const double mu0 = block_total(0), mu1 = block_total(1), mu2 = block_total(2);
                    if (lane == 0) {
                        const double Lb = mu1 / mu0;
                        const double rc = (c - tgt[2 * m]) / rms_c, rL = (Lb - tgt[2 * m + 1]) / rms_L;
                        loss += rc * rc + rL * rL;
                        if (rank == 0) {
                            double* r = kp.rec + ((size_t)s * kp.M + m) * 6;
                            r[0] = t; r[1] = c; r[2] = mu0; r[3] = mu1; r[4] = mu2; r[5] = mu3;
                            const double gL = 2.0 * rL / rms_L;             // d loss / d Lbar
                            double* tr = trs + (size_t)k * ADJ_TR;
                            tr[TR_LC] = 2.0 * rc / rms_c;
                            tr[TR_L0] = -gL * mu1 / (mu0 * mu0);
                            tr[TR_L1] = gL / mu0;
                        }
                    }
                }
                if (landing) { ++m; if (m < kp.M) tn_c = kp.t_samples[m]; }
                PBE_ATS(tk0);
                PBE_ATA(12, tq2, tk0);
                if (m >= kp.M) go = false;
                else if (nstep >= kp.max_steps) { status = ST_MAXSTEPS; go = false; }
                else go = kinetics(k + 1);
                PBE_ATS(tk1);
                PBE_ATA(13, tk0, tk1);
            }
            if (lane == 0) { s_go = go; s_sample = go && landing; s_nsteps = nstep; s_cm[0] = c; s_cm[1] = mu3p; }
        }
        PBE_ATS(tq3);
        PBE_ATA(7, tq2, tq3);
        __syncthreads();
        q ^= 1;
        ++k;
    }
    if (ap.traj) {                                         // the final state n^K closes the trajectory
        double* ckp = cks + (size_t)k * CP;
#pragma unroll
        for (int j = 0; j < K; ++j) if (i0 + j < N) ckp[i0 + j] = nb[q * NP + PX(j + 2)];
    }
    PBE_ATS(tf1);
    PBE_ATA(0, tf0, tf1);
    if (warp == 0 && lane == 0) {
        if (rank == 0) {
            kp.status[s] = status;
            kp.steps[s] = nstep;
            kp.loss[s] = status == ST_OK ? loss : __longlong_as_double(0x7ff8000000000000ll);
        }
        s_ok = status == ST_OK;
    }
    if constexpr (CL) __threadfence();                     // trace, records, trajectory rows -> cluster
    cl_sync();                                             // (CL: no CTA leaves while others read its smem)
    if (!s_ok) {
        if (rank == 0)
            for (int j = tid; j < kp.n_params; j += NT) ap.gtheta[(size_t)s * kp.n_params + j] = __longlong_as_double(0x7ff8000000000000ll);
        return;
    }
    const long long Ktot = s_nsteps;

    // ---- reverse pass ---------------------------------------------------------------------------
    // dL/dtheta_j = sum_k lambda_G^k dG^k/dtheta_j is left to k_adjoint_theta (the whole GPU, after
    // this kernel): the reverse pass only records lambda_G^k in the trace
    // warp-0 adjoint scalars: of c^{k+1} (before the sample term of step k), t^{k+1}, mu3p^{k+1}
    double lam_c = 0.0, lam_t = 0.0, lam_mu = 0.0;
    long long k0s = 0;                             // first step of the staged trace segment
    auto pre_step = [&](long long kk) {            // warp 0: broadcast what the vector phase of kk needs
        const double* r = s_trs + (size_t)(kk - k0s) * ADJ_TR;
        const double lcp = lam_c + r[TR_LC];
        if (lane == 0) {
            s_sc[SC_LM] = -rho * lcp + lam_mu;     // adjoint of mu3(n^{kk+1})
            s_sc[SC_L0] = r[TR_L0]; s_sc[SC_L1] = r[TR_L1];
            s_sc[SC_C] = r[TR_C]; s_sc[SC_KAP2] = r[TR_KAP2]; s_sc[SC_BETA2] = r[TR_BETA2];
        }
    };
    int ql = 0;                                    // lb[ql] = lambda of n^{k+1} (raw)
    const long long nseg = (Ktot + Kseg - 1) / Kseg;
    if (ap.traj && Ktot > 0) {                             // n^K and n^{K-1} before the first step
        __syncthreads();                                   // the final state's global stores are done
        __threadfence_block();                             // (CL: fenced + cluster-synced above)
        fetch_state(Ktot);
        fetch_state(Ktot - 1);
        cp_async_commit_wait_all();
    }
    for (long long sg = nseg - 1; sg >= 0; --sg) {
        const long long k0 = sg * Kseg, k1 = min(k0 + (long long)Kseg, Ktot);
        // stage the segment's trace rows (read by every step below)
        __syncthreads();                                       // previous segment's readers are done
        for (int e = tid; e < (int)(k1 - k0) * ADJ_TR; e += NT) s_trs[e] = __ldcg(trs + (size_t)k0 * ADJ_TR + e);
        k0s = k0;
        __syncthreads();
        // re-march the segment from its checkpoint (C^k from the trace): states n^{k0..k1}
        PBE_ATS(tr0);
        if (!ap.traj) {
            const double* ckp = cks + (size_t)sg * N;
#pragma unroll
            for (int j = 0; j < K; ++j) if (i0 + j < N) nb[PX(j + 2)] = ckp[i0 + j];
            __syncthreads();
            int qq = 0;
            for (long long kk = k0; kk < k1; ++kk) {
                double* sp = sgs + (size_t)(kk - k0) * NP;
#pragma unroll
                for (int j = 0; j < K; ++j) if (i0 + j < N) sp[PX(j + 2)] = nb[qq * NP + PX(j + 2)];
                const double* r = s_trs + (size_t)(kk - k0) * ADJ_TR;
                update(qq, r[TR_C], r[TR_KAP2], clip);
                __syncthreads();
                qq ^= 1;
            }
            double* sp = sgs + (size_t)(k1 - k0) * NP;
#pragma unroll
            for (int j = 0; j < K; ++j) if (i0 + j < N) sp[PX(j + 2)] = nb[qq * NP + PX(j + 2)];
        }
        if (warp == 0) pre_step(k1 - 1);
        __syncthreads();
        PBE_ATS(tr1);
        PBE_ATA(1, tr0, tr1);
        for (long long kk = k1 - 1; kk >= k0; --kk) {
            PBE_ATS(tb0);
            // ---- vector phase: lambda^{kk+1} (+ mass-balance and sample terms, clip marks) ->
            //      lambda^kk, partial lambda_C -------------------------------------------------
            PBE_ATS(tv0);
            PBE_ATA(8, tb0, tv0);
            const double C = s_sc[SC_C], kap2 = s_sc[SC_KAP2], beta2 = s_sc[SC_BETA2];
            const double lm = s_sc[SC_LM], l0 = s_sc[SC_L0], l1 = s_sc[SC_L1];
            const double* nk = sgs + (size_t)(ap.traj ? kk % 3 : kk - k0) * NP;              // n^kk
            const double* nk1 = ap.traj ? sgs + (size_t)((kk + 1) % 3) * NP : nk + NP;       // n^{kk+1}
            const double* lin = lb + ql * NP;                           // lin[PX(j)] = raw lambda of bin i0-2+j
            double w[K + 4], lam[K + 4];
#pragma unroll
            for (int j = 0; j < K + 4; ++j) {
                const int i = i0 - 2 + j;
                const bool in = i >= 0 && i < N;
                w[j] = in ? nk[PX(j)] : 0.0;
                const double v1 = in ? nk1[PX(j)] : 0.0;
                const bool clipped = in && v1 == 0.0 && signbit(v1);
                double l = lin[PX(j)];
                if (in) {
                    const double L = fma((double)i, kp.dL, kp.L_lo + 0.5 * kp.dL);
                    const double w0 = kp.dL, w1 = w0 * L, w3 = w1 * L * L;
                    l = fma(lm, w3, fma(l1, w1, fma(l0, w0, l)));
                }
                lam[j] = (in && !clipped) ? l : 0.0;
            }
            // prefetch n^{kk-1} into the free ring slot (after this step's window loads, so the
            // copies do not queue in front of them); lands while we work
            if (ap.traj && kk >= 1) { fetch_state(kk - 1); cp_async_commit(); }
            PBE_ATS(tv1);
            PBE_ATA(9, tv0, tv1);
            // face partials (as k_resident's tangent lanes): faces f = i0 - 1 + e, e = 0..K+2
            double Lf[K + 3], whi[K + 3], wmid[K + 3], wlo[K + 3];
            double lamC = 0.0;
            with_kind(C, [&](auto negc, auto limc) {
                constexpr bool NEG = decltype(negc)::value;
#pragma unroll
                for (int e = 0; e < K + 3; ++e) {
                    const int f = i0 - 1 + e;                            // face between bins f-1 | f
                    // window index of bin f: f - (i0 - 2) = e + 1
                    if ((!NEG && e < 1) || (NEG && e > K + 1)) { Lf[e] = 0.0; whi[e] = wmid[e] = wlo[e] = 0.0; continue; }
                    const double a = NEG ? w[e + 2] - w[e + 1] : w[e] - w[e - 1];
                    const double b = w[e + 1] - w[e];
                    const double nup = NEG ? w[e + 1] : w[e];
                    double h, qa, qb;
                    half_slope(limc, a, b, h, qa, qb);
                    const double pak = kap2 * qa, pbk = kap2 * qb;
                    if (!NEG) { whi[e] = pbk; wmid[e] = C + (pak - pbk); wlo[e] = -pak; }
                    else      { whi[e] = pak; wmid[e] = C - (pak - pbk); wlo[e] = -pbk; }
                    Lf[e] = lam[e + 1] - lam[e];                         // lambda_f - lambda_{f-1}
                    // faces [i0, i0+K) of a thread holding real bins, plus the outflow face N for the
                    // thread whose last bin is N-1 (a thread starting at i0 = N owns none: when N % K == 0
                    // it would otherwise count face N a second time)
                    const bool owned = i0 < N && ((f >= i0 && f < i0 + K && f <= N) || (f == N && i0 + K == N));
                    if (owned) lamC = fma(Lf[e], fma(beta2, h, nup), lamC); // dF/dC = n_up + beta psi
                }
            });
            PBE_ATS(tv2);
            PBE_ATA(10, tv1, tv2);
            double* lout = lb + (ql ^ 1) * NP;
#pragma unroll
            for (int kq = 0; kq < K; ++kq) {
                if (i0 + kq >= N) continue;
                const int e = kq + 1;                                    // face index of face j = bin j
                double v = lam[kq + 2];
                if (C >= 0.0) v += Lf[e] * whi[e] + Lf[e + 1] * wmid[e + 1] + Lf[e + 2] * wlo[e + 2];
                else          v += Lf[e + 1] * wlo[e + 1] + Lf[e] * wmid[e] + Lf[e - 1] * whi[e - 1];
                lout[PX(kq + 2)] = v;
            }
            push_halo(lout, (int)(kk & 1));
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) lamC += __shfl_xor_sync(0xffffffffu, lamC, off);
            {
                const double a[5] = {lamC, 0.0, 0.0, 0.0, 0.0};
                put_partials((int)(kk & 1), a);
            }
            PBE_ATS(tv3);
            PBE_ATA(11, tv2, tv3);
            exchange((int)(kk & 1), true);
            rpar = (int)(kk & 1);
            PBE_ATS(tb1);
            PBE_ATA(2, tb0, tb1);
            // ---- scalar phase (warp 0): adjoints of c^kk, t^kk, mu3p^kk; lambda_G^kk ------------
            if (warp == 0) {
                const double* r = s_trs + (size_t)(kk - k0) * ADJ_TR;
                const double LC = block_total(0);
                const double lcp = lam_c + r[TR_LC];
                const double nc = lcp + LC * r[TR_CC] + lam_t * r[TR_TC];
                const double nt = LC * r[TR_CT] + lam_t * r[TR_TT];
                const double lG = LC * r[TR_CG] + lam_t * r[TR_TG];
                lam_mu = rho * lcp;
                lam_c = nc; lam_t = nt;
                if (lane == 0 && rank == 0) trs[(size_t)kk * ADJ_TR + TR_LG] = lG;
                if (kk > k0) pre_step(kk - 1);
            }
            if (ap.traj) asm volatile("cp.async.wait_group 0;" ::: "memory");   // n^{kk-1}: this thread's part
            __syncthreads();
            ql ^= 1;
            PBE_ATS(tb2);
            PBE_ATA(3, tb1, tb2);
        }
        __syncthreads();
    }
    if constexpr (CL) cg::this_cluster().sync();          // no CTA leaves while others read its smem
#if PBE_TIMING
    if (blockIdx.x == 0 && tid == 0) { t_acc[4] = (unsigned long long)Ktot; for (int i = 0; i < 16; ++i) g_adj_cycles[i] = t_acc[i]; }
#endif
}

#undef PX

// dL/dtheta_j = sum_{k < K} lambda_G^k dG/dtheta_j(S^k, T^k) from the trace rows (TR_LG, TR_S,
// TR_T) of every simulation whose march succeeded (failed ones keep the NaN k_adjoint wrote).
// Grid (ceil(n_params / 32), n_sims), 256 threads: lane = parameter j within the block's 32, the
// 8 warps take contiguous step chunks, partials summed in warp order (deterministic).  POLY:
// dG/da_j = (S - 1)^(j+1) for S > 1 (ipow); other laws: dG_dtheta.
__global__ void __launch_bounds__(256) k_adjoint_theta(const AdjParams ap) {
    const KParams& kp = ap.kp;
    const int s = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = blockIdx.x * 32 + lane;
    if (kp.status[s] != ST_OK) return;
    const long long Ktot = kp.steps[s];
    const double* trs = ap.tr + (size_t)s * kp.max_steps * ADJ_TR;
    const double* th = kp.theta + (size_t)s * kp.n_params;
    const long long ch = (Ktot + 7) / 8, ka = warp * ch, kb = min(Ktot, ka + ch);
    double acc = 0.0;
    if (j < kp.n_params) {
        if (kp.law == LAW_POLY) {
            for (long long k = kb - 1; k >= ka; --k) {
                const double* r = trs + (size_t)k * ADJ_TR;
                const double S = __ldg(r + TR_S);
                if (S > 1.0) acc = fma(__ldg(r + TR_LG), ipow(S - 1.0, j + 1), acc);
            }
        } else if (j < 6) {
            for (long long k = kb - 1; k >= ka; --k) {
                const double* r = trs + (size_t)k * ADJ_TR;
                acc = fma(__ldg(r + TR_LG), dG_dtheta(kp, th, __ldg(r + TR_S), __ldg(r + TR_T), j), acc);
            }
        }
    }
    __shared__ double red[8][32];
    red[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && j < kp.n_params) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w][lane];
        ap.gtheta[(size_t)s * kp.n_params + j] = t;
    }
}
}  // namespace pbe
