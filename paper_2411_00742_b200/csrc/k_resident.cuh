// =====================================================================================
//  k_resident — persistent one-CTA-per-simulation march with the distribution (and its
//  P tangent lanes) resident in REGISTERS across all time steps (rows a1-a8).
//
//  Thread t owns bins [t K, t K + K) of its CTA's simulation.  One step:
//    compute phase (all threads)
//        read the neighbours' boundary bins (published in smem by the previous step)
//        -> in-place sweep of eq-highRes_growth in flux form: right-to-left for C >= 0,
//           left-to-right for C < 0, so every face sees OLD values without a copy
//        -> round-off clip (R-17) -> moment partials (mu3 every step; mu0..mu2 and all
//           tangents on sample steps) -> warp transpose-reduce -> smem
//    bar1
//    publish phase (all threads): write own first/last two bins to smem (single buffer:
//        every read of the previous buffer happened before bar1)
//    scalar phase (warp 0): fixed-order cross-warp sums, mass balance
//        c^{n+1} = c^n - rho_c k_v (mu3^{n+1} - mu3^n), clock, sample
//        record + loss, then kinetics + time step of the NEXT step (L285, L693-705,
//        SI L857-861) in lane-parallel dual numbers (lane p carries tangent p)
//    bar2
//  The only global traffic inside the time loop is the sample records.
//
//  Flux form (R-3/R-6; LeVeque's wave-limiter form, cited by the paper at L290):
//     C >= 0: F_{i-1/2} = C n_{i-1} + kap psi(d_{i-1}, d_i)
//     C <  0: F_{i-1/2} = C n_i     + kap psi(d_{i+1}, d_i)
//     n_i <- n_i - (F_{i+1/2} - F_{i-1/2}),  kap = |C| (1 - |C|) / 2,  d_i = n_i - n_{i-1}
//  = eq-highRes_growth (L292-298) with phi_{i-1/2} (f_i - f_{i-1}) = psi(d_{i-1}, d_i).
//  Tangent lane p (row a8), using kapdot = beta Cdot, beta = sgn(C) (1 - 2|C|) / 2:
//     Fdot = Cdot (n_up + beta psi) + C ndot_up + kap (pa adot + pb bdot)
//  so only Cdot is lane-specific (8 FP64 ops per bin and lane).
// =====================================================================================
#pragma once
#include <cooperative_groups.h>

#include <type_traits>

#include "pbe_device.cuh"

namespace pbe {

#if PBE_TIMING
__device__ unsigned long long g_phase_cycles[12];   // sweep, moments+publish, barrier, scalar, steps, [scalar: sums, mass balance, kinetics]
#define PBE_TSTAMP(v) long long v = clock64()
#define PBE_TACC(i, a, b) t_acc[i] += (unsigned long long)((b) - (a))   // registers; written at exit
#else
#define PBE_TSTAMP(v)
#define PBE_TACC(i, a, b)
#endif

// Smem halo: s_halo[(side * V + v) * HS + t + 1], HS = NT + 2, side 0/1 = bins 0/1 of
// thread t, side 2/3 = bins K-2/K-1 (transposed so a warp's accesses are consecutive).
// Columns 0 and NT + 1 stay zero: the ghost cells n_{-2} = n_{-1} = n_N = n_{N+1} = 0.
template <int P, int K, bool NEG, int LK, class CdT>   // LK: 0 upwind, 1 van Leer, 2 minmod/superbee/MC
__device__ __forceinline__ bool sweep_bins(double (&x)[1 + P][K], const double* __restrict__ s_halo,
                                           int NT, int tid, double C, double kap, double beta,
                                           const CdT& Cd, int lim, int i0, int N,
                                           double clip_thr) {
    constexpr int V = 1 + P;
    bool bad = false;
    const int HS = NT + 2;
    const double kap2 = 2.0 * kap, beta2 = 2.0 * beta;
    // value of variable v at local bin j in [-2, K+1] (OLD values: the sweep order
    // guarantees x[v][j] is not yet updated when it is read here)
    auto X = [&](int v, int j) -> double {
        if (j >= 0 && j < K) return x[v][j];
        if (j == -1) return s_halo[(3 * V + v) * HS + tid];
        if (j == -2) return s_halo[(2 * V + v) * HS + tid];
        if (j == K) return s_halo[(0 * V + v) * HS + tid + 2];
        return s_halo[(1 * V + v) * HS + tid + 2];                 // j == K + 1
    };
    // Face between local bins (f-1, f).  For C >= 0: a = d_{f-1}, b = d_f, upwind f-1;
    // for C < 0: a = d_{f+1}, b = d_f, upwind f.  Primal parts first (shared by all lanes).
    double Fc = 0.0, Fdc[P > 0 ? P : 1];        // fluxes of the face shared with the previous bin
    // Face between local bins (f-1, f): primal flux F and the lane-flux coefficients.
    //   C >= 0: a = d_{f-1}, b = d_f, upwind f-1;   C < 0: a = d_{f+1}, b = d_f, upwind f.
    // Lane flux  Fdot = Cdot (n_up + beta psi) + C ndot_up + kap (pa adot + pb bdot)
    // regrouped over the three cells it touches (lo = f-2 | f-1, mid, hi = f | f+1):
    //   C >= 0: w_hi ndot_f + w_mid ndot_{f-1} + w_lo ndot_{f-2},
    //           w_hi = kap pb, w_mid = C + kap (pa - pb), w_lo = -kap pa
    //   C <  0: w_hi ndot_{f+1} + w_mid ndot_f + w_lo ndot_{f-1},
    //           w_hi = kap pa, w_mid = C - kap (pa - pb), w_lo = -kap pb
    struct FaceP { double F, g, w_lo, w_mid, w_hi; };
    auto face_primal = [&](int f) -> FaceP {
        const int u = NEG ? f : f - 1;
        const int ja = NEG ? f + 1 : f - 1;
        const double a = X(0, ja) - X(0, ja - 1), b = X(0, f) - X(0, f - 1);
        double h = 0.0, qa = 0.0, qb = 0.0;          // psi = 2h, d psi/da = 2qa, d psi/db = 2qb
        if (LK == 2) psi_half_other(lim, a, b, h, qa, qb);     // minmod / superbee / MC (NEXT-4)
        else if (LK == 1) psi_half_d_bf(a, b, h, qa, qb);      // no branch: faces overlap
        const double nup = X(0, u);
        FaceP r;
        r.F = fma(C, nup, kap2 * h);                   // C n_up + kap psi
        r.g = fma(beta2, h, nup);                      // n_up + beta psi
        const double pak = kap2 * qa, pbk = kap2 * qb; // kap d psi/da, kap d psi/db
        if (!NEG) { r.w_hi = pbk; r.w_mid = C + (pak - pbk); r.w_lo = -pak; }
        else      { r.w_hi = pak; r.w_mid = C - (pak - pbk); r.w_lo = -pbk; }
        return r;
    };
    auto face_lane = [&](int f, int p, const FaceP& fp) -> double {
        const int lo = NEG ? f - 1 : f - 2;
        return fma(Cd[p], fp.g, fma(fp.w_hi, X(1 + p, lo + 2), fma(fp.w_mid, X(1 + p, lo + 1), fp.w_lo * X(1 + p, lo))));
    };
    // update bin k from its two faces; the lane fluxes of the far face come from Fdc and
    // are replaced in place by the near face's (so only one array of lane fluxes is live)
    bool neg = false;
    // update bin k from its new face (primal part fp, computed one iteration ahead so its
    // reciprocal chain overlaps the previous face's lane work) and the carried face fluxes
    auto step_bin = [&](int k, int f_new, bool new_is_left, const FaceP& fp) {
        const double dF = new_is_left ? (Fc - fp.F) : (fp.F - Fc);
        const double nn = x[0][k] - dF;
        neg |= (nn < 0.0);
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const double fl = face_lane(f_new, p, fp);     // reads OLD x[1+p][*] only
            const double dFd = new_is_left ? (Fdc[p] - fl) : (fl - Fdc[p]);
            Fdc[p] = fl;
            x[1 + p][k] = x[1 + p][k] - dFd;
        }
        x[0][k] = nn;
        Fc = fp.F;
    };
    if (!NEG) {
        {   // right face of bin K-1
            const FaceP fp = face_primal(K);
            Fc = fp.F;
#pragma unroll
            for (int p = 0; p < P; ++p) Fdc[p] = face_lane(K, p, fp);
        }
        FaceP fp = face_primal(K - 1);
#pragma unroll
        for (int k = K - 1; k >= 0; --k) {          // left face of bin k: reads bins < k (old)
            const FaceP fnext = k > 0 ? face_primal(k - 1 > 0 ? k - 1 : 0) : fp;
            step_bin(k, k, true, fp);
            fp = fnext;
        }
    } else {
        {   // left face of bin 0
            const FaceP fp = face_primal(0);
            Fc = fp.F;
#pragma unroll
            for (int p = 0; p < P; ++p) Fdc[p] = face_lane(0, p, fp);
        }
        FaceP fp = face_primal(1);
#pragma unroll
        for (int k = 0; k < K; ++k) {               // right face of bin k: reads bins > k (old)
            const FaceP fnext = k + 1 < K ? face_primal(k + 2 < K + 1 ? k + 2 : K) : fp;
            step_bin(k, k + 1, false, fp);
            fp = fnext;
        }
    }
    // Clip (R-17), applied after the sweep (every face above used OLD values, so deferring
    // it is exact): round-off negatives and ghost bins i >= N become exactly 0 together with
    // their tangents; a negative below -clip_thr flags PBE_ERR_NEGATIVE.  Warp-uniform slow
    // path, taken only by warps holding padding bins or a negative.
    if (__any_sync(0xffffffffu, neg || (i0 + K > N))) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int i = i0 + k;
            const double nn = x[0][k];
            const bool zero = (i >= N) || (nn < 0.0 && nn >= -clip_thr);
            bad |= (nn < -clip_thr) && (i < N);
            x[0][k] = zero ? 0.0 : nn;
#pragma unroll
            for (int p = 0; p < P; ++p) x[1 + p][k] = zero ? 0.0 : x[1 + p][k];
        }
    }
    return bad;
}

// Long polynomial growth law WITH parameter seeds (tangent lanes, n > MAXTH): as
// poly_long_warp, and lane l's chunk also accumulates, for every tangent p of the CTA,
// sum_{j in chunk} seed_{p,j} x^(j+1) (P Horner chains); butterfly sums give every lane all P
// totals; lane p's tangent is its total + dG/dx dS.  O(n/32 * P) steps instead of O(n).
template <int PP>
__device__ __forceinline__ D1 poly_long_warp_seeded(const double* __restrict__ a, const double* __restrict__ seed,
                                                     int nsd, int lane0, int nl, int n, D1 S, int pl) {
    if (!(S.v > 1.0)) return mk(0.0);
    const int lane = threadIdx.x & 31;
    const double x = S.v - 1.0;
    const int m = (n + 31) >> 5;
    const int j0 = lane * m;
    double q = 0.0, dq = 0.0, sp[PP];
#pragma unroll
    for (int p = 0; p < PP; ++p) sp[p] = 0.0;
    for (int i = m - 1; i >= 0; --i) {
        const int j = j0 + i;
        const bool on = j < n;
        const double aj = on ? __ldg(a + j) : 0.0;
        dq = fma(dq, x, q);
        q = fma(q, x, aj);
#pragma unroll
        for (int p = 0; p < PP; ++p)
            sp[p] = fma(sp[p], x, (on && p < nl) ? __ldg(seed + (size_t)(lane0 + p) * nsd + j) : 0.0);
    }
    const double xl = ipow(x, j0), xl1 = xl * x;          // x^(l m), x^(l m + 1)
    double t = xl1 * q;
    double dt = xl * fma((double)(j0 + 1), q, x * dq);
#pragma unroll
    for (int p = 0; p < PP; ++p) sp[p] *= xl1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        t += __shfl_xor_sync(0xffffffffu, t, off);
        dt += __shfl_xor_sync(0xffffffffu, dt, off);
#pragma unroll
        for (int p = 0; p < PP; ++p) sp[p] += __shfl_xor_sync(0xffffffffu, sp[p], off);
    }
    double mine = 0.0;
#pragma unroll
    for (int p = 0; p < PP; ++p) if (p == pl) mine = sp[p];
    return {t, fma(dt, S.d, mine)};
}

// Grid: one CTA per simulation.  Block: NT = 32 NW threads with NT K >= N.
// P = tangent lanes per CTA.  The kp.P lanes of a simulation are split into kp.G lane
// groups of P: CTA b runs simulation b / G, group g = b % G, i.e. lanes [g P, g P + P)
// (lanes >= kp.P carry zero seeds and stay 0).  Every group recomputes the primal march
// (bitwise identically), so groups never communicate; group 0 writes the primal records.
// Dynamic smem: 2 parities x 4 V (NT + 2) doubles of halo.
//
// ONE CTA barrier per step: every warp keeps its own copy of the scalar state (c, t, mu3,
// sample index, status) and evaluates the kinetics redundantly from the same smem partial
// sums in the same order, so all warps take bitwise-identical decisions.  Halos, partial
// sums and the negative-density flag are double-buffered by step parity.
//
// CL = true: thread-block-cluster mode (k_cluster, 10^4 - 10^5 bins).  A cluster of CS CTAs
// (launch attribute, <= 16) marches one simulation; CTA rank r owns bins
// [(r NT + t) K, ...).  The boundary bins of neighbouring CTAs are written straight into
// the neighbour's ghost column through distributed shared memory, every CTA pre-reduces
// its warps' moment partials, and the scalar phase sums the CS CTA totals over DSMEM in
// rank order.  The one barrier per step becomes a cluster barrier.
template <int P, int K, int MAXT, bool CL = false, int MINB = 1>
__global__ void __launch_bounds__(MAXT, MINB) k_resident(const KParams kp) {
    namespace cg = cooperative_groups;
#if PBE_TIMING
    unsigned long long t_acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif
    constexpr int V = 1 + P;
    constexpr int PP = P > 0 ? P : 1;
    static_assert(K >= 2, "K >= 2");
    const int CS = CL ? (int)cg::this_cluster().num_blocks() : 1;
    const int rank = CL ? (int)cg::this_cluster().block_rank() : 0;
    const int unit = blockIdx.x / CS;
    const int s = unit / kp.G;
    const int grp = unit - s * kp.G;
    const int lane0 = grp * P;                                 // first tangent lane of the group
    const int nl = P > 0 ? max(0, min(P, kp.P - lane0)) : 0;   // lanes of this group in use
    const bool primal_out = (grp == 0) && (rank == 0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NT = blockDim.x, NW = NT >> 5;
    const int N = kp.N;
    const int i0 = (rank * NT + tid) * K;
    auto block_barrier = [&]() {
        if (CL) cg::this_cluster().sync(); else __syncthreads();
    };
    const int HS = NT + 2;
    const int HP = 4 * V * HS;                  // doubles per halo parity
    const bool steps_mode = kp.n_steps > 0;
    const double L_half = kp.L_lo + 0.5 * kp.dL;          // centre of bin 0
    const int red_idx = reduce_index<V>(lane);

    extern __shared__ double s_halo[];          // [2][4][V][NT + 2], WarpPart[32], LanePart[NT]
    __shared__ double s_red[2][32][4][V];       // [parity][warp][moment][value]
    __shared__ long long s_bad[2];              // step index that produced a negative
    __shared__ double s_nscale;
    __shared__ double s_cta[2][4][V];           // cluster mode: this CTA's moment totals
    __shared__ double s_cdw[MINB > 1 ? 32 * PP : 1];   // per-warp Cdot slots (MINB = 2 variants)

    double x[V][K];
    // ---- load n0 (tangents start at 0: n0 does not depend on theta, R-20) --------------
    const double* n0 = kp.n0 + (size_t)s * kp.n0_stride;
    double lmax = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int i = i0 + k;
        x[0][k] = (i < N) ? __ldg(n0 + i) : 0.0;
        lmax = fmax(lmax, x[0][k]);
#pragma unroll
        for (int p = 0; p < P; ++p) x[1 + p][k] = 0.0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, off));
    if (lane == 0) s_red[0][warp][0][0] = lmax;
    if (tid < 2) s_bad[tid] = -1;
    for (int j = tid; j < 8 * V; j += NT) { s_halo[j * HS] = 0.0; s_halo[j * HS + NT + 1] = 0.0; }
    __syncthreads();
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < NW; ++w) m = fmax(m, s_red[0][w][0][0]);
        s_nscale = m;
    }
    if (CL) {   // clip scale = max over the whole simulation
        cg::this_cluster().sync();
        if (tid == 0) {
            double m = 0.0;
            for (int r = 0; r < CS; ++r) m = fmax(m, *cg::this_cluster().map_shared_rank(&s_nscale, r));
            s_red[1][0][0][0] = m;
        }
        cg::this_cluster().sync();
        if (tid == 0) s_nscale = s_red[1][0][0][0];
    }

    auto publish_halo = [&](int q) {
        double* h = s_halo + q * HP;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            h[(0 * V + v) * HS + tid + 1] = x[v][0];
            h[(1 * V + v) * HS + tid + 1] = x[v][1];
            h[(2 * V + v) * HS + tid + 1] = x[v][K - 2];
            h[(3 * V + v) * HS + tid + 1] = x[v][K - 1];
        }
        if (CL) {   // DSMEM: my edge bins -> the neighbour CTAs' ghost columns
            if (tid == NT - 1 && rank + 1 < CS) {
                double* hr = cg::this_cluster().map_shared_rank(h, rank + 1);
#pragma unroll
                for (int v = 0; v < V; ++v) { hr[(2 * V + v) * HS] = x[v][K - 2]; hr[(3 * V + v) * HS] = x[v][K - 1]; }
            }
            if (tid == 0 && rank > 0) {
                double* hl = cg::this_cluster().map_shared_rank(h, rank - 1);
#pragma unroll
                for (int v = 0; v < V; ++v) { hl[(0 * V + v) * HS + NT + 1] = x[v][0]; hl[(1 * V + v) * HS + NT + 1] = x[v][1]; }
            }
        }
    };
    // cluster mode: this CTA's totals of the warp partials (fixed warp order) -> s_cta[q]
    auto cta_totals = [&](int q, bool all_moments) {
        if (!CL) return;
        __syncthreads();
        if (warp == 0) {
            for (int e = lane; e < 4 * V; e += 32) {
                const int km = e / V, v = e - km * V;
                if (km == 3 || all_moments) {
                    double a = 0.0;
                    for (int w = 0; w < NW; ++w) a += s_red[q][w][km][v];
                    s_cta[q][km][v] = a;
                }
            }
        }
    };
    // moment KM partials of all V variables, warp-reduced into s_red[q][warp][KM][*]
    // mu3 weights dL L_i^3 of this thread's bins, computed once (same formula as below, so the
    // per-step moments are bitwise those of the on-the-fly weights); [K][NT] after the halo
    double* s_w3 = s_halo + 2 * HP;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double Lc = fma((double)(i0 + k), kp.dL, L_half);
        s_w3[k * NT + tid] = ((kp.dL * Lc) * Lc) * Lc;
    }
    auto moment_partials = [&](int q, auto kmc) {
        constexpr int KM = decltype(kmc)::value;
        double acc[V];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double w;
            if (KM == 3) w = s_w3[k * NT + tid];
            else {
                const double Lc = fma((double)(i0 + k), kp.dL, L_half);   // bin centre
                w = kp.dL;
#pragma unroll
                for (int e = 0; e < KM; ++e) w *= Lc;
            }
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v] = fma(w, x[v][k], acc[v]);
        }
        warp_transpose_reduce<V>(acc, lane);
        if (red_idx < V) s_red[q][warp][KM][red_idx] = acc[0];
    };

    __syncthreads();
    const double clip_thr = 1e-12 * s_nscale;
    moment_partials(1, std::integral_constant<int, 3>{});   // mu3(n0): "step -1" outputs in parity 1
    publish_halo(1);
    cta_totals(1, false);
    block_barrier();

    // ---- per-warp scalar state (lane p: primal + tangent p) ------------------------------
    // Kept in smem between scalar phases (one slot per thread) so that the sweep has the
    // register file to itself; only C, kap, beta and the lane tangents Cdot live across it.
    struct LaneScal {
        D1 c, t, mu3p, dt;
        double loss, gacc, rms_c, rms_L, tn;       // tn = t_samples[m] (read once per sample)
        long long nstep;
        int m, status, landing;
    };
    // smem copy: primal part once per warp (identical in all lanes), tangent part per lane
    struct WarpPart { double c, t, mu3p, dt, loss, rms_c, rms_L, tn; long long nstep; int m, status, landing; };
    struct LanePart { double c, t, mu3p, dt, gacc; };
    // static shared arrays (direct LDS/STS; a pointer carved out of the dynamic buffer makes the
    // compiler form generic addresses, rematerialised every step)
    // (primal-only variants keep no tangent part: every .d is 0 and small CTAs stay small, so
    // many fit per SM)
    __shared__ WarpPart s_wp[MAXT / 32];
    __shared__ LanePart s_lp[P > 0 ? MAXT : 1];
    auto load_ls = [&]() -> LaneScal {
        const WarpPart w = s_wp[warp];
        const LanePart l = P > 0 ? s_lp[tid] : LanePart{0.0, 0.0, 0.0, 0.0, 0.0};
        LaneScal L;
        L.c = mk(w.c, l.c); L.t = mk(w.t, l.t); L.mu3p = mk(w.mu3p, l.mu3p); L.dt = mk(w.dt, l.dt);
        L.loss = w.loss; L.gacc = l.gacc; L.rms_c = w.rms_c; L.rms_L = w.rms_L; L.tn = w.tn;
        L.nstep = w.nstep; L.m = w.m; L.status = w.status; L.landing = w.landing;
        return L;
    };
    auto store_ls = [&](const LaneScal& L) {
        __syncwarp();
        if (lane == 0)
            s_wp[warp] = WarpPart{L.c.v, L.t.v, L.mu3p.v, L.dt.v, L.loss, L.rms_c, L.rms_L, L.tn, L.nstep, L.m,
                                  L.status, L.landing};
        if (P > 0) s_lp[tid] = LanePart{L.c.d, L.t.d, L.mu3p.d, L.dt.d, L.gacc};
    };
    const int pl = lane < nl ? lane : -1;                      // this lane's tangent within the group
    const KinLoader KL{kp.theta + (size_t)s * kp.n_params, kp.sol, kp.seed, pl >= 0 ? lane0 + pl : -1, kp.n_params,
                       kp.n_params + kp.n_sol};
    const double* kT = kp.knot_T + (size_t)s * kp.knotT_stride;
    const bool has_target = kp.target != nullptr;
    const double* tgt = has_target ? kp.target + (size_t)s * kp.M * 2 : nullptr;
    double C = 0.0, kap = 0.0, beta = 0.0, Cd_l = 0.0;

    // kinetics + time step of the next step from scalar state L (row a1, a2).  Parameters and this
    // group's seed rows are staged in shared memory (read by every warp every step).
    const KinCache KC = kin_cache(kp, KL, kT);
    const bool kin_smem = kp.n_params <= MAXTH;
    const int nsd = kp.n_params + kp.n_sol;
    __shared__ double s_th[MAXTH], s_sol[3], s_seed[PP * (MAXTH + 3)];
    // POLY fast path: coefficient j as lane l's dual number, lane-major, zero-padded to MAXTH
    // (a zero term changes no Horner step: g x + 0 == g x), read with direct shared indexing
    __shared__ double2 s_poly[MAXTH][32];
    const bool poly_fast = kin_smem && kp.law == LAW_POLY && KC.const_T;
    if (kin_smem) {
        const double* th = kp.theta + (size_t)s * kp.n_params;
        for (int j = tid; j < kp.n_params; j += NT) s_th[j] = th[j];
        for (int j = tid; j < kp.n_sol; j += NT) s_sol[j] = kp.sol[j];
        for (int j = tid; j < nl * nsd; j += NT) s_seed[j] = kp.seed[(size_t)lane0 * nsd + j];
        for (int e = tid; e < MAXTH * 32; e += NT) {
            const int j = e >> 5, l = e & 31;
            const bool on = j < kp.n_params;
            const bool seeded = on && l < nl;
            s_poly[j][l] = make_double2(on ? th[j] : 0.0, seeded ? kp.seed[(size_t)(lane0 + l) * nsd + j] : 0.0);
        }
    }
    __syncthreads();
    const KinLoaderS KLS{s_th, s_sol, s_seed, pl, kp.n_params, nsd};
    auto kinetics_with = [&](const auto& LDR, LaneScal& L) -> bool {
        PBE_TSTAMP(tk0);
        D1 T;
        D1 G;
        if (poly_fast) {                               // S = c / c*(T) at constant T, eq-poly_growth_rate
            T = KC.T;
            const D1 S = L.c * KC.ics;
            G = mk(0.0);
            if (S.v > 1.0) {
                const D1 x = S - 1.0;
#pragma unroll
                for (int j = MAXTH - 1; j >= 0; --j) {
                    const double2 a = s_poly[j][lane];
                    G = G * x + mk(a.x, a.y);
                }
                G = G * x;
            }
        } else if (kp.law == LAW_POLY && kp.n_params > MAXTH) {            // long polynomial: warp-cooperative
            const D1 S = supersaturation(kp, LDR, kT, KC, L.t, L.c, T);
            if (P == 0) G = poly_long_warp(kp.theta + (size_t)s * kp.n_params, kp.n_params, S);
            else G = poly_long_warp_seeded<PP>(kp.theta + (size_t)s * kp.n_params, kp.seed, nsd, lane0, nl,
                                               kp.n_params, S, pl);
        } else {
            const D1 S = supersaturation(kp, LDR, kT, KC, L.t, L.c, T);
            G = growth_rate(kp, LDR, S, T);
        }
#if PBE_TIMING
        volatile double sink_g = G.v + G.d; (void)sink_g;          // pin the stamp after G
#endif
        PBE_TSTAMP(tk1);
        PBE_TACC(8, tk0, tk1);
        const double tn = steps_mode ? 0.0 : L.tn;
        const StepScalars sc = time_step(kp, G, L.t, tn, steps_mode);
#if PBE_TIMING
        volatile double sink_c = sc.C.v + sc.kap.v; (void)sink_c;
#endif
        PBE_TSTAMP(tk2);
        PBE_TACC(9, tk1, tk2);
        if (sc.err != ST_OK) { L.status = sc.err; return false; }
        L.dt = sc.dt;
        L.landing = sc.landing;
        C = sc.C.v;
        kap = sc.kap.v;
        beta = C > 0.0 ? 0.5 * (1.0 - 2.0 * C) : (C < 0.0 ? -0.5 * (1.0 + 2.0 * C) : 0.0);  // kapdot = beta Cdot
        Cd_l = sc.C.d;
        return true;
    };
    auto kinetics = [&](LaneScal& L) -> bool { return kin_smem ? kinetics_with(KLS, L) : kinetics_with(KL, L); };

    bool go = true, sample = false;
    {
        LaneScal L;
        double a = 0.0;
        if (CL) {
            for (int r = 0; r < CS; ++r) a += cg::this_cluster().map_shared_rank(&s_cta[1][3][0], r)[0];
        } else {
            a = sum4u<(MAXT + 31) / 32>(&s_red[1][0][3][0], 4 * V, NW);
        }
        L.c = mk(kp.c0[s]); L.t = mk(0.0); L.mu3p = mk(a, 0.0); L.dt = mk(0.0);
        L.loss = 0.0; L.gacc = 0.0; L.rms_c = 1.0; L.rms_L = 1.0;
        L.tn = steps_mode ? 0.0 : kp.t_samples[0];
        L.nstep = 0; L.m = 0; L.status = ST_OK; L.landing = 0;
        if (warp == 0 && has_target) {
            double sc2 = 0.0, sl2 = 0.0;
            for (int j = lane; j < kp.M; j += 32) { sc2 += tgt[2 * j] * tgt[2 * j]; sl2 += tgt[2 * j + 1] * tgt[2 * j + 1]; }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                sc2 += __shfl_xor_sync(0xffffffffu, sc2, off);
                sl2 += __shfl_xor_sync(0xffffffffu, sl2, off);
            }
            L.rms_c = sqrt(sc2 / kp.M); L.rms_L = sqrt(sl2 / kp.M);
        }
        if (kp.max_steps <= 0) { L.status = ST_MAXSTEPS; go = false; }
        if (go) go = kinetics(L);
        sample = go && (L.landing || (steps_mode && kp.n_steps == 1));
        store_ls(L);
    }

    const int vl = kp.limiter;                                  // limiter id
    const bool gen = vl != LIM_VANLEER && vl != LIM_UPWIND;      // NEXT-4 limiters: generic sweep
    long long n = 0;
    while (go) {
        const int q = (int)(n & 1), qp = q ^ 1;
        bool bad;
        PBE_TSTAMP(tc0);
        const double* hin = s_halo + qp * HP;
        if (MINB == 1) {
            // lane tangents of C in registers
            double Cd[PP];
#pragma unroll
            for (int p = 0; p < PP; ++p) Cd[p] = (p < P) ? __shfl_sync(0xffffffffu, Cd_l, p) : 0.0;
            if (vl == LIM_VANLEER) {
                if (C >= 0.0) bad = sweep_bins<P, K, false, 1>(x, hin, NT, tid, C, kap, beta, Cd, vl, i0, N, clip_thr);
                else          bad = sweep_bins<P, K, true, 1>(x, hin, NT, tid, C, kap, beta, Cd, vl, i0, N, clip_thr);
            } else if (!gen) {
                if (C >= 0.0) bad = sweep_bins<P, K, false, 0>(x, hin, NT, tid, C, kap, beta, Cd, vl, i0, N, clip_thr);
                else          bad = sweep_bins<P, K, true, 0>(x, hin, NT, tid, C, kap, beta, Cd, vl, i0, N, clip_thr);
            } else {
                if (C >= 0.0) bad = sweep_bins<P, K, false, 2>(x, hin, NT, tid, C, kap, beta, Cd, vl, i0, N, clip_thr);
                else          bad = sweep_bins<P, K, true, 2>(x, hin, NT, tid, C, kap, beta, Cd, vl, i0, N, clip_thr);
            }
        } else {
            // 2 CTAs/SM (<= 128 registers): lane tangents of C re-read from this warp's smem slot
            volatile double* cdw = s_cdw + warp * PP;
            if (lane < PP) cdw[lane] = Cd_l;
            __syncwarp();
            if (vl == LIM_VANLEER) {
                if (C >= 0.0) bad = sweep_bins<P, K, false, 1>(x, hin, NT, tid, C, kap, beta, cdw, vl, i0, N, clip_thr);
                else          bad = sweep_bins<P, K, true, 1>(x, hin, NT, tid, C, kap, beta, cdw, vl, i0, N, clip_thr);
            } else if (!gen) {
                if (C >= 0.0) bad = sweep_bins<P, K, false, 0>(x, hin, NT, tid, C, kap, beta, cdw, vl, i0, N, clip_thr);
                else          bad = sweep_bins<P, K, true, 0>(x, hin, NT, tid, C, kap, beta, cdw, vl, i0, N, clip_thr);
            } else {
                if (C >= 0.0) bad = sweep_bins<P, K, false, 2>(x, hin, NT, tid, C, kap, beta, cdw, vl, i0, N, clip_thr);
                else          bad = sweep_bins<P, K, true, 2>(x, hin, NT, tid, C, kap, beta, cdw, vl, i0, N, clip_thr);
            }
        }
        PBE_TSTAMP(tc1);
        PBE_TACC(0, tc0, tc1);
        if (bad) s_bad[q] = n;
        moment_partials(q, std::integral_constant<int, 3>{});     // mu3 of n and every tangent lane
        if (sample) {
            moment_partials(q, std::integral_constant<int, 0>{});
            moment_partials(q, std::integral_constant<int, 1>{});
            moment_partials(q, std::integral_constant<int, 2>{});
        }
        publish_halo(q);
        cta_totals(q, sample);
        PBE_TSTAMP(tc2);
        PBE_TACC(1, tc1, tc2);
        block_barrier();                         // the one (cluster) barrier of the step
        PBE_TSTAMP(tc3);
        PBE_TACC(2, tc2, tc3);

        // ---- scalar phase (every warp, identical arithmetic) -----------------------------
        LaneScal L = load_ls();
        double tot[4] = {0.0, 0.0, 0.0, 0.0}, totd[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int km = 0; km < 4; ++km) {
            if (km == 3 || sample) {
                double a = 0.0, b = 0.0;
                if (CL) {
                    for (int r = 0; r < CS; ++r) {
                        const double* rc = cg::this_cluster().map_shared_rank(&s_cta[q][km][0], r);
                        a += rc[0];
                        if (pl >= 0) b += rc[1 + pl];
                    }
                } else {
                    // lane v < V sums component v over the warps (fixed order, sum4u), then the
                    // primal total and this lane's tangent total are broadcast by shuffles
                    const double tv = lane < V ? sum4u<(MAXT + 31) / 32>(&s_red[q][0][km][lane], 4 * V, NW) : 0.0;
                    a = __shfl_sync(0xffffffffu, tv, 0);
                    b = __shfl_sync(0xffffffffu, tv, pl >= 0 ? 1 + pl : 0);
                    if (pl < 0) b = 0.0;
                }
                tot[km] = a; totd[km] = b;
            }
        }
        PBE_TSTAMP(ts1);
        PBE_TACC(5, tc3, ts1);
        const D1 mu3n = mk(tot[3], totd[3]);
        const D1 cn = L.c - kp.rho_kv * (mu3n - L.mu3p);        // eq-discrete_mass_balance
        bool any_bad = s_bad[q] == n;
        if (CL)
            for (int r = 0; r < CS; ++r) any_bad |= (*cg::this_cluster().map_shared_rank(&s_bad[q], r) == n);
        if (any_bad) { L.status = ST_NEG; go = false; }
        else if (cn.v < 0.0) { L.status = ST_INFEAS; go = false; }
        else {
            L.c = cn; L.mu3p = mu3n;
            L.t = L.landing ? mk(kp.t_samples[L.m], 0.0) : L.t + L.dt;
            ++L.nstep;
            if (sample && warp == 0 && rank == 0) {
                const int mr = steps_mode ? 0 : L.m;
                double* r = kp.rec + ((size_t)s * kp.M + mr) * 6;
                if (lane == 0 && primal_out) { r[0] = L.t.v; r[1] = L.c.v; r[2] = tot[0]; r[3] = tot[1]; r[4] = tot[2]; r[5] = tot[3]; }
                if (pl >= 0) {
                    double* rt = kp.trec + (((size_t)s * kp.M + mr) * kp.P + lane0 + pl) * 5;
                    rt[0] = L.c.d; rt[1] = totd[0]; rt[2] = totd[1]; rt[3] = totd[2]; rt[4] = totd[3];
                }
                if (has_target) {
                    const double Lb = tot[1] / tot[0];
                    const double Lbd = (totd[1] * tot[0] - tot[1] * totd[0]) / (tot[0] * tot[0]);
                    const double rc = (L.c.v - tgt[2 * mr]) / L.rms_c, rL = (Lb - tgt[2 * mr + 1]) / L.rms_L;
                    L.loss += rc * rc + rL * rL;
                    L.gacc += 2.0 * (rc / L.rms_c) * L.c.d + 2.0 * (rL / L.rms_L) * Lbd;
                }
            }
            if (L.landing) { ++L.m; if (L.m < kp.M) L.tn = kp.t_samples[L.m]; }
            PBE_TSTAMP(ts2);
            PBE_TACC(6, ts1, ts2);
            if (steps_mode ? (L.nstep >= kp.n_steps) : (L.m >= kp.M)) go = false;
            else if (L.nstep >= kp.max_steps) { L.status = ST_MAXSTEPS; go = false; }
            else go = kinetics(L);
            PBE_TSTAMP(ts3);
            PBE_TACC(7, ts2, ts3);
        }
        sample = go && (L.landing || (steps_mode && L.nstep + 1 == kp.n_steps));
        store_ls(L);
        ++n;
        PBE_TSTAMP(tc4);
        PBE_TACC(3, tc3, tc4);
        PBE_TACC(4, 0, 1);
    }

    // ---- epilogue -----------------------------------------------------------------------
#if PBE_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int i = 0; i < 12; ++i) g_phase_cycles[i] = t_acc[i];
#endif
    if (kp.n_final && grp == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) { const int i = i0 + k; if (i < N) kp.n_final[(size_t)s * N + i] = x[0][k]; }
    }
    if (kp.ndot_final) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            if (p < nl) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int i = i0 + k;
                    if (i < N) kp.ndot_final[((size_t)s * kp.P + lane0 + p) * N + i] = x[1 + p][k];
                }
            }
        }
    }
    if (warp == 0) {
        __syncwarp();
        const LaneScal L = load_ls();
        const bool ok = (L.status == ST_OK);
        const double qnan = __longlong_as_double(0x7ff8000000000000ll);
        if (lane == 0 && primal_out) {
            kp.status[s] = L.status;
            kp.steps[s] = L.nstep;
            if (kp.loss) kp.loss[s] = (has_target && ok) ? L.loss : qnan;
        }
        if (pl >= 0 && kp.grad && rank == 0) kp.grad[(size_t)s * kp.P + lane0 + pl] = (has_target && ok) ? L.gacc : qnan;
    }
    if (CL) cg::this_cluster().sync();   // keep this CTA's smem alive for DSMEM readers
}

}  // namespace pbe
