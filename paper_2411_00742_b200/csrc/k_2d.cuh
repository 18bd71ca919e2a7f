// =====================================================================================
//  k_2d — NEXT-1: the paper's 2D model (eq-PBE_batch_2d) with Godunov
//  dimensional splitting (L291: "update the PSSD ... along each spatial dimension separately
//  (i.e. twice)"), for batches of simulations.  One cooperative launch runs the whole march:
//
//    phase 1  every row along L1 (Courant C1 = G1 dt / dL1):  A -> B
//    grid barrier
//    phase 2  every column along L2 (C2 = G2 dt / dL2) on the result of phase 1: B -> A,
//             fused with the cross moments mu_pq (SI eq-moment2D, L873): mu_12 every step
//             (mass balance, eq-discrete_mass_balance L304-312), all six on sample steps
//    grid barrier
//    scalar phase: every CTA evaluates the kinetics of every simulation from the per-CTA
//             partials, in a fixed order (bitwise identical decisions in all CTAs):
//             dt = nu min(dL1/|G1|, dL2/|G2|) (SI L859), capped by dt_max and sample times
//
//  State: two buffers [S][R2][P1] (P1 = 4 ceil(N1/4) + 4, R2 = 4 ceil(N2/4) + 4), bin (j, i)
//  at row j + 2, column i + 2; ghost rows/columns are zero and never written (boundary
//  conditions); the padding covers the last 8-cell windows of both sweep directions.
//  Work split: K = 4 consecutive bins per thread along the sweep direction; row sweeps
//  load a contiguous 8-cell window (16-byte loads), column sweeps put consecutive threads on
//  consecutive columns (coalesced).  A unit u of simulation s goes to CTA u mod G, so the
//  order of every partial sum depends on the simulation alone, never on the batch.
//  Algorithmic traffic: 2 x (8 B read + 8 B write) per cell and step (two sweeps).
// =====================================================================================
#pragma once
#include "pbe_device.cuh"
#include "k_stream.cuh"   // grid_sync, ld_acquire

namespace pbe {

constexpr int K2D_NT = 256;
constexpr int K2D_K = 4;
constexpr int K2D_MAXS = 64;     // simulations per launch (smem coefficient cache)

struct Params2D {
    KParams kp;          // kp.N = N1, kp.dL = dL1; theta = [dim 1 | dim 2] (n_params even)
    int N2;
    double L2_lo, dL2, inv_dL2;
    double* A;           // [S][R2][P1]
    double* B;
    long long P1;        // row pitch (doubles)
    long long R2;        // rows per plane
    double* part;        // [S][G][7]  (mu00, mu10, mu01, mu11, mu02, mu12, negative flag)
    unsigned* bar;       // grid barrier [2]
    const unsigned long long* nscale_bits;  // [S] max(f0_s) bits
};

// Update K consecutive cells of one line (window w[0..K+3] = cells -2 .. K+1) with Courant C.
template <bool NEG>
__device__ __forceinline__ void line_update(const double (&w)[K2D_K + 4], double C, double kap2, int lim,
                                            double (&y)[K2D_K]) {
    double F[K2D_K + 1];
#pragma unroll
    for (int f = 2; f <= K2D_K + 2; ++f) {           // face between window cells f-1 | f
        const int u = NEG ? f : f - 1;
        const int ja = NEG ? f + 1 : f - 1;
        const double a = w[ja] - w[ja - 1], b = w[f] - w[f - 1];
        const double h = psi_half(lim, a, b);
        F[f - 2] = fma(C, w[u], kap2 * h);
    }
#pragma unroll
    for (int k = 0; k < K2D_K; ++k) y[k] = w[k + 2] - (F[k + 1] - F[k]);
}

__global__ void __launch_bounds__(K2D_NT, 3) k_2d(const Params2D p2) {
    const KParams& kp = p2.kp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = K2D_NT / 32;
    const unsigned G = gridDim.x;
    const int S = kp.n_sims, N1 = kp.N, N2 = p2.N2;
    const long long P1 = p2.P1, PL = p2.R2 * P1;                   // plane size
    const bool steps_mode = kp.n_steps > 0;
    const int vl = kp.limiter;                 // limiter (name kept: van Leer is the paper's)
    const int H = kp.n_params / 2;

    // per-simulation coefficients of the current step + scalar state (identical in all CTAs)
    __shared__ double s_C1[K2D_MAXS], s_k1[K2D_MAXS], s_C2[K2D_MAXS], s_k2[K2D_MAXS];
    __shared__ int s_active[K2D_MAXS], s_sample[K2D_MAXS];
    struct SimState { double c, t, mu12p, dt, clip; long long nstep; int m, status, landing; };
    __shared__ SimState s_ss[K2D_MAXS];
    __shared__ double s_red[NW][7];

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
            if (fabs(G2) > 1e-300) dtc = fmin(dtc, kp.courant * p2.dL2 * rcp_nr(fabs(G2)));
            dt = fmin(dtc, kp.dt_max);
        }
        bool landing = false;
        if (!steps_mode) {
            const double tn = kp.t_samples[W.m];
            if (W.t + dt >= tn - 1e-9 * dt) { dt = tn - W.t; landing = true; }
        } else if (isinf(dt)) {
            dt = 0.0;
        }
        const double C1 = G1 * dt * kp.inv_dL, C2 = G2 * dt * p2.inv_dL2;
        if (fabs(C1) > 1.0 || fabs(C2) > 1.0) { W.status = ST_CFL; return false; }
        W.dt = dt;
        W.landing = landing;
        if (lane == 0) {
            s_C1[s] = C1; s_k1[s] = fabs(C1) * (1.0 - fabs(C1));     // 2 kap
            s_C2[s] = C2; s_k2[s] = fabs(C2) * (1.0 - fabs(C2));
        }
        return true;
    };

    // fixed-order totals of simulation s: sum over CTAs of part[s][b][k]
    auto totals = [&](int s, double (&mu)[6], double& badf) {
        const double* pt = p2.part + (size_t)s * G * 7;
        double a[7] = {0, 0, 0, 0, 0, 0, 0};
        for (unsigned b = lane; b < G; b += 32)
#pragma unroll
            for (int k = 0; k < 7; ++k) a[k] += pt[(size_t)b * 7 + k];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
            for (int k = 0; k < 7; ++k) a[k] += __shfl_xor_sync(0xffffffffu, a[k], off);
#pragma unroll
        for (int k = 0; k < 6; ++k) mu[k] = a[k];
        badf = a[6];
    };

    // ---- initial state: mu12(f0) per CTA partials were written by the load kernel -------------
    unsigned gen = 0;
    for (int s = warp; s < S; s += NW) {
        double mu[6], badf;
        totals(s, mu, badf);
        SimState W{};
        W.c = kp.c0[s]; W.t = 0.0; W.mu12p = mu[5]; W.dt = 0.0; W.nstep = 0; W.m = 0; W.status = ST_OK;
        W.landing = 0;
        W.clip = 1e-12 * __longlong_as_double((long long)p2.nscale_bits[s]);
        bool go = kp.max_steps > 0;
        if (!go) W.status = ST_MAXSTEPS;
        if (go) go = kinetics(s, W);
        if (lane == 0) {
            s_active[s] = go;
            s_sample[s] = go && (W.landing || (steps_mode && kp.n_steps == 1));
            s_ss[s] = W;
        }
    }
    grid_sync(p2.bar, G, gen);     // everyone has read the initial partials

    const int rows_units = N2 * ((N1 + K2D_K - 1) / K2D_K);        // phase-1 units per simulation
    const int col_units = N1 * ((N2 + K2D_K - 1) / K2D_K);         // phase-2 units per simulation
    const int seg1 = (N1 + K2D_K - 1) / K2D_K;
    while (true) {
        int any = 0;
        for (int s = 0; s < S; ++s) any |= s_active[s];
        if (!any) break;
        // ---- phase 1: rows along L1, A -> B ---------------------------------------------------
        for (int s = 0; s < S; ++s) {
            if (!s_active[s]) continue;
            const double C = s_C1[s], kap2 = s_k1[s];
            const double* a = p2.A + (size_t)s * PL;
            double* b = p2.B + (size_t)s * PL;
            for (int u = blockIdx.x * K2D_NT + tid; u < rows_units; u += G * K2D_NT) {
                const int j = u / seg1, i0 = (u - j * seg1) * K2D_K;
                const double* row = a + (size_t)(j + 2) * P1 + i0;     // window cells i0-2 .. i0+5
                double w[K2D_K + 4], y[K2D_K];
#pragma unroll
                for (int q = 0; q < (K2D_K + 4) / 2; ++q) {
                    const double2 d = reinterpret_cast<const double2*>(row)[q];
                    w[2 * q] = d.x; w[2 * q + 1] = d.y;
                }
                if (C >= 0.0) line_update<false>(w, C, kap2, vl, y); else line_update<true>(w, C, kap2, vl, y);
                double* o = b + (size_t)(j + 2) * P1 + i0 + 2;
#pragma unroll
                for (int k = 0; k < K2D_K; ++k)
                    if (i0 + k < N1) o[k] = y[k];
            }
        }
        grid_sync(p2.bar, G, gen);
        // ---- phase 2: columns along L2 (B -> A) + cross moments ------------------------------------
        for (int s = 0; s < S; ++s) {
            if (!s_active[s]) continue;            // (uniform over the CTA)
            const double C = s_C2[s], kap2 = s_k2[s];
            const bool sample = s_sample[s] != 0;
            const double clip = s_ss[s].clip;
            const double* b = p2.B + (size_t)s * PL;
            double* a = p2.A + (size_t)s * PL;
            double acc[6] = {0, 0, 0, 0, 0, 0};
            bool bad = false;
            for (int u = blockIdx.x * K2D_NT + tid; u < col_units; u += G * K2D_NT) {
                const int jb = u / N1, i = u - jb * N1, j0 = jb * K2D_K;   // consecutive threads: columns
                const double* col = b + (size_t)j0 * P1 + i + 2;            // window rows j0-2 .. j0+5
                double w[K2D_K + 4], y[K2D_K];
#pragma unroll
                for (int q = 0; q < K2D_K + 4; ++q) w[q] = col[(size_t)q * P1];
                if (C >= 0.0) line_update<false>(w, C, kap2, vl, y); else line_update<true>(w, C, kap2, vl, y);
                const double L1 = fma((double)i, kp.dL, kp.L_lo + 0.5 * kp.dL);
                const double wa = kp.dL * p2.dL2;
#pragma unroll
                for (int k = 0; k < K2D_K; ++k) {
                    const int j = j0 + k;
                    if (j < N2) {
                        double v = y[k];
                        if (v < 0.0) { if (v >= -clip) v = 0.0; else bad = true; }   // round-off clip (R-17)
                        a[(size_t)(j + 2) * P1 + i + 2] = v;
                        const double L2 = fma((double)j, p2.dL2, p2.L2_lo + 0.5 * p2.dL2);
                        const double w00 = wa * v, w01 = w00 * L2, w02 = w01 * L2;
                        acc[5] = fma(L1, w02, acc[5]);                  // mu12
                        if (sample) {
                            acc[0] += w00; acc[1] = fma(L1, w00, acc[1]); acc[2] += w01;
                            acc[3] = fma(L1, w01, acc[3]); acc[4] += w02;
                        }
                    }
                }
            }
            // block reduction (fixed order) -> part[s][block]
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                for (int k = 0; k < 6; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
            const int anybad = __syncthreads_or(bad);
            if (lane == 0)
#pragma unroll
                for (int k = 0; k < 6; ++k) s_red[warp][k] = acc[k];
            __syncthreads();
            if (tid < 6) {
                double t = 0.0;
                for (int w2 = 0; w2 < NW; ++w2) t += s_red[w2][tid];
                p2.part[((size_t)s * G + blockIdx.x) * 7 + tid] = t;
            }
            if (tid == 6) p2.part[((size_t)s * G + blockIdx.x) * 7 + 6] = anybad ? 1.0 : 0.0;
            __syncthreads();
        }
        grid_sync(p2.bar, G, gen);
        // ---- scalar phase (every CTA, all simulations; warp per simulation) ----------------------
        for (int s = warp; s < S; s += NW) {
            if (!s_active[s]) continue;
            SimState W = s_ss[s];
            double mu[6], badf;
            totals(s, mu, badf);
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
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && tid < S) {
        kp.status[tid] = s_ss[tid].status;
        kp.steps[tid] = s_ss[tid].nstep;
    }
}

// f0 [S or 1][N2][N1] -> buffer A interior; per-CTA mu12 partials in the k_2d layout
// (part[s][b][5], CTA b of the k_2d grid owning column-units b, b + G, ...); max(f0) bits.
__global__ void __launch_bounds__(K2D_NT) k_2d_load(const double* __restrict__ f0, long long f0_stride, int S,
                                                    int N1, int N2, double* A, long long P1, long long R2, double* part,
                                                    unsigned G, unsigned long long* nscale_bits, double L_lo,
                                                    double dL, double L2_lo, double dL2) {
    // grid (G, S): block b reproduces k_2d's phase-2 unit assignment for simulation s
    const int s = blockIdx.y, tid = threadIdx.x;
    const long long PL = R2 * P1;
    const int col_units = N1 * ((N2 + K2D_K - 1) / K2D_K);
    double acc = 0.0, m = 0.0;
    for (int u = blockIdx.x * K2D_NT + tid; u < col_units; u += gridDim.x * K2D_NT) {
        const int jb = u / N1, i = u - jb * N1, j0 = jb * K2D_K;
        const double L1 = fma((double)i, dL, L_lo + 0.5 * dL);
        for (int k = 0; k < K2D_K; ++k) {
            const int j = j0 + k;
            if (j < N2) {
                const double v = f0[(size_t)s * f0_stride + (size_t)j * N1 + i];
                A[(size_t)s * PL + (size_t)(j + 2) * P1 + i + 2] = v;
                m = fmax(m, v);
                const double L2 = fma((double)j, dL2, L2_lo + 0.5 * dL2);
                const double w02 = dL * dL2 * v * L2 * L2;
                acc = fma(L1, w02, acc);
            }
        }
    }
    __shared__ double s_a[K2D_NT / 32], s_m[K2D_NT / 32];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, off);
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    }
    if ((tid & 31) == 0) { s_a[tid >> 5] = acc; s_m[tid >> 5] = m; }
    __syncthreads();
    if (tid == 0) {
        double t = 0.0, mm = 0.0;
        for (int w = 0; w < K2D_NT / 32; ++w) { t += s_a[w]; mm = fmax(mm, s_m[w]); }
        double* pt = part + ((size_t)s * G + blockIdx.x) * 7;
        for (int k = 0; k < 7; ++k) pt[k] = 0.0;
        pt[5] = t;
        atomicMax(nscale_bits + s, (unsigned long long)__double_as_longlong(mm));
    }
}

__global__ void k_2d_store(const double* __restrict__ A, int S, int N1, int N2, long long P1, long long R2,
                           double* f_final) {
    const long long PL = R2 * P1;
    const long long n = (long long)S * N2 * N1;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int s = (int)(e / ((long long)N2 * N1));
        const long long r = e - (long long)s * N2 * N1;
        const int j = (int)(r / N1), i = (int)(r - (long long)j * N1);
        f_final[e] = A[(size_t)s * PL + (size_t)(j + 2) * P1 + i + 2];
    }
}

}  // namespace pbe
