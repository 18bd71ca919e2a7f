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
#include "pbe_device.cuh"

namespace pbe {

// Smem halo: s_halo[(side * V + v) * HS + t + 1], HS = NT + 2, side 0/1 = bins 0/1 of
// thread t, side 2/3 = bins K-2/K-1 (transposed so a warp's accesses are consecutive).
// Columns 0 and NT + 1 stay zero: the ghost cells n_{-2} = n_{-1} = n_N = n_{N+1} = 0.
template <int P, int K, bool NEG>
__device__ __forceinline__ bool sweep_bins(double (&x)[1 + P][K], const double* __restrict__ s_halo,
                                           int NT, int tid, double C, double kap, double beta,
                                           const double (&Cd)[P > 0 ? P : 1], bool vl, int i0, int N,
                                           double clip_thr) {
    constexpr int V = 1 + P;
    bool bad = false;
    const int HS = NT + 2;
    // value of variable v at local bin j in [-2, K+1] (OLD values: the sweep order
    // guarantees x[v][j] is not yet updated when it is read here)
    auto X = [&](int v, int j) -> double {
        if (j >= 0 && j < K) return x[v][j];
        if (j == -1) return s_halo[(3 * V + v) * HS + tid];
        if (j == -2) return s_halo[(2 * V + v) * HS + tid];
        if (j == K) return s_halo[(0 * V + v) * HS + tid + 2];
        return s_halo[(1 * V + v) * HS + tid + 2];                 // j == K + 1
    };
    // flux through the face between local bins (f-1, f); returns primal F and fills Fd
    auto face = [&](int f, double (&Fd)[V]) -> double {
        // C >= 0: a = d_{f-1}, b = d_f, upwind f-1.   C < 0: a = d_{f+1}, b = d_f, upwind f.
        const int u = NEG ? f : f - 1;
        const int ja = NEG ? f + 1 : f - 1;
        const double a = X(0, ja) - X(0, ja - 1), b = X(0, f) - X(0, f - 1);
        double ps = 0.0, pa = 0.0, pb = 0.0;
        if (vl) psi_vl_d(a, b, ps, pa, pb);
        const double nup = X(0, u);
        const double F = fma(C, nup, kap * ps);
        if (P > 0) {
            const double g = fma(beta, ps, nup);
            const double pak = kap * pa, pbk = kap * pb;
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const double ad = X(1 + p, ja) - X(1 + p, ja - 1), bd = X(1 + p, f) - X(1 + p, f - 1);
                Fd[1 + p] = fma(Cd[p], g, fma(C, X(1 + p, u), fma(pak, ad, pbk * bd)));
            }
        }
        return F;
    };
    auto update = [&](int k, double Fl, double Fr, const double (&Fdl)[V], const double (&Fdr)[V]) {
        const int i = i0 + k;
        const double nn = x[0][k] - (Fr - Fl);
        bool zero = (i >= N);
        if (nn < 0.0) { if (nn >= -clip_thr) zero = true; else if (i < N) bad = true; }
        x[0][k] = zero ? 0.0 : nn;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const double nd = x[1 + p][k] - (Fdr[1 + p] - Fdl[1 + p]);
            x[1 + p][k] = zero ? 0.0 : nd;
        }
    };

    double Fc, Fdc[V];
    if (!NEG) {
        Fc = face(K, Fdc);                       // right face of bin K-1
#pragma unroll
        for (int k = K - 1; k >= 0; --k) {
            double Fdl[V];
            const double Fl = face(k, Fdl);      // left face of bin k (reads bins < k: old)
            update(k, Fl, Fc, Fdl, Fdc);
            Fc = Fl;
#pragma unroll
            for (int p = 0; p < P; ++p) Fdc[1 + p] = Fdl[1 + p];
        }
    } else {
        Fc = face(0, Fdc);                       // left face of bin 0
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double Fdr[V];
            const double Fr = face(k + 1, Fdr);  // right face of bin k (reads bins > k: old)
            update(k, Fc, Fr, Fdc, Fdr);
            Fc = Fr;
#pragma unroll
            for (int p = 0; p < P; ++p) Fdc[1 + p] = Fdr[1 + p];
        }
    }
    return bad;
}

// Grid: one CTA per simulation.  Block: NT = 32 NW threads with NT K >= N.
// P = instantiated tangent lanes (>= kp.P; extra lanes carry zero seeds and stay 0).
// Dynamic smem: 4 V (NT + 2) doubles of halo.
template <int P, int K, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_resident(const KParams kp) {
    constexpr int V = 1 + P;
    constexpr int PP = P > 0 ? P : 1;
    static_assert(K >= 2, "K >= 2");
    const int s = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NT = blockDim.x, NW = NT >> 5;
    const int N = kp.N;
    const int i0 = tid * K;
    const bool steps_mode = kp.n_steps > 0;

    extern __shared__ double s_halo[];          // [4][V][NT + 2]
    __shared__ double s_red[32][4][V];          // warp partial sums [warp][moment][value]
    __shared__ double s_C, s_kap, s_beta, s_Cd[PP], s_nscale;
    __shared__ int s_go, s_sample, s_bad;

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
    if (lane == 0) s_red[warp][0][0] = lmax;
    if (tid == 0) s_bad = 0;
    if (tid < PP) s_Cd[tid] = 0.0;               // lanes >= kp.P stay exactly 0
    __syncthreads();
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < NW; ++w) m = fmax(m, s_red[w][0][0]);
        s_nscale = m;
    }

    const int HS = NT + 2;
    auto publish_halo = [&]() {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            s_halo[(0 * V + v) * HS + tid + 1] = x[v][0];
            s_halo[(1 * V + v) * HS + tid + 1] = x[v][1];
            s_halo[(2 * V + v) * HS + tid + 1] = x[v][K - 2];
            s_halo[(3 * V + v) * HS + tid + 1] = x[v][K - 1];
        }
    };
    for (int j = tid; j < 4 * V; j += NT) { s_halo[j * HS] = 0.0; s_halo[j * HS + NT + 1] = 0.0; }
    // moment k partials of all V variables, warp-reduced into s_red[warp][k][*]
    auto moment_partials = [&](int kmom, int nv) {
        double acc[V];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double Lc = kp.L_lo + ((double)(i0 + k) + 0.5) * kp.dL;
            double w = kp.dL;
            for (int e = 0; e < kmom; ++e) w *= Lc;
#pragma unroll
            for (int v = 0; v < V; ++v)
                if (v < nv) acc[v] = fma(w, x[v][k], acc[v]);
        }
        warp_transpose_reduce<V>(acc, lane);
        const int idx = reduce_index<V>(lane);
        if (idx < V) s_red[warp][kmom][idx] = acc[0];
    };

    __syncthreads();
    const double clip_thr = 1e-12 * s_nscale;
    moment_partials(3, 1);                       // mu3(n0)
    publish_halo();

    // ---- warp-0 scalar state (each lane: primal + its own tangent lane) ----------------
    const int pl = lane < kp.P ? lane : -1;
    const KinLoader KL{kp.theta + (size_t)s * kp.n_params, kp.sol, kp.seed, pl, kp.n_params,
                       kp.n_params + kp.n_sol};
    const double* kT = kp.knot_T + (size_t)s * kp.knotT_stride;
    D1 c = mk(kp.c0[s]), t = mk(0.0), mu3p = mk(0.0), dt = mk(0.0);
    bool landing = false;
    int m = 0, status = ST_OK;
    long long nstep = 0;
    double loss = 0.0, gacc = 0.0, rms_c = 1.0, rms_L = 1.0;
    const bool has_target = kp.target != nullptr;
    const double* tgt = has_target ? kp.target + (size_t)s * kp.M * 2 : nullptr;

    auto kinetics = [&]() -> bool {   // next step's C, kap (+ tangents); false on CFL error
        const D1 T = temperature(kp, kT, t);
        const D1 cs = solubility(kp, KL, T);
        const D1 S = c / cs;
        const D1 G = growth_rate(kp, KL, S, T);
        const double tn = steps_mode ? 0.0 : kp.t_samples[m];
        const StepScalars sc = time_step(kp, G, t, tn, steps_mode);
        if (sc.err != ST_OK) { status = sc.err; return false; }
        dt = sc.dt;
        landing = sc.landing;
        if (lane == 0) {
            s_C = sc.C.v;
            s_kap = sc.kap.v;
            s_beta = sc.C.v > 0.0 ? 0.5 * (1.0 - 2.0 * sc.C.v) : (sc.C.v < 0.0 ? -0.5 * (1.0 + 2.0 * sc.C.v) : 0.0);
        }
        if (pl >= 0) s_Cd[pl] = sc.C.d;
        return true;
    };

    __syncthreads();   // bar1 (prologue)
    if (warp == 0) {
        double a = 0.0;
        for (int w = 0; w < NW; ++w) a += s_red[w][3][0];
        mu3p = mk(a, 0.0);
        if (has_target) {
            double sc2 = 0.0, sl2 = 0.0;
            for (int j = lane; j < kp.M; j += 32) { sc2 += tgt[2 * j] * tgt[2 * j]; sl2 += tgt[2 * j + 1] * tgt[2 * j + 1]; }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                sc2 += __shfl_xor_sync(0xffffffffu, sc2, off);
                sl2 += __shfl_xor_sync(0xffffffffu, sl2, off);
            }
            rms_c = sqrt(sc2 / kp.M); rms_L = sqrt(sl2 / kp.M);
        }
        bool go = true;
        if (kp.max_steps <= 0) { status = ST_MAXSTEPS; go = false; }
        if (go) go = kinetics();
        if (lane == 0) {
            s_go = go;
            s_sample = go && (landing || (steps_mode && kp.n_steps == 1));
        }
    }
    __syncthreads();   // bar2 (prologue)

    const bool vl = kp.limiter == LIM_VANLEER;
    while (s_go) {
        const double C = s_C, kap = s_kap, beta = s_beta;
        const bool sample = s_sample;
        double Cd[PP];
#pragma unroll
        for (int p = 0; p < PP; ++p) Cd[p] = (p < P) ? s_Cd[p] : 0.0;

        bool bad;
        if (C >= 0.0) bad = sweep_bins<P, K, false>(x, s_halo, NT, tid, C, kap, beta, Cd, vl, i0, N, clip_thr);
        else          bad = sweep_bins<P, K, true>(x, s_halo, NT, tid, C, kap, beta, Cd, vl, i0, N, clip_thr);
        if (bad) s_bad = 1;
        moment_partials(3, V);                   // mu3 of n and every tangent lane
        if (sample) {
#pragma unroll 1
            for (int km = 0; km < 3; ++km) moment_partials(km, V);
        }
        __syncthreads();   // bar1
        publish_halo();

        // ---- scalar phase (warp 0) -------------------------------------------------------
        if (warp == 0) {
            double tot[4] = {0.0, 0.0, 0.0, 0.0}, totd[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int km = 0; km < 4; ++km) {
                if (km == 3 || sample) {
                    double a = 0.0, b = 0.0;
                    for (int w = 0; w < NW; ++w) {
                        a += s_red[w][km][0];
                        if (pl >= 0) b += s_red[w][km][1 + pl];
                    }
                    tot[km] = a; totd[km] = b;
                }
            }
            const D1 mu3n = mk(tot[3], totd[3]);
            const D1 cn = c - kp.rho_kv * (mu3n - mu3p);          // eq-discrete_mass_balance
            bool go = true;
            if (s_bad) { status = ST_NEG; go = false; }
            else if (cn.v < 0.0) { status = ST_INFEAS; go = false; }
            else {
                c = cn; mu3p = mu3n;
                t = landing ? mk(kp.t_samples[m], 0.0) : t + dt;
                ++nstep;
                if (sample) {
                    const int mr = steps_mode ? 0 : m;
                    double* r = kp.rec + ((size_t)s * kp.M + mr) * 6;
                    if (lane == 0) { r[0] = t.v; r[1] = c.v; r[2] = tot[0]; r[3] = tot[1]; r[4] = tot[2]; r[5] = tot[3]; }
                    if (pl >= 0) {
                        double* rt = kp.trec + (((size_t)s * kp.M + mr) * kp.P + pl) * 5;
                        rt[0] = c.d; rt[1] = totd[0]; rt[2] = totd[1]; rt[3] = totd[2]; rt[4] = totd[3];
                    }
                    if (has_target) {
                        const double Lb = tot[1] / tot[0];
                        const double Lbd = (totd[1] * tot[0] - tot[1] * totd[0]) / (tot[0] * tot[0]);
                        const double rc = (c.v - tgt[2 * mr]) / rms_c, rL = (Lb - tgt[2 * mr + 1]) / rms_L;
                        loss += rc * rc + rL * rL;
                        gacc += 2.0 * (rc / rms_c) * c.d + 2.0 * (rL / rms_L) * Lbd;
                    }
                }
                if (landing) ++m;
                if (steps_mode ? (nstep >= kp.n_steps) : (m >= kp.M)) go = false;
                else if (nstep >= kp.max_steps) { status = ST_MAXSTEPS; go = false; }
                else go = kinetics();
            }
            __syncwarp();
            if (lane == 0) {
                s_bad = 0;
                s_go = go;
                s_sample = go && (landing || (steps_mode && nstep + 1 == kp.n_steps));
            }
        }
        __syncthreads();   // bar2
    }

    // ---- epilogue -----------------------------------------------------------------------
    if (kp.n_final) {
#pragma unroll
        for (int k = 0; k < K; ++k) { const int i = i0 + k; if (i < N) kp.n_final[(size_t)s * N + i] = x[0][k]; }
    }
    if (kp.ndot_final) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            if (p < kp.P) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int i = i0 + k;
                    if (i < N) kp.ndot_final[((size_t)s * kp.P + p) * N + i] = x[1 + p][k];
                }
            }
        }
    }
    if (warp == 0) {
        const bool ok = (status == ST_OK);
        const double qnan = __longlong_as_double(0x7ff8000000000000ll);
        if (lane == 0) {
            kp.status[s] = status;
            kp.steps[s] = nstep;
            if (kp.loss) kp.loss[s] = (has_target && ok) ? loss : qnan;
        }
        if (pl >= 0 && kp.grad) kp.grad[(size_t)s * kp.P + pl] = (has_target && ok) ? gacc : qnan;
    }
}

}  // namespace pbe
