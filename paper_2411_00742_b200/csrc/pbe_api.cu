// =====================================================================================
//  pbe_api.cu — host side of libpbe: the C ABI declared in include/pbe.h.
//  Validation, context-owned device memory, stream-ordered launches, kernel dispatch
//  by (N, tangent lanes).  No computation of the method happens here: every step of
//  the march runs in the CUDA kernels (k_resident.cuh incl. its cluster mode, k_resident_ws.cuh, k_stream.cuh,
//  k_stream_tb.cuh, k_2d_fused.cuh, k_2d.cuh, k_adjoint.cuh).
// =====================================================================================
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pbe.h"
#include "pbe_device.cuh"
#include "k_resident.cuh"
#include "k_resident_ws.cuh"
#include "k_stream.cuh"
#include "k_2d.cuh"
#include "k_2d_fused.cuh"
#include "k_adjoint.cuh"
#include "k_stream_tb.cuh"

using pbe::KParams;

namespace {

thread_local std::string g_create_error;

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t b) {
        if (b <= bytes && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr; bytes = 0;
        if (b == 0) return cudaSuccess;
        cudaError_t e = cudaMalloc(&p, b);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
    void release() { if (p) cudaFree(p); p = nullptr; bytes = 0; }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

}  // namespace

struct pbe_ctx_s {
    pbe_config cfg{};
    int device = 0;
    std::string err;
    // kinetics
    bool have_kin = false;
    int law = 0, n_params = 0, kin_sims = 0, sol_kind = 0, n_sol = 0, n_knots = 0;
    bool knotT_per_sim = false;
    DevBuf theta, sol, knot_t, knot_T, seed;
    // run inputs
    DevBuf c0, tsamp, target, n0_staged;
    // outputs
    DevBuf rec, trec, status, steps, loss, grad;
    // streaming-kernel scratch (allocated on first use)
    DevBuf sbuf, spart, sbar, sfinal, snscale, sdyn;
    // adjoint (NEXT-3) scratch: step trace, checkpoints, segment states, dL/dtheta
    DevBuf atr, ack, aseg, agrad;
    bool last_adjoint = false;
    // last run
    bool have_run = false;
    int last_sims = 0;
    cudaStream_t last_stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    pbe_run_info info{};
    int group_max = 8;       // max tangent lanes per resident CTA (env PBE_LANES_PER_CTA)
    bool cluster2 = false;   // env PBE_CLUSTER2: 2-CTA clusters at 2 CTAs/SM for small N
    int resident_k = 0;      // env PBE_RESIDENT_K: preferred bins per thread (0 = heuristic)
    bool ws = true;          // env PBE_WS=0: lockstep k_resident instead of k_resident_ws for P >= 1
    int ws_variant = 0;      // env PBE_WS_VARIANT: k_resident_ws tuning variant (A/B only)
    bool ws_tail = true;     // env PBE_WS_TAIL=0: no half-lane CTAs for the last partial wave
    bool stream_static = false;   // env PBE_STREAM_STATIC=1: k_stream with static tile ranges (A/B)
    bool temporal_block = true;  // NEXT-4 temporal blocking for uncapped-CFL steps mode in
                                 // k_stream (1.27x plain streaming on 64 x 1e6); env
                                 // PBE_TEMPORAL_BLOCK=0 selects plain streaming
    bool unfused_2d = false;     // env PBE_2D_UNFUSED=1: two-sweep k_2d instead of k_2d_fused
};

static pbe_status fail(pbe_ctx ctx, pbe_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf; else g_create_error = buf;
    return st;
}

#define CUDA_TRY(ctx, call)                                                                  \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? PBE_ERR_NOMEM : PBE_ERR_CUDA, \
                        "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

// ------------------------------------------------------------------------------------
// Kernel dispatch table for k_resident<P, K, MAXT>
// ------------------------------------------------------------------------------------
namespace {

using KernelFn = void (*)(const KParams);

struct ResidentVariant {
    int P, K, maxt;
    KernelFn fn;
};
// dynamic smem: halo (2 parities); the scalar state (WarpPart, LanePart) and the kinetics
// tables are static shared arrays (<= 48 KB), accounted for by the 200 KB dynamic cap below
size_t resident_smem(const ResidentVariant& v, int nt) {
    return (size_t)2 * 4 * (1 + v.P) * (nt + 2) * sizeof(double)      // halo, 2 parities
           + (size_t)v.K * nt * sizeof(double);                        // mu3 weights [K][NT]
}

// k_resident_ws<P, K, NT>: scalar chain off the critical path (a scalar warp runs the next step's
// kinetics while NT - 32 bin threads sweep the tangent lanes), P >= 1 lanes
struct WsVariant {
    int P, K, nt;
    KernelFn fn;
    bool xs;
    int tag;              // A/B tuning variant (PBE_WS_VARIANT); 0 = default
    int bins() const { return (nt - 32) * K; }
    size_t smem() const { return pbe::ws_smem_doubles(P, K, nt - 32, xs) * sizeof(double); }
};
#define WV(P, K, T) WsVariant{P, K, T, &pbe::k_resident_ws<P, K, T, false, false, 0>, false, 0}
#define WVX(P, K, T, XS, HALF, LAG, TAG) WsVariant{P, K, T, &pbe::k_resident_ws<P, K, T, XS, HALF, LAG>, XS, TAG}
const WsVariant kResidentWS[] = {
    WV(8, 9, 64), WV(8, 9, 128), WV(8, 9, 256), WV(4, 9, 64), WV(4, 9, 128), WV(4, 9, 256),
    WVX(8, 9, 256, true, false, 2, 1), WVX(8, 9, 256, true, true, 2, 2), WVX(8, 9, 256, true, false, 0, 3),
    WVX(8, 9, 256, true, true, 0, 4), WVX(8, 9, 256, false, true, 2, 5), WVX(8, 9, 256, false, false, 2, 6),
};
#undef WVX
#undef WV

#define RV(P, K, T) ResidentVariant{P, K, T, &pbe::k_resident<P, K, T>}
const ResidentVariant kResident[] = {
    RV(0, 2, 512), RV(0, 4, 512), RV(0, 8, 512), RV(0, 16, 512), RV(0, 32, 256),
    RV(2, 2, 512), RV(2, 4, 512), RV(2, 8, 512), RV(2, 16, 256),
    RV(4, 2, 512), RV(4, 4, 512), RV(4, 8, 256),
    RV(5, 2, 512), RV(5, 4, 512), RV(5, 8, 256),
    RV(8, 2, 256), RV(8, 4, 256), RV(8, 8, 256),
};
#undef RV

// k_resident<P, K, MAXT, true> cluster variants (cluster size chosen at launch, <= 16)
#define CV(P, K, T) ResidentVariant{P, K, T, &pbe::k_resident<P, K, T, true>}
// 2 CTAs per SM (<= 128 registers/thread): a simulation split over a 2-CTA cluster keeps 16
// warps per SM in two independent barrier domains (PBE_CLUSTER2=1 selects it for N <= 2048)
const ResidentVariant kCluster2[] = {
    ResidentVariant{8, 4, 256, &pbe::k_resident<8, 4, 256, true, 2>},
    ResidentVariant{4, 4, 256, &pbe::k_resident<4, 4, 256, true, 2>},
    ResidentVariant{0, 4, 256, &pbe::k_resident<0, 4, 256, true, 2>},
};
const ResidentVariant kCluster[] = {
    CV(0, 8, 512), CV(0, 16, 512),
    CV(2, 4, 512), CV(2, 8, 512),
    CV(4, 4, 512), CV(4, 8, 256),
    CV(8, 4, 256), CV(8, 8, 256),
};
#undef CV
// smallest cluster (then smallest K) whose CTAs cover N bins
const ResidentVariant* pick_cluster(int N, int P, int* cs) {
    const int Pi = P == 0 ? 0 : (P <= 2 ? 2 : (P <= 4 ? 4 : (P <= 8 ? 8 : -1)));
    for (int c = 2; c <= 16; c *= 2) {
        const ResidentVariant* best = nullptr;
        for (const auto& v : kCluster) {
            if (v.P != Pi) continue;
            if ((long long)v.K * v.maxt * c < N) continue;
            if (!best || v.K < best->K) best = &v;
        }
        if (best) { *cs = c; return best; }
    }
    return nullptr;
}

// k_stream<P> variants: lanes per launch (the tangent lanes of a simulation are never split)
struct StreamVariant {
    int P;
    const void* fn;          // k_stream<P, true>: dynamic tile schedule
    const void* fn_static;   // k_stream<P, false>: static tile ranges (PBE_STREAM_STATIC=1, A/B)
    void (*load)(const double*, long long, int, int, double*, long long, unsigned long long*, int, int, double*,
                 double, double);
    void (*store)(const double*, const double*, const int*, int, int, long long, double*, double*);
};
#define SV(P) StreamVariant{P, (const void*)&pbe::k_stream<P, true>, (const void*)&pbe::k_stream<P, false>, \
                            &pbe::k_stream_load<1 + P>, &pbe::k_stream_store<1 + P>}
const StreamVariant kStream[] = {SV(0), SV(2), SV(4)};
#undef SV
const StreamVariant* pick_stream(int P) {
    for (const auto& v : kStream)
        if (v.P >= P) return &v;
    return nullptr;
}

// Tangent lanes per CTA.  More than `group_max` lanes are split into lane groups (one CTA
// each, primal recomputed): fewer registers per thread -> 16 warps per SM instead of 8.
int lanes_per_cta(int P, int group_max) {
    if (P == 0) return 0;
    if (P <= 2) return 2;
    if (P <= 4) return 4;
    if (group_max >= 8 && P <= 8) return 8;
    if (P <= 8) return 4;          // 2 groups of 4
    return 5;                      // 9..10 lanes: 2 groups of 5
}

// static shared memory of a kernel (cached per function by the runtime)
size_t static_smem(KernelFn fn) {
    cudaFuncAttributes a{};
    return cudaFuncGetAttributes(&a, (const void*)fn) == cudaSuccess ? a.sharedSizeBytes : 48 * 1024;
}

// Resident variant for N bins: one simulation alone wants the smallest K (most warps); a
// batch wants small CTAs so several simulations share an SM and hide each other's per-step
// latency (K_pref from PBE_RESIDENT_K or the heuristic in pbe_run_batch).
const ResidentVariant* pick_resident(int N, int P, int group_max, int* groups, int k_pref = 0) {
    const int Pi = lanes_per_cta(P, group_max);
    *groups = Pi ? (P + Pi - 1) / Pi : 1;
    const ResidentVariant* best = nullptr;
    for (const auto& v : kResident) {
        if (v.P != Pi) continue;
        if ((long long)v.K * v.maxt < N) continue;
        const int nt = ((N + v.K - 1) / v.K + 31) / 32 * 32;
        if (resident_smem(v, nt) + static_smem(v.fn) > 227 * 1024) continue;   // dynamic + static per CTA
        if (!best) { best = &v; continue; }
        const bool closer = k_pref ? (abs(v.K - k_pref) < abs(best->K - k_pref) ||
                                      (abs(v.K - k_pref) == abs(best->K - k_pref) && v.K < best->K))
                                   : v.K < best->K;
        if (closer) best = &v;
    }
    return best;
}

// scalar-chain-overlapped variant for P tangent lanes (lanes_per_cta(P) exactly: no idle lane
// padding) and N bins: the fewest threads that cover N
const WsVariant* pick_ws(int N, int P, int tag) {
    const WsVariant* best = nullptr;
    for (const auto& v : kResidentWS) {
        if (v.tag != tag) continue;
        if (v.P != lanes_per_cta(P, 8) || v.bins() < N) continue;
        if (v.smem() + static_smem(v.fn) > 227 * 1024) continue;
        if (!best || v.nt < best->nt) best = &v;
    }
    return best;
}

}  // namespace

// ------------------------------------------------------------------------------------
// k_stream launch: padded ping-pong state in ctx scratch, load kernel, one cooperative
// launch for the whole march, store kernel for n_final / ndot_final.
// ------------------------------------------------------------------------------------
static pbe_status launch_stream(pbe_ctx ctx, const StreamVariant& sv, KParams kp, int S, const double* n0,
                                long long n0_stride, cudaStream_t st) {
    const int N = kp.N, V = 1 + sv.P;
    const long long pitch = ((long long)N + 4 + 3) / 4 * 4;
    int dev = ctx->device, sms = 0;
    CUDA_TRY(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // tile size depends on N and V only (batch-independent partial-sum order)
    const int TB = pbe::stream_tile(N, V);
    const int stages = V == 1 ? pbe::StreamCfg<1>::STAGES : pbe::StreamCfg<3>::STAGES;
    const size_t smem = (size_t)stages * V * (TB + 4) * sizeof(double);
    const bool dyn = !ctx->stream_static;
    const void* fn = dyn ? sv.fn : sv.fn_static;
    CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, pbe::STREAM_NT, smem));
    if (per_sm < 1) return fail(ctx, PBE_ERR_CUDA, "k_stream does not fit on an SM (smem %zu)", smem);
    const int cap_sm = V == 1 && pbe::StreamCfg<1>::MINB > 2 ? pbe::StreamCfg<1>::MINB : 2;
    per_sm = per_sm > cap_sm ? cap_sm : per_sm;
    const int G = per_sm * sms;
    const int T_sim = (N + TB - 1) / TB;
    const long long n_tiles = (long long)S * T_sim;
    const long long chunk = (n_tiles + G - 1) / G;
    if (dyn ? (S + G - 1) / G > pbe::STREAM_MAXS : (chunk + T_sim - 1) / T_sim + 1 > pbe::STREAM_MAXS)
        return fail(ctx, PBE_ERR_ARG, "too many simulations per CTA for the streaming kernel (S = %d, N = %d)", S, N);

    const size_t buf_el = (size_t)S * V * pitch;
    CUDA_TRY(ctx, ctx->sbuf.ensure(2 * buf_el * sizeof(double)));
    CUDA_TRY(ctx, ctx->spart.ensure((size_t)S * T_sim * pbe::STREAM_NWC * 5 * V * sizeof(double)));
    CUDA_TRY(ctx, ctx->sbar.ensure(8 * sizeof(unsigned)));
    CUDA_TRY(ctx, ctx->sfinal.ensure((size_t)S * sizeof(int)));
    CUDA_TRY(ctx, ctx->snscale.ensure((size_t)S * sizeof(unsigned long long)));
    // dynamic schedule: [4] tile counters, [S] coefficient steps, then [S] coefficients (16-B aligned)
    CUDA_TRY(ctx, ctx->sdyn.ensure((4 + (size_t)S) * sizeof(unsigned) + 16 + (size_t)S * 16 * sizeof(double)));
    double* b0 = ctx->sbuf.as<double>();
    double* b1 = b0 + buf_el;
    // ghosts and padding must be zero in both buffers (only interior bins are ever written)
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->sbuf.p, 0, 2 * buf_el * sizeof(double), st));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->sbar.p, 0, 8 * sizeof(unsigned), st));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->snscale.p, 0, (size_t)S * sizeof(unsigned long long), st));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->sdyn.p, 0, 4 * sizeof(unsigned), st));                  // tile counters
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->sdyn.as<unsigned>() + 4, 0xff, (size_t)S * sizeof(unsigned), st));  // no step yet
    sv.load<<<dim3(T_sim, S), 256, 0, st>>>(n0, n0_stride, N, S, b0, pitch, ctx->snscale.as<unsigned long long>(),
                                            TB, T_sim, ctx->spart.as<double>(), kp.L_lo, kp.dL);
    CUDA_TRY(ctx, cudaGetLastError());
    const dim3 lg((N + 255) / 256 < 64 ? (N + 255) / 256 : 64, S);

    pbe::StreamParams sp{};
    sp.kp = kp;
    sp.buf0 = b0; sp.buf1 = b1; sp.pitch = pitch; sp.TB = TB; sp.T_sim = T_sim; sp.n_tiles = n_tiles;
    sp.part = ctx->spart.as<double>();
    sp.bar = ctx->sbar.as<unsigned>();
    sp.active = reinterpret_cast<int*>(ctx->sbar.as<unsigned>() + 4);
    sp.final_buf = ctx->sfinal.as<int>();
    sp.nscale_bits = ctx->snscale.as<unsigned long long>();
    sp.tile_ctr = ctx->sdyn.as<unsigned>();
    sp.coef_step = ctx->sdyn.as<unsigned>() + 4;
    sp.coef = reinterpret_cast<char*>(ctx->sdyn.p) + (((4 + (size_t)S) * sizeof(unsigned) + 15) / 16) * 16;
    void* args[] = {&sp};
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
    CUDA_TRY(ctx, cudaLaunchCooperativeKernel(fn, dim3(G), dim3(pbe::STREAM_NT), args, smem, st));
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
    int launches = 2;
    if (kp.n_final || kp.ndot_final) {
        sv.store<<<lg, 256, 0, st>>>(b0, b1, sp.final_buf, N, kp.P, pitch, kp.n_final, kp.ndot_final);
        CUDA_TRY(ctx, cudaGetLastError());
        ++launches;
    }
    ctx->info.kernel = PBE_KERNEL_STREAM;
    ctx->info.launches = launches;
    ctx->info.threads_per_cta = pbe::STREAM_NT;
    ctx->info.ctas = G;
    ctx->info.cluster = 1;
    ctx->info.bins_per_thread = 0;
    return PBE_OK;
}

// ------------------------------------------------------------------------------------
// k_stream_tb launch (NEXT-4): temporal blocking of uncapped CFL steps (steps mode, primal)
// ------------------------------------------------------------------------------------
static pbe_status launch_stream_tb(pbe_ctx ctx, KParams kp, int S, const double* n0, long long n0_stride,
                                   double* n_final, cudaStream_t st) {
    const int N = kp.N;
    int TB = pbe::stream_tb_tile(N);
    if (const char* e = getenv("PBE_TB_TILE")) {           // A/B only: 512, 1024 or 2048
        const int v = atoi(e);
        if (v == 512 || v == 1024 || v == 2048) TB = v;
    }
    const int T_sim = (N + TB - 1) / TB;
    const long long pitch = ((long long)T_sim * TB + 2 * pbe::TB_GH + 3) / 4 * 4;
    int sms = 0, per_sm = 0;
    CUDA_TRY(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    const int WL = TB + 2 * pbe::TB_GH;
    const size_t smem = (size_t)(pbe::TB_STAGES + 2) * WL * sizeof(double);
    CUDA_TRY(ctx, cudaFuncSetAttribute((const void*)pbe::k_stream_tb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pbe::k_stream_tb, pbe::TB_NT, smem));
    if (per_sm < 1) return fail(ctx, PBE_ERR_CUDA, "k_stream_tb does not fit on an SM (smem %zu)", smem);
    per_sm = per_sm > 2 ? 2 : per_sm;
    const int G = per_sm * sms;
    const long long n_tiles = (long long)S * T_sim;
    const long long chunk = (n_tiles + G - 1) / G;
    if ((chunk + T_sim - 1) / T_sim + 1 > pbe::STREAM_MAXS)
        return fail(ctx, PBE_ERR_ARG, "too many simulations per CTA for the streaming kernel (S = %d, N = %d)", S, N);
    const size_t buf_el = (size_t)S * pitch;
    CUDA_TRY(ctx, ctx->sbuf.ensure(2 * buf_el * sizeof(double)));
    CUDA_TRY(ctx, ctx->spart.ensure((size_t)S * T_sim * pbe::TB_NWC * pbe::TB_KB * 5 * sizeof(double)));
    CUDA_TRY(ctx, ctx->sbar.ensure(8 * sizeof(unsigned)));
    CUDA_TRY(ctx, ctx->sfinal.ensure((size_t)S * sizeof(int)));
    CUDA_TRY(ctx, ctx->snscale.ensure((size_t)S * sizeof(unsigned long long)));
    double* b0 = ctx->sbuf.as<double>();
    double* b1 = b0 + buf_el;
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->sbuf.p, 0, 2 * buf_el * sizeof(double), st));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->sbar.p, 0, 8 * sizeof(unsigned), st));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->snscale.p, 0, (size_t)S * sizeof(unsigned long long), st));
    pbe::k_stream_tb_load<<<dim3(T_sim, S), 256, 0, st>>>(n0, n0_stride, N, b0, pitch, ctx->snscale.as<unsigned long long>(),
                                                          TB, T_sim, ctx->spart.as<double>(), kp.L_lo, kp.dL);
    CUDA_TRY(ctx, cudaGetLastError());
    pbe::StreamTBParams sp{};
    sp.kp = kp;
    sp.buf0 = b0; sp.buf1 = b1; sp.pitch = pitch; sp.TB = TB; sp.T_sim = T_sim; sp.n_tiles = n_tiles;
    sp.part = ctx->spart.as<double>();
    sp.bar = ctx->sbar.as<unsigned>();
    sp.active = reinterpret_cast<int*>(ctx->sbar.as<unsigned>() + 4);
    sp.final_buf = ctx->sfinal.as<int>();
    sp.nscale_bits = ctx->snscale.as<unsigned long long>();
    void* args[] = {&sp};
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
    CUDA_TRY(ctx, cudaLaunchCooperativeKernel((const void*)pbe::k_stream_tb, dim3(G), dim3(pbe::TB_NT), args, smem, st));
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
    int launches = 2;
    if (n_final) {
        const dim3 lg((N + 255) / 256 < 64 ? (N + 255) / 256 : 64, S);
        pbe::k_stream_tb_store<<<lg, 256, 0, st>>>(b0, b1, sp.final_buf, N, pitch, n_final);
        CUDA_TRY(ctx, cudaGetLastError());
        ++launches;
    }
    ctx->info.kernel = PBE_KERNEL_STREAM;
    ctx->info.launches = launches;
    ctx->info.threads_per_cta = pbe::TB_NT;
    ctx->info.ctas = G;
    ctx->info.cluster = 1;
    ctx->info.bins_per_thread = 0;
    ctx->info.steps_per_pass = pbe::TB_KB;
    return PBE_OK;
}

// ------------------------------------------------------------------------------------
// k_2d launch (NEXT-1): padded ping-pong planes, load kernel (+ mu12 partials), one
// cooperative launch for the whole 2D march, store kernel for n_final.
// ------------------------------------------------------------------------------------
static pbe_status launch_2d(pbe_ctx ctx, KParams kp, int S, const double* f0, long long f0_stride,
                            double* f_final, cudaStream_t st) {
    const pbe_config& cf = ctx->cfg;
    const int N1 = cf.n_bins, N2 = cf.n_bins2;
    const long long P1 = 4LL * ((N1 + 3) / 4) + 4, R2 = 4LL * ((N2 + 3) / 4) + 4;
    int sms = 0, per_sm = 0;
    CUDA_TRY(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pbe::k_2d, pbe::K2D_NT, 0));
    if (per_sm < 1) return fail(ctx, PBE_ERR_CUDA, "k_2d does not fit on an SM");
    per_sm = per_sm > 4 ? 4 : per_sm;
    const unsigned G = (unsigned)(per_sm * sms);
    const size_t plane = (size_t)R2 * P1, buf = (size_t)S * plane;
    CUDA_TRY(ctx, ctx->sbuf.ensure(2 * buf * sizeof(double)));
    CUDA_TRY(ctx, ctx->spart.ensure((size_t)S * G * 7 * sizeof(double)));
    CUDA_TRY(ctx, ctx->sbar.ensure(8 * sizeof(unsigned)));
    CUDA_TRY(ctx, ctx->snscale.ensure((size_t)S * sizeof(unsigned long long)));
    double* A = ctx->sbuf.as<double>();
    double* B = A + buf;
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->sbuf.p, 0, 2 * buf * sizeof(double), st));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->sbar.p, 0, 8 * sizeof(unsigned), st));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->snscale.p, 0, (size_t)S * sizeof(unsigned long long), st));
    pbe::k_2d_load<<<dim3(G, S), pbe::K2D_NT, 0, st>>>(f0, f0_stride, S, N1, N2, A, P1, R2, ctx->spart.as<double>(), G,
                                                       ctx->snscale.as<unsigned long long>(), cf.L_lo, cf.dL, cf.L2_lo,
                                                       cf.dL2);
    CUDA_TRY(ctx, cudaGetLastError());
    pbe::Params2D p2{};
    p2.kp = kp;
    p2.N2 = N2; p2.L2_lo = cf.L2_lo; p2.dL2 = cf.dL2; p2.inv_dL2 = 1.0 / cf.dL2;
    p2.A = A; p2.B = B; p2.P1 = P1; p2.R2 = R2;
    p2.part = ctx->spart.as<double>();
    p2.bar = ctx->sbar.as<unsigned>();
    p2.nscale_bits = ctx->snscale.as<unsigned long long>();
    void* args[] = {&p2};
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
    CUDA_TRY(ctx, cudaLaunchCooperativeKernel((const void*)pbe::k_2d, dim3(G), dim3(pbe::K2D_NT), args, 0, st));
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
    int launches = 2;
    if (f_final) {
        pbe::k_2d_store<<<2 * sms, 256, 0, st>>>(A, S, N1, N2, P1, R2, f_final);
        CUDA_TRY(ctx, cudaGetLastError());
        ++launches;
    }
    ctx->info.kernel = PBE_KERNEL_2D;
    ctx->info.launches = launches;
    ctx->info.threads_per_cta = pbe::K2D_NT;
    ctx->info.ctas = (int)G;
    ctx->info.cluster = 1;
    ctx->info.bins_per_thread = pbe::K2D_K;
    return PBE_OK;
}

// ------------------------------------------------------------------------------------
// k_2d_fused launch (NEXT-1, default): both sweeps of a split step per HBM pass, warp strips
// of 28 columns x 32 rows, 8 strips per tile/CTA; planes padded to whole tiles + ghost cells.
// ------------------------------------------------------------------------------------
static pbe_status launch_2d_fused(pbe_ctx ctx, KParams kp, int S, const double* f0, long long f0_stride,
                                  double* f_final, cudaStream_t st) {
    const pbe_config& cf = ctx->cfg;
    const int N1 = cf.n_bins, N2 = cf.n_bins2;
    const int NTX = (N1 + pbe::F2_TXC - 1) / pbe::F2_TXC, NTY = (N2 + pbe::F2_H - 1) / pbe::F2_H;
    const long long P1 = (long long)NTX * pbe::F2_TXC + 8, R2 = (long long)NTY * pbe::F2_H + 4;
    const int T2 = NTX * NTY;
    const size_t smem = 0;
    int sms = 0, per_sm = 0;
    CUDA_TRY(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pbe::k_2d_fused, pbe::F2_NT, smem));
    if (per_sm < 1) return fail(ctx, PBE_ERR_CUDA, "k_2d_fused does not fit on an SM");
    unsigned G = (unsigned)(per_sm * sms);
    if ((long long)G > (long long)S * T2) G = (unsigned)((long long)S * T2);   // no idle CTAs
    const size_t plane = (size_t)R2 * P1, buf = (size_t)S * plane;
    CUDA_TRY(ctx, ctx->sbuf.ensure(2 * buf * sizeof(double)));
    CUDA_TRY(ctx, ctx->spart.ensure(((size_t)S * T2 * 7 + (size_t)S * 8) * sizeof(double)));
    CUDA_TRY(ctx, ctx->sbar.ensure(8 * sizeof(unsigned)));
    CUDA_TRY(ctx, ctx->sfinal.ensure((size_t)2 * S * sizeof(int)));
    CUDA_TRY(ctx, ctx->snscale.ensure((size_t)S * sizeof(unsigned long long)));
    double* A = ctx->sbuf.as<double>();
    double* B = A + buf;
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->sbuf.p, 0, 2 * buf * sizeof(double), st));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->sbar.p, 0, 8 * sizeof(unsigned), st));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->sfinal.p, 0, (size_t)2 * S * sizeof(int), st));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->snscale.p, 0, (size_t)S * sizeof(unsigned long long), st));
    pbe::k_2d_fused_load<<<dim3(T2, S), 256, 0, st>>>(f0, f0_stride, N1, N2, A, P1, R2, NTX, ctx->spart.as<double>(),
                                                      ctx->snscale.as<unsigned long long>(), cf.L_lo, cf.dL, cf.L2_lo,
                                                      cf.dL2);
    CUDA_TRY(ctx, cudaGetLastError());
    pbe::Params2DF p{};
    p.kp = kp;
    p.N2 = N2; p.L2_lo = cf.L2_lo; p.dL2 = cf.dL2; p.inv_dL2 = 1.0 / cf.dL2;
    p.A = A; p.B = B; p.P1 = P1; p.R2 = R2; p.NTX = NTX; p.NTY = NTY;
    p.part = ctx->spart.as<double>();
    p.bar = ctx->sbar.as<unsigned>();
    p.nscale_bits = ctx->snscale.as<unsigned long long>();
    p.final_buf = ctx->sfinal.as<int>();
    p.cnt = reinterpret_cast<unsigned*>(ctx->sfinal.as<int>() + S);
    p.tot = ctx->spart.as<double>() + (size_t)S * T2 * 7;
    p.work = ctx->sbar.as<unsigned>() + 6;
    void* args[] = {&p};
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
    CUDA_TRY(ctx, cudaLaunchCooperativeKernel((const void*)pbe::k_2d_fused, dim3(G), dim3(pbe::F2_NT), args, smem, st));
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
    int launches = 2;
    if (f_final) {
        pbe::k_2d_fused_store<<<2 * sms, 256, 0, st>>>(A, B, p.final_buf, S, N1, N2, P1, R2, f_final);
        CUDA_TRY(ctx, cudaGetLastError());
        ++launches;
    }
    ctx->info.kernel = PBE_KERNEL_2D;
    ctx->info.launches = launches;
    ctx->info.threads_per_cta = pbe::F2_NT;
    ctx->info.ctas = (int)G;
    ctx->info.cluster = 1;
    ctx->info.bins_per_thread = pbe::K2D_K;
    return PBE_OK;
}

// ------------------------------------------------------------------------------------
// Run set-up shared by pbe_run_batch and pbe_run_adjoint
// ------------------------------------------------------------------------------------
// Argument checks (synchronous PBE_ERR_ARG).
static pbe_status validate_run(pbe_ctx ctx, int32_t n_sims, const double* n0, int64_t n0_stride,
                               int32_t n0_on_device, const double* c0, const double* t_samples,
                               const double* ndot_final) {
    if (!ctx) return fail(nullptr, PBE_ERR_ARG, "NULL context");
    if (!ctx->have_kin) return fail(ctx, PBE_ERR_STATE, "pbe_set_kinetics must precede pbe_run_batch");
    const pbe_config& cf = ctx->cfg;
    const int N = cf.n_bins, M = cf.n_samples, P = cf.n_tangents;
    const bool steps_mode = cf.n_steps > 0;
    if (n_sims < 1 || n_sims > cf.max_sims) return fail(ctx, PBE_ERR_ARG, "n_sims must be in [1, max_sims]");
    if (n_sims != ctx->kin_sims) return fail(ctx, PBE_ERR_ARG, "n_sims (%d) != kinetics n_sims (%d)", n_sims, ctx->kin_sims);
    if (!n0 || !c0) return fail(ctx, PBE_ERR_ARG, "NULL n0 or c0");
    const bool two_d = cf.n_bins2 > 0;
    const long long cells = (long long)N * (two_d ? cf.n_bins2 : 1);
    if (n0_stride != 0 && n0_stride != cells) return fail(ctx, PBE_ERR_ARG, "n0_stride must be 0 or the cells per simulation");
    if (!steps_mode && !t_samples) return fail(ctx, PBE_ERR_ARG, "NULL t_samples");
    for (int s = 0; s < n_sims; ++s)
        if (!(c0[s] >= 0.0) || !std::isfinite(c0[s])) return fail(ctx, PBE_ERR_ARG, "c0[%d] must be finite and >= 0", s);
    if (!steps_mode) {
        if (!(t_samples[0] > 0.0)) return fail(ctx, PBE_ERR_ARG, "t_samples[0] must be > 0");
        for (int m = 1; m < M; ++m)
            if (!(t_samples[m] > t_samples[m - 1])) return fail(ctx, PBE_ERR_ARG, "t_samples must be strictly increasing");
        if (!std::isfinite(t_samples[M - 1])) return fail(ctx, PBE_ERR_ARG, "t_samples must be finite");
    }
    if (!n0_on_device) {
        const size_t rows = n0_stride ? (size_t)n_sims : 1;
        for (size_t j = 0; j < rows * (size_t)cells; ++j)
            if (!(n0[j] >= 0.0) || !std::isfinite(n0[j])) return fail(ctx, PBE_ERR_ARG, "n0[%zu] must be finite and >= 0", j);
    }
    if (ndot_final && P == 0) return fail(ctx, PBE_ERR_ARG, "ndot_final requires n_tangents > 0");
    (void)M;
    (void)two_d;
    return PBE_OK;
}

// Copies the run inputs on stream st (c0, sample times, target, host n0) and presets the
// records to NaN (unreached samples).  *n0_dev: device n0 (caller's or staged).
static pbe_status stage_run(pbe_ctx ctx, int32_t n_sims, const double* n0, int64_t n0_stride,
                            int32_t n0_on_device, const double* c0, const double* t_samples,
                            const double* target, cudaStream_t st, const double** n0_dev_out) {
    const pbe_config& cf = ctx->cfg;
    const int N = cf.n_bins, M = cf.n_samples, P = cf.n_tangents;
    const bool steps_mode = cf.n_steps > 0;
    const bool two_d = cf.n_bins2 > 0;
    const long long cells = (long long)N * (two_d ? cf.n_bins2 : 1);
    CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    // the ctx-owned input and output buffers are reused run after run: a run on another stream
    // waits for the previous run's kernel (ev1) before they are overwritten
    if (ctx->have_run && ctx->last_stream != st) CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->ev1, 0));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->c0.p, c0, n_sims * sizeof(double), cudaMemcpyHostToDevice, st));
    if (!steps_mode)
        CUDA_TRY(ctx, cudaMemcpyAsync(ctx->tsamp.p, t_samples, M * sizeof(double), cudaMemcpyHostToDevice, st));
    if (target) {
        CUDA_TRY(ctx, ctx->target.ensure((size_t)n_sims * M * 2 * sizeof(double)));
        CUDA_TRY(ctx, cudaMemcpyAsync(ctx->target.p, target, (size_t)n_sims * M * 2 * sizeof(double),
                                      cudaMemcpyHostToDevice, st));
    }
    const double* n0_dev = n0;
    if (!n0_on_device) {
        const size_t bytes = (n0_stride ? (size_t)n_sims : 1) * (size_t)cells * sizeof(double);
        CUDA_TRY(ctx, ctx->n0_staged.ensure(bytes));
        CUDA_TRY(ctx, cudaMemcpyAsync(ctx->n0_staged.p, n0, bytes, cudaMemcpyHostToDevice, st));
        n0_dev = ctx->n0_staged.as<double>();
    }
    // unreached samples read as NaN (all-ones bytes)
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->rec.p, 0xff, (size_t)n_sims * M * (two_d ? 8 : 6) * sizeof(double), st));
    if (P) CUDA_TRY(ctx, cudaMemsetAsync(ctx->trec.p, 0xff, (size_t)n_sims * M * P * 5 * sizeof(double), st));
    // loss reads NaN unless the kernel writes it (no target, 2D runs): never stale or uninitialised
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->loss.p, 0xff, (size_t)n_sims * sizeof(double), st));
    *n0_dev_out = n0_dev;
    return PBE_OK;
}

static KParams make_kparams(pbe_ctx ctx, int n_sims, const double* n0_dev, long long n0_stride,
                            const double* target, double* n_final, double* ndot_final, int groups) {
    const pbe_config& cf = ctx->cfg;
    const int N = cf.n_bins, M = cf.n_samples, P = cf.n_tangents;
    KParams kp{};
    kp.N = N; kp.L_lo = cf.L_lo; kp.dL = cf.dL; kp.inv_dL = 1.0 / cf.dL; kp.limiter = cf.limiter;
    kp.courant = cf.courant; kp.dt_fixed = cf.dt_fixed; kp.dt_max = cf.dt_max;
    kp.max_steps = cf.max_steps; kp.n_steps = cf.n_steps; kp.rho_kv = cf.rho_c * cf.k_v;
    kp.law = ctx->law; kp.n_params = ctx->n_params; kp.sol_kind = ctx->sol_kind; kp.n_sol = ctx->n_sol;
    kp.n_knots = ctx->n_knots; kp.knotT_stride = ctx->knotT_per_sim ? ctx->n_knots : 0;
    kp.theta = ctx->theta.as<double>(); kp.sol = ctx->sol.as<double>(); kp.knot_t = ctx->knot_t.as<double>();
    kp.knot_T = ctx->knot_T.as<double>(); kp.seed = ctx->seed.as<double>();
    kp.n_sims = n_sims; kp.M = M; kp.P = P; kp.G = groups;
    kp.n0 = n0_dev; kp.n0_stride = n0_stride; kp.c0 = ctx->c0.as<double>();
    kp.t_samples = ctx->tsamp.as<double>(); kp.target = target ? ctx->target.as<double>() : nullptr;
    kp.rec = ctx->rec.as<double>(); kp.trec = ctx->trec.as<double>(); kp.status = ctx->status.as<int>();
    kp.steps = ctx->steps.as<long long>(); kp.loss = ctx->loss.as<double>(); kp.grad = ctx->grad.as<double>();
    kp.n_final = n_final; kp.ndot_final = ndot_final;
    return kp;
}

// ------------------------------------------------------------------------------------
// k_adjoint launch (NEXT-3): one CTA per simulation; K from N (smem: 4 (NT K + 4) doubles)
// ------------------------------------------------------------------------------------
struct AdjointVariant { int K, ntb; const void* fn; };
const AdjointVariant kAdjoint[] = {
    {4, 256, (const void*)&pbe::k_adjoint<4>}, {8, 256, (const void*)&pbe::k_adjoint<8>},
    {4, 512, (const void*)&pbe::k_adjoint<4, 512>},   // PBE_ADJ_K=4 A/B only (N = 2000: 99 vs 87 ms)
    {16, 256, (const void*)&pbe::k_adjoint<16>}, {24, 256, (const void*)&pbe::k_adjoint<24>},
};
// cluster variants (trajectory mode): 64 threads x K bins per CTA, CS CTAs per simulation
const AdjointVariant kAdjointCL[] = {
    {2, 64, (const void*)&pbe::k_adjoint<2, 64, true>}, {4, 64, (const void*)&pbe::k_adjoint<4, 64, true>},
    {8, 64, (const void*)&pbe::k_adjoint<8, 64, true>},
};

// ------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------
extern "C" {

const char* pbe_version(void) { return "libpbe 0.1 (sm_100a)"; }

#if PBE_TIMING
// Diagnostics build only (tools/build_variant.py ... -DPBE_TIMING=1): cycle sums of the
// resident kernel's step phases measured by warp 0 of CTA 0.
int pbe_debug_phase_cycles(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, pbe::g_phase_cycles, sizeof(pbe::g_phase_cycles)) == cudaSuccess ? 0 : 1;
}
int pbe_debug_ws_cycles(unsigned long long* out) {       // [8], see k_resident_ws.cuh
    return cudaMemcpyFromSymbol(out, pbe::g_ws_cycles, sizeof(pbe::g_ws_cycles)) == cudaSuccess ? 0 : 1;
}
int pbe_debug_stream_cycles(unsigned long long* out) {    // [1024][5], see k_stream.cuh
    return cudaMemcpyFromSymbol(out, pbe::g_stream_cycles, sizeof(pbe::g_stream_cycles)) == cudaSuccess ? 0 : 1;
}
int pbe_debug_adjoint_cycles(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, pbe::g_adj_cycles, sizeof(pbe::g_adj_cycles)) == cudaSuccess ? 0 : 1;
}
#endif

const char* pbe_last_error(pbe_ctx ctx) { return ctx ? ctx->err.c_str() : g_create_error.c_str(); }

pbe_status pbe_create(const pbe_config* cfg, int device, pbe_ctx* out) {
    if (!cfg || !out) return fail(nullptr, PBE_ERR_ARG, "pbe_create: NULL cfg or out");
    *out = nullptr;
    const pbe_config& c = *cfg;
    if (c.n_bins < 3) return fail(nullptr, PBE_ERR_ARG, "n_bins must be >= 3 (got %d)", c.n_bins);
    if (!(c.dL > 0.0) || !std::isfinite(c.dL)) return fail(nullptr, PBE_ERR_ARG, "dL must be finite and > 0");
    if (!std::isfinite(c.L_lo)) return fail(nullptr, PBE_ERR_ARG, "L_lo must be finite");
    if (c.limiter < PBE_LIM_UPWIND || c.limiter > PBE_LIM_MC)
        return fail(nullptr, PBE_ERR_ARG, "unknown limiter %d", c.limiter);
    if (!(c.courant > 0.0 && c.courant <= 1.0)) return fail(nullptr, PBE_ERR_ARG, "courant must be in (0, 1]");
    if (!(c.dt_fixed >= 0.0) || !std::isfinite(c.dt_fixed)) return fail(nullptr, PBE_ERR_ARG, "dt_fixed must be >= 0");
    if (!(c.dt_max > 0.0)) return fail(nullptr, PBE_ERR_ARG, "dt_max must be > 0 (INFINITY for no cap)");
    if (c.max_steps <= 0) return fail(nullptr, PBE_ERR_ARG, "max_steps must be > 0");
    if (c.n_steps < 0) return fail(nullptr, PBE_ERR_ARG, "n_steps must be >= 0");
    if (!(c.rho_c > 0.0) || !(c.k_v > 0.0)) return fail(nullptr, PBE_ERR_ARG, "rho_c and k_v must be > 0");
    if (c.n_samples < 1) return fail(nullptr, PBE_ERR_ARG, "n_samples must be >= 1");
    if (c.n_steps > 0 && c.n_samples != 1) return fail(nullptr, PBE_ERR_ARG, "steps mode needs n_samples == 1");
    if (c.n_tangents < 0 || c.n_tangents > pbe::MAXP) return fail(nullptr, PBE_ERR_ARG, "n_tangents must be in [0, 10]");
    if (c.max_sims < 1) return fail(nullptr, PBE_ERR_ARG, "max_sims must be >= 1");
    if (c.kernel < PBE_KERNEL_AUTO || c.kernel > PBE_KERNEL_2D) return fail(nullptr, PBE_ERR_ARG, "unknown kernel %d", c.kernel);
    if (c.n_bins2 < 0) return fail(nullptr, PBE_ERR_ARG, "n_bins2 must be >= 0");
    if (c.n_bins2 > 0) {
        if (c.n_bins2 < 3) return fail(nullptr, PBE_ERR_ARG, "n_bins2 must be >= 3 in 2D mode");
        if (!(c.dL2 > 0.0) || !std::isfinite(c.dL2) || !std::isfinite(c.L2_lo))
            return fail(nullptr, PBE_ERR_ARG, "dL2 must be finite and > 0 in 2D mode");
        if (c.n_tangents != 0) return fail(nullptr, PBE_ERR_ARG, "2D mode has no tangent lanes (n_tangents = 0)");
        if (c.max_sims > pbe::K2D_MAXS) return fail(nullptr, PBE_ERR_ARG, "2D mode: max_sims <= %d", pbe::K2D_MAXS);
    }

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) return fail(nullptr, PBE_ERR_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(nullptr, PBE_ERR_ARG, "device %d out of range [0, %d)", device, ndev);
    e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail(nullptr, PBE_ERR_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));

    pbe_ctx ctx = new pbe_ctx_s();
    ctx->cfg = c;
    if (const char* e = getenv("PBE_LANES_PER_CTA")) ctx->group_max = atoi(e);
    if (const char* e = getenv("PBE_CLUSTER2")) ctx->cluster2 = atoi(e) != 0;
    if (const char* e = getenv("PBE_RESIDENT_K")) ctx->resident_k = atoi(e);
    if (const char* e = getenv("PBE_WS")) ctx->ws = atoi(e) != 0;
    if (const char* e = getenv("PBE_WS_VARIANT")) ctx->ws_variant = atoi(e);
    if (const char* e = getenv("PBE_WS_TAIL")) ctx->ws_tail = atoi(e) != 0;
    if (const char* e = getenv("PBE_STREAM_STATIC")) ctx->stream_static = atoi(e) != 0;
    if (const char* e = getenv("PBE_TEMPORAL_BLOCK")) ctx->temporal_block = atoi(e) != 0;
    if (const char* e = getenv("PBE_2D_UNFUSED")) ctx->unfused_2d = atoi(e) != 0;
    ctx->device = device;
    const size_t S = c.max_sims, M = c.n_samples, P = c.n_tangents;
    cudaError_t ea = cudaSuccess;
    const size_t RW = c.n_bins2 > 0 ? 8 : 6;                      // record width
    if (ea == cudaSuccess) ea = ctx->rec.ensure(S * M * RW * sizeof(double));
    if (ea == cudaSuccess) ea = ctx->trec.ensure(S * M * (P ? P : 1) * 5 * sizeof(double));
    if (ea == cudaSuccess) ea = ctx->status.ensure(S * sizeof(int));
    if (ea == cudaSuccess) ea = ctx->steps.ensure(S * sizeof(long long));
    if (ea == cudaSuccess) ea = ctx->loss.ensure(S * sizeof(double));
    if (ea == cudaSuccess) ea = ctx->grad.ensure(S * (P ? P : 1) * sizeof(double));
    if (ea == cudaSuccess) ea = ctx->c0.ensure(S * sizeof(double));
    if (ea == cudaSuccess) ea = ctx->tsamp.ensure(M * sizeof(double));
    if (ea == cudaSuccess) ea = cudaEventCreate(&ctx->ev0);
    if (ea == cudaSuccess) ea = cudaEventCreate(&ctx->ev1);
    if (ea != cudaSuccess) {
        const pbe_status st = ea == cudaErrorMemoryAllocation ? PBE_ERR_NOMEM : PBE_ERR_CUDA;
        fail(nullptr, st, "pbe_create: %s", cudaGetErrorString(ea));
        pbe_destroy(ctx);
        return st;
    }
    *out = ctx;
    return PBE_OK;
}

void pbe_destroy(pbe_ctx ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    for (DevBuf* b : {&ctx->theta, &ctx->sol, &ctx->knot_t, &ctx->knot_T, &ctx->seed, &ctx->c0, &ctx->tsamp,
                      &ctx->target, &ctx->n0_staged, &ctx->rec, &ctx->trec, &ctx->status, &ctx->steps,
                      &ctx->loss, &ctx->grad, &ctx->sbuf, &ctx->spart, &ctx->sbar, &ctx->sfinal, &ctx->snscale, &ctx->sdyn, &ctx->atr, &ctx->ack, &ctx->aseg, &ctx->agrad})
        b->release();
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    delete ctx;
}

pbe_status pbe_set_kinetics(pbe_ctx ctx, int32_t law, int32_t n_params, int32_t n_sims, const double* theta,
                            int32_t sol_kind, int32_t n_sol, const double* sol_params, int32_t n_knots,
                            const double* knot_t, const double* knot_T, int32_t knot_T_per_sim,
                            const double* tangent_seed) {
    if (!ctx) return fail(nullptr, PBE_ERR_ARG, "NULL context");
    if (law < PBE_LAW_CONST || law > PBE_LAW_POLY) return fail(ctx, PBE_ERR_ARG, "unknown law %d", law);
    if (n_params < 1 || n_params > pbe::MAX_PARAMS) return fail(ctx, PBE_ERR_ARG, "n_params must be in [1, %d]", pbe::MAX_PARAMS);
    const bool two_d = ctx->cfg.n_bins2 > 0;
    if (two_d && (n_params % 2) != 0) return fail(ctx, PBE_ERR_ARG, "2D mode: theta = [dim-1 law | dim-2 law] (even n_params)");
    const int per_dim = two_d ? n_params / 2 : n_params;
    if (law == PBE_LAW_CONST && per_dim != 1) return fail(ctx, PBE_ERR_ARG, "PBE_LAW_CONST takes 1 parameter per dimension");
    if (law == PBE_LAW_ARRHENIUS_GD && per_dim != 3 && per_dim != 6)
        return fail(ctx, PBE_ERR_ARG, "PBE_LAW_ARRHENIUS_GD takes 3 or 6 parameters per dimension");
    if (n_sims < 1 || n_sims > ctx->cfg.max_sims) return fail(ctx, PBE_ERR_ARG, "n_sims must be in [1, max_sims]");
    if (!theta || !sol_params || !knot_t || !knot_T) return fail(ctx, PBE_ERR_ARG, "NULL kinetics array");
    if (sol_kind == PBE_SOL_EXP ? n_sol != 2 : (sol_kind == PBE_SOL_POLY ? n_sol != 3 : true))
        return fail(ctx, PBE_ERR_ARG, "solubility: EXP takes 2 parameters, POLY takes 3");
    if (n_knots < 1) return fail(ctx, PBE_ERR_ARG, "n_knots must be >= 1");
    for (int k = 1; k < n_knots; ++k)
        if (!(knot_t[k] > knot_t[k - 1])) return fail(ctx, PBE_ERR_ARG, "knot_t must be strictly increasing");
    const size_t nth = (size_t)n_sims * n_params;
    for (size_t j = 0; j < nth; ++j)
        if (!std::isfinite(theta[j])) return fail(ctx, PBE_ERR_ARG, "theta[%zu] is not finite", j);
    const size_t nT = (size_t)(knot_T_per_sim ? n_sims : 1) * n_knots;
    for (size_t j = 0; j < nT; ++j)
        if (!std::isfinite(knot_T[j])) return fail(ctx, PBE_ERR_ARG, "knot_T[%zu] is not finite", j);
    const int P = ctx->cfg.n_tangents, nsd = n_params + n_sol;
    std::vector<double> seed((size_t)(P ? P : 1) * nsd, 0.0);
    if (tangent_seed) std::memcpy(seed.data(), tangent_seed, (size_t)P * nsd * sizeof(double));
    else for (int p = 0; p < P && p < n_params; ++p) seed[(size_t)p * nsd + p] = 1.0;

    CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    // a previous run may still be reading theta / sol / knots / seed on its (non-blocking) stream:
    // the synchronous copies below must not overwrite them under it
    if (ctx->have_run) CUDA_TRY(ctx, cudaStreamSynchronize(ctx->last_stream));
    CUDA_TRY(ctx, ctx->theta.ensure(nth * sizeof(double)));
    CUDA_TRY(ctx, ctx->sol.ensure(3 * sizeof(double)));
    CUDA_TRY(ctx, ctx->knot_t.ensure(n_knots * sizeof(double)));
    CUDA_TRY(ctx, ctx->knot_T.ensure(nT * sizeof(double)));
    CUDA_TRY(ctx, ctx->seed.ensure(seed.size() * sizeof(double)));
    CUDA_TRY(ctx, cudaMemcpy(ctx->theta.p, theta, nth * sizeof(double), cudaMemcpyHostToDevice));
    CUDA_TRY(ctx, cudaMemcpy(ctx->sol.p, sol_params, n_sol * sizeof(double), cudaMemcpyHostToDevice));
    CUDA_TRY(ctx, cudaMemcpy(ctx->knot_t.p, knot_t, n_knots * sizeof(double), cudaMemcpyHostToDevice));
    CUDA_TRY(ctx, cudaMemcpy(ctx->knot_T.p, knot_T, nT * sizeof(double), cudaMemcpyHostToDevice));
    CUDA_TRY(ctx, cudaMemcpy(ctx->seed.p, seed.data(), seed.size() * sizeof(double), cudaMemcpyHostToDevice));
    ctx->law = law; ctx->n_params = n_params; ctx->kin_sims = n_sims; ctx->sol_kind = sol_kind;
    ctx->n_sol = n_sol; ctx->n_knots = n_knots; ctx->knotT_per_sim = knot_T_per_sim != 0;
    ctx->have_kin = true;
    return PBE_OK;
}

pbe_status pbe_run_batch(pbe_ctx ctx, int32_t n_sims, const double* n0, int64_t n0_stride, int32_t n0_on_device,
                         const double* c0, const double* t_samples, const double* target, double* n_final,
                         double* ndot_final, void* cuda_stream) {
    {
        const pbe_status v = validate_run(ctx, n_sims, n0, n0_stride, n0_on_device, c0, t_samples, ndot_final);
        if (v != PBE_OK) return v;
    }
    const pbe_config& cf = ctx->cfg;
    const int N = cf.n_bins, P = cf.n_tangents;
    const bool two_d = cf.n_bins2 > 0;
    const bool steps_mode = cf.n_steps > 0;
    if (two_d && target) return fail(ctx, PBE_ERR_ARG, "the 2D model has no RSS objective: target must be NULL");

    // kernel choice: register-resident when the simulation fits one CTA, else streaming
    int groups = 1;
    int k_pref = ctx->resident_k;
    // batches of >= 2 simulations per SM: fat threads, small CTAs (several per SM overlap
    // their per-step latency); measured 4.4x at N = 1000
    if (!k_pref && P == 0 && n_sims >= 2 * 148) k_pref = 16;
    const ResidentVariant* rv = pick_resident(N, P, ctx->group_max, &groups, k_pref);
    const StreamVariant* sv = pick_stream(P);
    int cs = 1;
    const ResidentVariant* cv = pick_cluster(N, P, &cs);
    if (ctx->cluster2 && cf.kernel == PBE_KERNEL_AUTO) {
        const int Pi = P == 0 ? 0 : (P <= 4 ? 4 : (P <= 8 ? 8 : -1));
        for (const auto& v : kCluster2)
            if (v.P == Pi && v.K * v.maxt * 2 >= N) { cv = &v; cs = 2; rv = nullptr; break; }
    }
    int kind = cf.kernel;
    if (kind == PBE_KERNEL_AUTO) kind = rv ? PBE_KERNEL_RESIDENT : (cv ? PBE_KERNEL_CLUSTER : PBE_KERNEL_STREAM);
    // uncapped-CFL steps mode, primal: temporal blocking in k_stream beats the cluster kernel on
    // large meshes and large batches (measured: 1e5 x 64 2.38e11 vs 1.01e11, 1e4 x 1184 1.82e11
    // vs 1.56e11, 1e5 x 1 1.81e10 vs 1.59e10; cluster wins at 3e4 x 64 and 1e4 x 64)
    const bool tb_ok = ctx->temporal_block && steps_mode && cf.dt_fixed == 0.0 && std::isinf(cf.dt_max) && P == 0;
    if (cf.kernel == PBE_KERNEL_AUTO && kind == PBE_KERNEL_CLUSTER && tb_ok && sv &&
        (N >= 65536 || (long long)n_sims * N >= 8000000LL))
        kind = PBE_KERNEL_STREAM;
    if (kind == PBE_KERNEL_CLUSTER && !cv)
        return fail(ctx, PBE_ERR_ARG, "N = %d with %d tangent lanes does not fit a 16-CTA cluster", N, P);
    if (two_d) kind = PBE_KERNEL_2D;
    // P >= 1 lanes in one CTA: the warp-specialised resident kernel (primal and tangent warps
    // overlap the per-step scalar chain with the sweep); lane groups (PBE_LANES_PER_CTA) keep k_resident
    const WsVariant* ws = (kind == PBE_KERNEL_RESIDENT && P >= 1 && ctx->ws && groups == 1 && !two_d)
                              ? pick_ws(N, P, ctx->ws_variant) : nullptr;
    if (kind == PBE_KERNEL_RESIDENT && !rv && !ws)
        return fail(ctx, PBE_ERR_ARG, "N = %d with %d tangent lanes does not fit the resident kernel", N, P);
    if (kind == PBE_KERNEL_STREAM && !sv)
        return fail(ctx, PBE_ERR_ARG, "the streaming kernel supports at most 4 tangent lanes (got %d)", P);

    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    const double* n0_dev = nullptr;
    {
        const pbe_status v = stage_run(ctx, n_sims, n0, n0_stride, n0_on_device, c0, t_samples, target, st, &n0_dev);
        if (v != PBE_OK) return v;
    }
    KParams kp = make_kparams(ctx, n_sims, n0_dev, n0_stride, target, n_final, ndot_final, groups);

    ctx->info = pbe_run_info{};
    ctx->info.steps_per_pass = 1;
    if (two_d) {
        pbe_status r = ctx->unfused_2d ? launch_2d(ctx, kp, n_sims, n0_dev, n0_stride, n_final, st)
                                       : launch_2d_fused(ctx, kp, n_sims, n0_dev, n0_stride, n_final, st);
        if (r != PBE_OK) return r;
    } else if (kind == PBE_KERNEL_RESIDENT && ws) {
        const int nt = ws->nt;
        const size_t smem = ws->smem();
        CUDA_TRY(ctx, cudaFuncSetAttribute(ws->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        // one CTA per simulation runs in waves of `sms` CTAs.  A last partial wave of at most
        // sms/2 simulations runs as two half-lane CTAs per simulation instead (a second launch of
        // the P/2-lane variant with kp.G = 2; results are bitwise the same), so the tail wave
        // takes the time of a half-lane march: 512 sims on 148 SMs = 3 full waves + 68 x 2 CTAs
        int sms = 148;
        CUDA_TRY(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        const int tail = n_sims % sms;
        const WsVariant* half = nullptr;
        if (ctx->ws_tail && ws->P >= 2 && tail > 0 && 2 * tail <= sms) {
            for (const auto& v : kResidentWS)
                if (v.tag == 0 && v.P == ws->P / 2 && v.K == ws->K && v.nt == ws->nt) half = &v;
        }
        const int n_full = half ? n_sims - tail : n_sims;
        kp.G = 1;
        kp.sim0 = 0;
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
        if (n_full > 0) ws->fn<<<n_full, nt, smem, st>>>(kp);
        CUDA_TRY(ctx, cudaGetLastError());
        if (half) {
            const size_t hs = half->smem();
            CUDA_TRY(ctx, cudaFuncSetAttribute(half->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hs));
            KParams kh = kp;
            kh.G = 2;
            kh.sim0 = n_full;
            half->fn<<<2 * tail, nt, hs, st>>>(kh);
            CUDA_TRY(ctx, cudaGetLastError());
        }
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
        ctx->info.kernel = PBE_KERNEL_RESIDENT;
        ctx->info.launches = (n_full > 0) + (half != nullptr);
        ctx->info.threads_per_cta = nt;
        ctx->info.ctas = n_full + (half ? 2 * tail : 0);
        ctx->info.cluster = 1;
        ctx->info.bins_per_thread = ws->K;
        ctx->info.warp_specialized = 1;
    } else if (kind == PBE_KERNEL_RESIDENT) {
        const int nt = ((N + rv->K - 1) / rv->K + 31) / 32 * 32;
        const size_t smem = resident_smem(*rv, nt);
        CUDA_TRY(ctx, cudaFuncSetAttribute(rv->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
        rv->fn<<<n_sims * groups, nt, smem, st>>>(kp);
        CUDA_TRY(ctx, cudaGetLastError());
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
        ctx->info.kernel = PBE_KERNEL_RESIDENT;
        ctx->info.launches = 1;
        ctx->info.threads_per_cta = nt;
        ctx->info.ctas = n_sims * groups;
        ctx->info.cluster = 1;
        ctx->info.bins_per_thread = rv->K;
    } else if (kind == PBE_KERNEL_CLUSTER) {
        const int nt = ((N + cv->K * cs - 1) / (cv->K * cs) + 31) / 32 * 32;
        const size_t smem = resident_smem(*cv, nt);
        CUDA_TRY(ctx, cudaFuncSetAttribute(cv->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (cs > 8) CUDA_TRY(ctx, cudaFuncSetAttribute(cv->fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        kp.G = 1;                                   // tangent lanes are not split in cluster mode
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(n_sims * cs);
        lc.blockDim = dim3(nt);
        lc.dynamicSmemBytes = smem;
        lc.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        lc.attrs = attr;
        lc.numAttrs = 1;
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
        CUDA_TRY(ctx, cudaLaunchKernelEx(&lc, cv->fn, kp));
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
        ctx->info.kernel = PBE_KERNEL_CLUSTER;
        ctx->info.launches = 1;
        ctx->info.threads_per_cta = nt;
        ctx->info.ctas = n_sims * cs;
        ctx->info.cluster = cs;
        ctx->info.bins_per_thread = cv->K;
    } else if (ctx->temporal_block && steps_mode && cf.dt_fixed == 0.0 && std::isinf(cf.dt_max) && P == 0) {
        pbe_status r = launch_stream_tb(ctx, kp, n_sims, n0_dev, n0_stride, n_final, st);
        if (r != PBE_OK) return r;
    } else {
        pbe_status r = launch_stream(ctx, *sv, kp, n_sims, n0_dev, n0_stride, st);
        if (r != PBE_OK) return r;
    }
    ctx->info.main_ms = -1.0;
    ctx->have_run = true;
    ctx->last_sims = n_sims;
    ctx->last_stream = st;
    ctx->last_adjoint = false;
    return PBE_OK;
}

static pbe_status finish_run(pbe_ctx ctx) {
    if (!ctx) return fail(nullptr, PBE_ERR_ARG, "NULL context");
    if (!ctx->have_run) return fail(ctx, PBE_ERR_STATE, "no run to read (call pbe_run_batch first)");
    CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->last_stream));
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1) == cudaSuccess) ctx->info.main_ms = ms;
    return PBE_OK;
}

// D2H/D2D copies are stream-ordered on the run's stream, then the stream is synchronized
// (so CUDA events recorded on that stream afterwards bracket the copies too).
static pbe_status copy_out(pbe_ctx ctx, void* dst, const void* src, size_t bytes, int32_t on_device) {
    if (!dst || bytes == 0) return PBE_OK;
    CUDA_TRY(ctx, cudaMemcpyAsync(dst, src, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                  ctx->last_stream));
    return PBE_OK;
}

pbe_status pbe_moments(pbe_ctx ctx, double* moments, int32_t* sim_status, int64_t* sim_steps, double* loss,
                       int32_t on_device) {
    pbe_status r = finish_run(ctx);
    if (r != PBE_OK) return r;
    const size_t S = ctx->last_sims, M = ctx->cfg.n_samples;
    const size_t RW = ctx->cfg.n_bins2 > 0 ? 8 : 6;
    if ((r = copy_out(ctx, moments, ctx->rec.p, S * M * RW * sizeof(double), on_device)) != PBE_OK) return r;
    if ((r = copy_out(ctx, sim_status, ctx->status.p, S * sizeof(int), on_device)) != PBE_OK) return r;
    if ((r = copy_out(ctx, sim_steps, ctx->steps.p, S * sizeof(long long), on_device)) != PBE_OK) return r;
    if ((r = copy_out(ctx, loss, ctx->loss.p, S * sizeof(double), on_device)) != PBE_OK) return r;
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->last_stream));
    return PBE_OK;
}

pbe_status pbe_tangents(pbe_ctx ctx, double* tangents, double* grad, int32_t on_device) {
    pbe_status r = finish_run(ctx);
    if (r != PBE_OK) return r;
    const size_t S = ctx->last_sims, M = ctx->cfg.n_samples, P = ctx->cfg.n_tangents;
    if (P == 0) return fail(ctx, PBE_ERR_STATE, "context has no tangent lanes");
    if (ctx->last_adjoint) return fail(ctx, PBE_ERR_STATE, "the last run was pbe_run_adjoint (no tangent records)");
    if ((r = copy_out(ctx, tangents, ctx->trec.p, S * M * P * 5 * sizeof(double), on_device)) != PBE_OK) return r;
    if ((r = copy_out(ctx, grad, ctx->grad.p, S * P * sizeof(double), on_device)) != PBE_OK) return r;
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->last_stream));
    return PBE_OK;
}

pbe_status pbe_run_adjoint(pbe_ctx ctx, int32_t n_sims, const double* n0, int64_t n0_stride, int32_t n0_on_device,
                           const double* c0, const double* t_samples, const double* target, int32_t checkpoint_every,
                           void* cuda_stream) {
    {
        const pbe_status v = validate_run(ctx, n_sims, n0, n0_stride, n0_on_device, c0, t_samples, nullptr);
        if (v != PBE_OK) return v;
    }
    const pbe_config& cf = ctx->cfg;
    const int N = cf.n_bins;
    if (cf.n_bins2 > 0) return fail(ctx, PBE_ERR_ARG, "pbe_run_adjoint: 1D model only");
    if (cf.n_steps > 0) return fail(ctx, PBE_ERR_ARG, "pbe_run_adjoint: needs sample mode (n_steps = 0)");
    if (!target) return fail(ctx, PBE_ERR_ARG, "pbe_run_adjoint: needs a target (the loss to differentiate)");
    if (checkpoint_every < 0) return fail(ctx, PBE_ERR_ARG, "checkpoint_every must be >= 0");
    const AdjointVariant* av = nullptr;
    int nt = 0;
    size_t smem = 0;
    const int force_k = getenv("PBE_ADJ_K") ? atoi(getenv("PBE_ADJ_K")) : 0;   // A/B only
    for (const auto& v : kAdjoint) {
        const int t = ((N + v.K - 1) / v.K + 31) / 32 * 32;
        const size_t sm = (size_t)4 * pbe::adj_row(t, v.K) * sizeof(double);
        if (force_k && v.K != force_k) continue;
        if (t <= v.ntb && sm <= 212 * 1024) {
            av = &v; nt = t; smem = sm; break;
        }
    }
    if (!av) return fail(ctx, PBE_ERR_ARG, "pbe_run_adjoint: N = %d exceeds the adjoint kernel (N <= 6144)", N);
    const long long ms = cf.max_steps;
    // trajectory mode (checkpoint_every = 0): every state in HBM when it takes <= 16 GB (NEXT-3:
    // 9 x 12,001 x 2000 doubles = 1.7 GB) -- no re-march in the reverse pass; else O(sqrt) checkpoints
    const bool traj_mem = checkpoint_every == 0 &&
                          (double)n_sims * (ms + 1) * N * sizeof(double) <= 16.0 * (1ull << 30) &&
                          !getenv("PBE_ADJ_RECOMPUTE");
    // cluster mode (trajectory only): CS CTAs per simulation when the batch leaves SMs idle and the
    // mesh is large enough for the per-step latency to be the vector phases' (N >= 1024);
    // PBE_ADJ_CLUSTER = 0 disables it, = CS forces CS
    int cs = 1;
    {
        const char* e = getenv("PBE_ADJ_CLUSTER");
        const int want = e ? atoi(e) : -1;
        int sms = 0;
        CUDA_TRY(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        if (traj_mem && want != 0 && (want > 0 || N >= 1024)) {
            for (int c : {16, 8, 4, 2}) {
                if (want > 0 && c != want) continue;
                if (want < 0 && n_sims * c > sms) continue;
                for (const auto& v : kAdjointCL) {
                    const int nb = 64 * v.K;          // bins per CTA; every CTA but the last is full
                    if (c * nb >= N && (c - 1) * nb < N) {
                        // the cluster shape must be schedulable on this device (16 is non-portable)
                        if (c > 8) cudaFuncSetAttribute(v.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                        cudaLaunchConfig_t oc{};
                        oc.gridDim = dim3(c);
                        oc.blockDim = dim3(64);
                        oc.dynamicSmemBytes = (size_t)4 * pbe::adj_row(64, v.K) * sizeof(double) +
                                              64 * (size_t)pbe::ADJ_TR * sizeof(double);
                        cudaLaunchAttribute oa[1];
                        oa[0].id = cudaLaunchAttributeClusterDimension;
                        oa[0].val.clusterDim.x = c; oa[0].val.clusterDim.y = 1; oa[0].val.clusterDim.z = 1;
                        oc.attrs = oa;
                        oc.numAttrs = 1;
                        int ncl = 0;
                        if (cudaOccupancyMaxActiveClusters(&ncl, v.fn, &oc) != cudaSuccess || ncl < 1) {
                            cudaGetLastError();
                            break;
                        }
                        av = &v; cs = c; nt = 64;
                        smem = (size_t)4 * pbe::adj_row(64, v.K) * sizeof(double);
                        break;
                    }
                }
                if (cs > 1) break;
            }
        }
    }
    // segment length: the segment's trace rows are staged in shared memory every segment, and
    // its states n^{k0..k1} live there too when they fit (else in a global buffer)
    const size_t smem_cap = 220 * 1024, row = (size_t)pbe::adj_row(nt, av->K) * sizeof(double), trow = pbe::ADJ_TR * sizeof(double);
    int Kseg = checkpoint_every;
    const int NRr = (N + 1) & ~1;
    const bool traj = traj_mem && smem + 3 * row + 64 * (size_t)pbe::ADJ_TR * sizeof(double) <= 220 * 1024;
    if (Kseg == 0) Kseg = std::max(8, (int)std::ceil(std::sqrt((double)ms)));       // O(sqrt) memory
    int seg_smem = 0;
    if (traj) {
        Kseg = 64;                                        // trace rows staged per segment
        smem += 3 * row;
    } else {
        // largest K' <= Kseg with the states in shared memory; take it when K' >= min(Kseg, 4)
        long long kfit = ((long long)smem_cap - (long long)smem - (long long)row) / (long long)(row + trow);
        if (kfit >= std::min(Kseg, 4)) { Kseg = (int)std::min<long long>(Kseg, kfit); seg_smem = 1; }
        else {
            const long long ktr = ((long long)smem_cap - (long long)smem) / (long long)trow;   // trace only
            if (ktr < 1) return fail(ctx, PBE_ERR_ARG, "pbe_run_adjoint: no shared memory left for the trace");
            Kseg = (int)std::min<long long>(Kseg, ktr);
        }
    }
    smem += (size_t)Kseg * trow + (seg_smem ? (size_t)(Kseg + 1) * row : 0);
    const long long n_ck = traj ? ms + 1 : (ms + Kseg - 1) / Kseg;
    const size_t tr_b = (size_t)n_sims * ms * pbe::ADJ_TR * sizeof(double);
    const size_t ck_b = (size_t)n_sims * n_ck * (traj ? NRr : N) * sizeof(double);
    const size_t sg_b = (seg_smem || traj) ? sizeof(double) : (size_t)n_sims * (Kseg + 1) * row;
    if ((double)tr_b + ck_b + sg_b > 64.0 * (1ull << 30))
        return fail(ctx, PBE_ERR_ARG, "pbe_run_adjoint: trace + checkpoints need %.1f GB (> 64 GB): lower max_steps or n_sims",
                    ((double)tr_b + ck_b + sg_b) / (1ull << 30));

    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    const double* n0_dev = nullptr;
    {
        const pbe_status v = stage_run(ctx, n_sims, n0, n0_stride, n0_on_device, c0, t_samples, target, st, &n0_dev);
        if (v != PBE_OK) return v;
    }
    CUDA_TRY(ctx, ctx->atr.ensure(tr_b));
    CUDA_TRY(ctx, ctx->ack.ensure(ck_b));
    CUDA_TRY(ctx, ctx->aseg.ensure(sg_b));
    CUDA_TRY(ctx, ctx->agrad.ensure((size_t)n_sims * ctx->n_params * sizeof(double)));
    pbe::AdjParams ap{};
    ap.kp = make_kparams(ctx, n_sims, n0_dev, n0_stride, target, nullptr, nullptr, 1);
    ap.kp.P = 0;
    ap.ck = ctx->ack.as<double>(); ap.seg = ctx->aseg.as<double>(); ap.tr = ctx->atr.as<double>();
    ap.gtheta = ctx->agrad.as<double>(); ap.n_ck = n_ck; ap.Kseg = Kseg; ap.seg_smem = seg_smem; ap.traj = traj;
    CUDA_TRY(ctx, cudaFuncSetAttribute(av->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ctx->info = pbe_run_info{};
    void* args[] = {&ap};
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
    if (cs > 1) {
        if (cs > 8) CUDA_TRY(ctx, cudaFuncSetAttribute(av->fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(n_sims * cs);
        lc.blockDim = dim3(nt);
        lc.dynamicSmemBytes = smem;
        lc.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        lc.attrs = attr;
        lc.numAttrs = 1;
        CUDA_TRY(ctx, cudaLaunchKernelExC(&lc, av->fn, args));
    } else {
        CUDA_TRY(ctx, cudaLaunchKernel(av->fn, dim3(n_sims), dim3(nt), args, smem, st));
    }
    CUDA_TRY(ctx, cudaGetLastError());
    if (ctx->n_params > 0) {
        pbe::k_adjoint_theta<<<dim3((ctx->n_params + 31) / 32, n_sims), 256, 0, st>>>(ap);
        CUDA_TRY(ctx, cudaGetLastError());
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
    ctx->info.kernel = PBE_KERNEL_ADJOINT;
    ctx->info.launches = ctx->n_params > 0 ? 2 : 1;
    ctx->info.threads_per_cta = nt;
    ctx->info.ctas = n_sims * cs;
    ctx->info.cluster = cs;
    ctx->info.bins_per_thread = av->K;
    ctx->info.steps_per_pass = 1;
    ctx->info.main_ms = -1.0;
    ctx->have_run = true;
    ctx->last_sims = n_sims;
    ctx->last_stream = st;
    ctx->last_adjoint = true;
    return PBE_OK;
}

pbe_status pbe_adjoint_gradient(pbe_ctx ctx, double* grad, double* loss, int32_t on_device) {
    if (!ctx) return fail(nullptr, PBE_ERR_ARG, "NULL context");
    if (!ctx->have_run || !ctx->last_adjoint) return fail(ctx, PBE_ERR_STATE, "pbe_run_adjoint must precede pbe_adjoint_gradient");
    pbe_status r = finish_run(ctx);
    if (r != PBE_OK) return r;
    const size_t S = ctx->last_sims;
    if ((r = copy_out(ctx, grad, ctx->agrad.p, S * ctx->n_params * sizeof(double), on_device)) != PBE_OK) return r;
    if ((r = copy_out(ctx, loss, ctx->loss.p, S * sizeof(double), on_device)) != PBE_OK) return r;
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->last_stream));
    return PBE_OK;
}

pbe_status pbe_last_run_info(pbe_ctx ctx, pbe_run_info* info) {
    if (!ctx || !info) return fail(ctx, PBE_ERR_ARG, "NULL argument");
    if (!ctx->have_run) return fail(ctx, PBE_ERR_STATE, "no run yet");
    if (ctx->info.main_ms < 0.0 && cudaEventQuery(ctx->ev1) == cudaSuccess) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1) == cudaSuccess) ctx->info.main_ms = ms;
    }
    *info = ctx->info;
    return PBE_OK;
}

}  // extern "C"
