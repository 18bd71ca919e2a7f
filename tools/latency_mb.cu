// Latency microbenchmarks for the resident kernel's per-step scalar chain (diagnostic tool,
// not product code): dependent-chain latency of DFMA/DADD/DMUL, MUFU.RCP64H + Newton,
// LDS.64, SHFL of a double, BAR.SYNC of 256 threads, and a D1 (dual) Horner step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/latency_mb tools/latency_mb.cu
#include <cstdio>
#include <cuda_runtime.h>

#define REP 1024

__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

__global__ void k_lat(long long* out, double a, double b, int mode) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (double)((i * 7) & 1023);
    __syncthreads();
    double x = a + threadIdx.x * 1e-30;
    double y = b;
    int idx = threadIdx.x & 1023;
    long long t0 = clock64();
    switch (mode) {
        case 0:   // DFMA chain
#pragma unroll 16
            for (int i = 0; i < REP; ++i) x = fma(x, a, b);
            break;
        case 1:   // DADD chain
#pragma unroll 16
            for (int i = 0; i < REP; ++i) x = x + b;
            break;
        case 2:   // DMUL chain
#pragma unroll 16
            for (int i = 0; i < REP; ++i) x = x * a;
            break;
        case 3:   // rcp_nr chain
#pragma unroll 4
            for (int i = 0; i < REP; ++i) x = rcp_nr(x) + 1e-300;
            break;
        case 4:   // LDS chain (pointer chase in smem)
#pragma unroll 16
            for (int i = 0; i < REP; ++i) idx = (int)sm[idx];
            x = idx;
            break;
        case 5:   // SHFL of a double chain
#pragma unroll 16
            for (int i = 0; i < REP; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
            break;
        case 6:   // BAR.SYNC (whole CTA)
            for (int i = 0; i < REP; ++i) __syncthreads();
            break;
        case 7: { // D1 Horner step: g = g * x + a  (value and derivative)
            double gv = x, gd = y, xv = a, xd = b;
#pragma unroll 16
            for (int i = 0; i < REP; ++i) {
                const double nv = fma(gv, xv, 0.25);
                const double nd = fma(gd, xv, fma(gv, xd, 0.5));
                gv = nv; gd = nd;
            }
            x = gv + gd;
            break;
        }
        case 8:   // DSETP + FSEL dependent (compare/select on doubles)
#pragma unroll 16
            for (int i = 0; i < REP; ++i) x = (x > b) ? x * 0.5 : x + a;
            break;
        case 9:   // exp() chain
#pragma unroll 4
            for (int i = 0; i < REP; ++i) x = exp(x * 1e-3);
            break;
        case 10:  // log() chain
#pragma unroll 4
            for (int i = 0; i < REP; ++i) x = log(x + 2.0);
            break;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (x == 12345.678) out[1000] = (long long)x;
}

int main() {
    long long* d;
    cudaMalloc(&d, 2048 * sizeof(long long));
    const char* names[] = {"DFMA", "DADD", "DMUL", "rcp_nr(MUFU+4FMA)+DADD", "LDS.64 chase", "SHFL.f64",
                           "BAR.SYNC 256t", "D1 Horner step", "DSETP+select", "exp", "log"};
    for (int mode = 0; mode < 11; ++mode) {
        for (int threads : {32, 256}) {
            long long h = 0;
            k_lat<<<1, threads>>>(d, 0.9999999, 1e-9, mode);
            k_lat<<<1, threads>>>(d, 0.9999999, 1e-9, mode);
            cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
            printf("%-26s threads %3d : %.2f cycles/op\n", names[mode], threads, (double)h / REP);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
