// Diagnostic microbenchmark (not product code): cluster.sync() round trip and DSMEM load latency
// for cluster sizes 2..16.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_lat tools/cluster_lat.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(long long* out, int reps, int mode) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double buf[64];
    buf[threadIdx.x & 63] = threadIdx.x;
    cl.sync();
    const int r = cl.block_rank(), cs = cl.num_blocks();
    double* peer = cl.map_shared_rank(buf, (r + 1) % cs);
    double acc = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < reps; ++i) {
        if (mode == 0) cl.sync();
        else if (mode == 1) { acc += peer[(int)acc & 63]; }          // dependent DSMEM load chain
        else { if (threadIdx.x < 32) acc += peer[(threadIdx.x + (int)acc) & 63]; cl.sync(); }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / reps;
    if (acc == 12345.0) out[1] = 1;
}

int main() {
    long long* d; cudaMalloc(&d, 16);
    for (int mode = 0; mode < 3; ++mode)
        for (int cs : {1, 2, 4, 8, 16})
            for (int nt : {64, 256}) {
                cudaFuncSetAttribute(k_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(cs * 9); cfg.blockDim = dim3(nt);
                cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                cfg.attrs = at; cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, k_sync, d, 2000, mode);
                cudaLaunchKernelEx(&cfg, k_sync, d, 2000, mode);
                long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
                printf("%s cs %2d threads %3d : %lld cycles/op (%s)\n",
                       mode == 0 ? "cluster.sync      " : mode == 1 ? "DSMEM load chain  " : "DSMEM load + sync ",
                       cs, nt, h, cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
