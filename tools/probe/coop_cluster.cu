// Probe: cooperative launch combined with thread-block clusters (grid.sync + cluster.sync + DSMEM).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k(int* out, int iters) {
    extern __shared__ int sm[];
    cg::grid_group g = cg::this_grid();
    cg::cluster_group c = cg::this_cluster();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) sm[0] = blockIdx.x + i;
        c.sync();
        int v = *c.map_shared_rank(sm, (c.block_rank() + 1) % c.num_blocks());
        g.sync();
        if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = v;
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (int)((clock64() - t0) / iters);
}

int main() {
    int* d;
    CK(cudaMalloc(&d, 8));
    for (int cs : {8, 16}) {
        if (cs == 16) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        cudaLaunchConfig_t cfg = {};
        int nclusters = 0;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = 200 * 1024;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(cs);
        CK(cudaOccupancyMaxActiveClusters(&nclusters, (void*)k, &cfg));
        cfg.numAttrs = 2;
        cfg.gridDim = dim3(nclusters * cs);
        int iters = 1000;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t err = cudaLaunchKernelEx(&cfg, k, d, iters);
        cudaEventRecord(e1);
        cudaError_t err2 = cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        int h[2] = {0, 0}; cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("cluster %d: max active clusters %d grid %d launch=%s sync=%s  %.3f us/iter (cluster.sync+dsmem+grid.sync), %d cycles\n",
               cs, nclusters, nclusters * cs, cudaGetErrorString(err), cudaGetErrorString(err2), 1000.f * ms / iters, h[1]);
    }
    return 0;
}
