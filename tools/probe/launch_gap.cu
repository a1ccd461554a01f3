// Event-timed cost of launching an (almost) empty kernel with the solve kernel's launch
// shape: 120 CTAs x 288 threads, clusters of 8, ~212 KB dynamic shared memory, after a
// 512 MiB memset (the bench's L2 flush).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_gap launch_gap.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_k(int* p) {
    if (threadIdx.x == 0 && blockIdx.x == 100000) p[0] = 1;
}
int main() {
    int* d;
    cudaMalloc(&d, 4);
    void* fl;
    cudaMalloc(&fl, 512 << 20);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 << 10);
    cudaFuncSetAttribute(empty_k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaEvent_t x0, x1;
    cudaEventCreate(&x0);
    cudaEventCreate(&x1);
    int shapes[][3] = {{120, 8, 212504}, {120, 1, 0}};
    for (auto& sh : shapes) {
      for (int nev = 2; nev <= 4; nev += 2)
        for (int flush = 1; flush >= 0; --flush) {
            float tot = 0;
            for (int k = 0; k < 25; ++k) {
                if (flush) cudaMemsetAsync(fl, k, 512 << 20, s);
                cudaEventRecord(e0, s);
                if (nev == 4) cudaEventRecord(x0, s);
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = sh[1];
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.gridDim = dim3(sh[0]);
                cfg.blockDim = dim3(288);
                cfg.dynamicSmemBytes = sh[2];
                cfg.stream = s;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, empty_k, d);
                if (nev == 4) cudaEventRecord(x1, s);
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (k >= 5) tot += ms;
            }
            printf("grid %d cluster %d smem %d events %d flush %d: %.2f us  (%s)\n", sh[0], sh[1], sh[2], nev, flush, tot / 20 * 1e3,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
}
