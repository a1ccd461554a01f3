// Design probe: measures the primitives the device-resident L-BFGS design
// depends on (graph WHILE conditional loop overhead, cooperative grid-sync
// cost, read-stream bandwidth).  Not part of the product.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

__global__ void body_kernel(int* counter, int limit, cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int c = ++(*counter);
    cudaGraphSetConditional(h, c < limit ? 1 : 0);
  }
}
__global__ void empty_kernel(int* p) { if (p && threadIdx.x == 1023) p[0] = 0; }

__global__ void gridsync_kernel(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

__global__ void stream_read(const float4* __restrict__ a, size_t n4, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a + i));
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s sm_%d%d SMs=%d L2=%d MB smemOptin=%zu clock=%d kHz\n", p.name, p.major, p.minor,
         p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, p.clockRate);
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  int* d_counter;
  CK(cudaMalloc(&d_counter, sizeof(int)));

  // 1. WHILE conditional graph with K kernels per iteration.
  for (int K : {1, 3, 5}) {
    cudaGraph_t graph;
    CK(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle handle;
    CK(cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cparams = {};
    cparams.type = cudaGraphNodeTypeConditional;
    cparams.conditional.handle = handle;
    cparams.conditional.type = cudaGraphCondTypeWhile;
    cparams.conditional.size = 1;
    cudaGraphNode_t cnode;
    CK(cudaGraphAddNode(&cnode, graph, nullptr, 0, &cparams));
    cudaGraph_t bodyg = cparams.conditional.phGraph_out[0];
    const int limit = 1000;
    cudaGraphNode_t prev = nullptr;
    for (int k = 0; k < K; ++k) {
      cudaKernelNodeParams kp = {};
      void* args_e[] = {&d_counter};
      int* nullp = nullptr;
      void* args_n[] = {&nullp};
      int lim = limit;
      void* args_b[] = {&d_counter, &lim, &handle};
      if (k == K - 1) { kp.func = (void*)body_kernel; kp.kernelParams = args_b; kp.gridDim = dim3(1); kp.blockDim = dim3(32); }
      else { kp.func = (void*)empty_kernel; kp.kernelParams = args_n; kp.gridDim = dim3(148); kp.blockDim = dim3(256); }
      (void)args_e;
      cudaGraphNode_t node;
      CK(cudaGraphAddKernelNode(&node, bodyg, prev ? &prev : nullptr, prev ? 1 : 0, &kp));
      prev = node;
    }
    cudaGraphExec_t exec;
    CK(cudaGraphInstantiate(&exec, graph, 0));
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaMemsetAsync(d_counter, 0, sizeof(int), s));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
      CK(cudaGraphLaunch(exec, s));
      cudaEventRecord(e1, s);
      CK(cudaStreamSynchronize(s));
      cudaEventElapsedTime(&ms, e0, e1);
    }
    int hc = 0;
    CK(cudaMemcpy(&hc, d_counter, sizeof(int), cudaMemcpyDeviceToHost));
    printf("while-graph K=%d kernels/iter: iters=%d  %.3f us/iter  %.3f us/kernel\n", K, hc,
           1000.f * ms / hc, 1000.f * ms / hc / K);
  }

  // 1b. plain stream launches of an empty kernel (host launch rate).
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 100; ++i) empty_kernel<<<148, 256, 0, s>>>(nullptr);
    cudaEventRecord(e0, s);
    for (int i = 0; i < 2000; ++i) empty_kernel<<<148, 256, 0, s>>>(nullptr);
    cudaEventRecord(e1, s);
    CK(cudaStreamSynchronize(s));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("stream launches: %.3f us/kernel\n", 1000.f * ms / 2000);
  }

  // 2. cooperative grid sync cost.
  for (int threads : {256, 512, 1024}) {
    int nb = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, gridsync_kernel, threads, 0));
    unsigned long long* d_out;
    CK(cudaMalloc(&d_out, 8));
    int iters = 1000;
    void* args[] = {&iters, &d_out};
    dim3 grid(p.multiProcessorCount), block(threads);
    CK(cudaLaunchCooperativeKernel((void*)gridsync_kernel, grid, block, args, 0, s));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    CK(cudaLaunchCooperativeKernel((void*)gridsync_kernel, grid, block, args, 0, s));
    cudaEventRecord(e1, s);
    CK(cudaStreamSynchronize(s));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc; cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
    printf("grid.sync 148x%d (occ %d): %.3f us/sync (%.0f cycles)\n", threads, nb, 1000.f * ms / iters,
           (double)cyc / iters);
    cudaFree(d_out);
  }

  // 3. stream read bandwidth, 2 GiB (HBM) and 32 MiB (L2-resident).
  for (size_t bytes : {(size_t)2 << 30, (size_t)32 << 20, (size_t)420 << 20}) {
    float4* a; float* o;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&o, 4));
    CK(cudaMemset(a, 0, bytes));
    size_t n4 = bytes / 16;
    for (int blocksPerSM : {4, 8}) {
      int grid = p.multiProcessorCount * blocksPerSM;
      for (int i = 0; i < 3; ++i) stream_read<<<grid, 256, 0, s>>>(a, n4, o);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      int reps = 20;
      cudaEventRecord(e0, s);
      for (int i = 0; i < reps; ++i) stream_read<<<grid, 256, 0, s>>>(a, n4, o);
      cudaEventRecord(e1, s);
      CK(cudaStreamSynchronize(s));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("read %zu MiB grid=%d: %.1f GB/s (%.2f us/pass)\n", bytes >> 20, grid,
             bytes * reps / (ms * 1e-3) / 1e9, 1000.f * ms / reps);
    }
    cudaFree(a); cudaFree(o);
  }
  // fp64 / fp32 FMA rate
  printf("done\n");
  return 0;
}
