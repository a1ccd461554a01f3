// Measurement hooks used by bench.py: per-step CUDA-event timing on the
// context's stream, with an L2 flush (a write of a buffer larger than L2)
// before every timed step so W_out is re-read from HBM each step.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <functional>
#include <vector>

#include "../../include/lipsub_b200.h"
#include "lsb_context.hpp"

namespace lsb {

// L2 flush as a kernel with the solve kernel's shared-memory carveout (LSB_FLUSH_MODE=kernel,
// experiment): a memset runs with the default L1/shared split, and switching the split back
// costs the next kernel its startup.
__global__ void flush_kernel(uint4* p, size_t n, unsigned v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(v, v, v, v);
}
// Diagnostic (LSB_FLUSH_MODE=readback): after the write flush, read a second buffer larger than
// L2 so the dirty lines are written back outside the timed region and L2 holds clean lines --
// separates the flush's write-back cost from the evaluation's own traffic.
__global__ void flush_read_kernel(const uint4* p, size_t n, unsigned* sink) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc ^= __ldcg(p + i).x;
    if (acc == 0x12345678u) *sink = acc;
}

void bench_evals(Context& c, int K, const double* Z, size_t flush_bytes, double* eval_ms, double* out_ms,
                 double* E, bool want_grad) {
    const int r = c.r;
    double* dZ = nullptr;
    cuda_check(cudaMalloc(&dZ, sizeof(double) * (size_t)K * r), "bench Z");
    c.copy(dZ, Z, sizeof(double) * (size_t)K * r, cudaMemcpyHostToDevice, "bench Z");
    void* flush = nullptr;
    if (flush_bytes) cuda_check(cudaMalloc(&flush, flush_bytes), "bench flush");
    cudaEvent_t ev[4];
    for (auto& e : ev) cuda_check(cudaEventCreate(&e), "event");
    const char* fm = getenv("LSB_FLUSH_MODE");
    const bool fkern = fm && !strcmp(fm, "kernel");
    const bool fread = fm && !strcmp(fm, "readback");
    void* flush2 = nullptr;
    if (fread && flush_bytes) cuda_check(cudaMalloc(&flush2, flush_bytes), "bench flush2");
    if (fkern) {
        cudaFuncSetAttribute(flush_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(flush_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
    }
    for (int k = 0; k < K; ++k) {
        if (flush && fkern)
            flush_kernel<<<148 * 2, 512, 200 << 10, c.stream>>>((uint4*)flush, flush_bytes / 16, (unsigned)k);
        else if (flush) cuda_check(cudaMemsetAsync(flush, k & 0xff, flush_bytes, c.stream), "flush");
        if (flush2)
            flush_read_kernel<<<148 * 4, 512, 0, c.stream>>>((const uint4*)flush2, flush_bytes / 16,
                                                            (unsigned*)flush2);
        cuda_check(cudaMemcpyAsync(c.d_state->zt, dZ + (size_t)k * r, sizeof(double) * r, cudaMemcpyDeviceToDevice,
                                   c.stream),
                   "z");
        const int nev = c.impl->eval_timed(c, ev, want_grad);
        cuda_check(cudaEventSynchronize(ev[3]), "bench sync");
        float t0, t1;
        cudaEventElapsedTime(&t0, ev[0], ev[3]);
        if (nev == 4) cudaEventElapsedTime(&t1, ev[1], ev[2]);
        else t1 = t0;
        eval_ms[k] = t0;
        out_ms[k] = t1;
        if (E) c.copy(&E[k], &c.d_state->f_eval, sizeof(double), cudaMemcpyDeviceToHost, "E");
    }
    for (auto& e : ev) cudaEventDestroy(e);
    if (flush) cudaFree(flush);
    if (flush2) cudaFree(flush2);
    cudaFree(dZ);
}

void bench_steps(Context& c, int K, size_t flush_bytes, double* step_ms, lsb_exit_report* reps) {
    void* flush = nullptr;
    if (flush_bytes) cuda_check(cudaMalloc(&flush, flush_bytes), "bench flush");
    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
    for (int k = 0; k < K; ++k) {
        if (flush) cuda_check(cudaMemsetAsync(flush, k & 0xff, flush_bytes, c.stream), "flush");
        cuda_check(cudaEventRecord(e0, c.stream), "ev");
        c.impl->step(c);
        cuda_check(cudaEventRecord(e1, c.stream), "ev");
        cuda_check(cudaEventSynchronize(e1), "bench sync");
        float t;
        cudaEventElapsedTime(&t, e0, e1);
        step_ms[k] = t;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (flush) cudaFree(flush);
    if (reps) c.copy(reps, c.d_reports, sizeof(lsb_exit_report) * K, cudaMemcpyDeviceToHost, "reports");
}

// One library call (batched evaluation or Lipschitz loss, `call`) per rep, each preceded by an L2
// flush and bracketed by CUDA events on the context stream.  The bracket holds everything the
// call enqueues on that stream, including its small host<->device copies of Z and results.
void bench_call(Context& c, int reps, size_t flush_bytes, double* ms, const std::function<void()>& call) {
    void* flush = nullptr;
    if (flush_bytes) cuda_check(cudaMalloc(&flush, flush_bytes), "bench flush");
    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
    for (int k = 0; k < reps; ++k) {
        if (flush) cuda_check(cudaMemsetAsync(flush, k & 0xff, flush_bytes, c.stream), "flush");
        cuda_check(cudaEventRecord(e0, c.stream), "ev");
        call();
        cuda_check(cudaEventRecord(e1, c.stream), "ev");
        cuda_check(cudaEventSynchronize(e1), "bench sync");
        float t;
        cudaEventElapsedTime(&t, e0, e1);
        ms[k] = t;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (flush) cudaFree(flush);
}

}  // namespace lsb
