// Shared device-side helpers for the B200-native reduced-objective path.
// Precision model: `T` is the storage/arithmetic type of the bandwidth-bound
// data (decoder output layer, displacements, element records, forces):
// double in fp64 mode, float in fp32 mode.  The latent-space work (hidden MLP,
// L-BFGS state, final reductions) is always fp64: it is tiny and latency-bound.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lsb {

constexpr int kMaxLatent = 64;    // d (latent dim) upper bound
constexpr int kMaxHistory = 16;   // L-BFGS memory upper bound
constexpr int kMaxHidden = 512;   // hidden width upper bound
constexpr int kMaxLayers = 16;    // hidden layers upper bound

enum Act : int { kIdentity = 0, kSilu = 1, kTanh = 2, kElu = 3 };

template <typename T> struct Vec4;
template <> struct alignas(16) Vec4<float> { float x, y, z, w; };
template <> struct alignas(32) Vec4<double> { double x, y, z, w; };

// ---- activation derivatives of order 0..3 (reference net.cpp:34-64; ELU is
// the BASELINE.json extension, the x <= 0 branch owns x == 0). ----------------
__device__ __forceinline__ double act_eval(int a, double x, int order) {
    switch (a) {
        case kIdentity: return order == 0 ? x : (order == 1 ? 1.0 : 0.0);
        case kSilu: {
            const double s = 1.0 / (1.0 + exp(-x));
            const double s1 = s * (1.0 - s);
            const double s2 = s1 * (1.0 - 2.0 * s);
            const double s3 = s2 * (1.0 - 2.0 * s) - 2.0 * s1 * s1;
            if (order == 0) return x * s;
            if (order == 1) return s + x * s1;
            if (order == 2) return 2.0 * s1 + x * s2;
            return 3.0 * s2 + x * s3;
        }
        case kTanh: {
            const double t = tanh(x);
            const double t1 = 1.0 - t * t;
            if (order == 0) return t;
            if (order == 1) return t1;
            if (order == 2) return -2.0 * t * t1;
            return -2.0 * t1 * t1 + 4.0 * t * t * t1;
        }
        default: {  // kElu
            if (x > 0.0) return order == 0 ? x : (order == 1 ? 1.0 : 0.0);
            return order == 0 ? expm1(x) : exp(x);
        }
    }
}

// ---- warp / block reductions ---------------------------------------------------------
template <typename V>
__device__ __forceinline__ V warp_sum(V v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic block sum (fixed tree); result valid in every thread.
// `scratch` needs blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < nw ? scratch[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) scratch[0] = t;
    }
    __syncthreads();
    const double r = scratch[0];
    __syncthreads();
    return r;
}

// ---- streaming loads (read-once data: skip L1, evict first from L2) -----------------------
// sm_100 supports 256-bit per-thread global loads; the L2::evict_first hint
// requires them.  One 32-byte vector = 8 floats or 4 doubles.
struct alignas(32) F8 { float v[8]; };
struct alignas(32) D4 { double v[4]; };

__device__ __forceinline__ F8 ld_stream(const F8* p) {
    F8 r;
    asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                   "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ D4 ld_stream(const D4* p) {
    D4 r;
    asm("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
                 : "l"(p));
    return r;
}

// ---- asynchronous global -> shared staging (LDGSTS): issue everything, wait once ----------
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// Block-cooperative copy of `count` doubles (8-byte aligned) into shared memory.
__device__ __forceinline__ void stage_doubles(double* dst, const double* src, int count) {
    const uintptr_t sa = reinterpret_cast<uintptr_t>(src), da = reinterpret_cast<uintptr_t>(dst);
    if (((sa ^ da) & 15u) == 0) {
        const int head = (sa & 15u) ? 1 : 0;
        if (head && threadIdx.x == 0 && count > 0) cp_async8(dst, src);
        const int body = (count - head) / 2;
        for (int k = threadIdx.x; k < body; k += blockDim.x) cp_async16(dst + head + 2 * k, src + head + 2 * k);
        const int tail = head + 2 * body;
        if (tail < count && threadIdx.x == 0) cp_async8(dst + tail, src + tail);
    } else {
        for (int k = threadIdx.x; k < count; k += blockDim.x) cp_async8(dst + k, src + k);
    }
}

// ---- mbarrier + TMA bulk copies (cp.async.bulk, global -> shared) ----------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t l2_policy(int keep) {
    uint64_t pol;
    if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// 1-D bulk copy of `bytes` (multiple of 16, 16B-aligned ends) completing on `bar`.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// Bulk L2 prefetch of [p, p + bytes) (16-byte granules, evict_last), in 32 KB
// pieces spread over the lanes-0 of the CTA's warps.
__device__ __forceinline__ void prefetch_l2_range(const void* p, size_t bytes, uintptr_t kPiece = 32768) {
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) != 0 || p == nullptr) return;
    const uintptr_t a0 = (reinterpret_cast<uintptr_t>(p) + 15) & ~(uintptr_t)15;
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + bytes) & ~(uintptr_t)15;
    const uint64_t pol = l2_policy(1);
    for (uintptr_t a = a0 + (uintptr_t)warp * kPiece; a < a1; a += (uintptr_t)nw * kPiece) {
        const unsigned n = (unsigned)((a1 - a) < kPiece ? (a1 - a) : kPiece);
        asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(a), "r"(n), "l"(pol)
                     : "memory");
    }
}

// DSMEM: address of the same shared variable in cluster CTA `rank`, remote store/load
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
    return r;
}
__device__ __forceinline__ void dsmem_st_f64(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ double dsmem_ld_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}

// Order this thread's generic-proxy global writes before later async-proxy
// (cp.async.bulk) reads of them; used before the barrier that publishes them.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// Programmatic dependent launch (no-ops unless the kernel was launched with a programmatic
// dependency): let the next kernel's CTAs start, and wait for the previous kernel's completion
// and memory before touching anything it writes.
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <typename T> struct VecT;
template <> struct VecT<float> { using type = F8; static constexpr int N = 8; };
template <> struct VecT<double> { using type = D4; static constexpr int N = 4; };

template <typename V, typename T>
__device__ __forceinline__ void vec_fma(T& acc, const V& w, const T* y) {
#pragma unroll
    for (int q = 0; q < (int)(sizeof(V) / sizeof(T)); ++q) acc = fma(w.v[q], y[q], acc);
}
template <typename V, typename T>
__device__ __forceinline__ void vec_axpy(T* acc, const V& w, T t) {
#pragma unroll
    for (int q = 0; q < (int)(sizeof(V) / sizeof(T)); ++q) acc[q] = fma(w.v[q], t, acc[q]);
}

// ---- stable neo-Hookean, cancellation-free (reference energy.cpp:178-221) ---------------
// log1p(x) - x, accurate for small |x| in either precision.
__device__ __forceinline__ double log1p_minus_x(double x) {
    if (fabs(x) < 1e-2) {
        const double x2 = x * x;
        return x2 * (-0.5 + x * (1.0 / 3.0 + x * (-0.25 + x * (0.2 + x * (-1.0 / 6.0 + x * (1.0 / 7.0))))));
    }
    return log1p(x) - x;
}
__device__ __forceinline__ float log1p_minus_x(float x) {
    if (fabsf(x) < 5e-2f) {
        const float x2 = x * x;
        return x2 * (-0.5f + x * (1.0f / 3.0f + x * (-0.25f + x * (0.2f + x * (-1.0f / 6.0f + x * (1.0f / 7.0f))))));
    }
    return log1pf(x) - x;
}

// Given the strain increment A = (Ds - Ds_rest) Dm^-1 (row-major 3x3), Lame mu,
// lambda, returns psi and the first Piola-Kirchhoff stress P (row-major),
// algebraically identical to the reference density
//   psi = mu/2 i - mu/2 log1p(i/4) + lambda/2 (J-1)^2 - 3/4 mu (J-1)
// with i = |F|^2 - 3 and P = 2 psi_I F + psi_J cof(F), but regrouped so that no
// O(1) or O(|A|) terms cancel:
//   psi = 3/8 mu |A|^2 - 3/4 mu (m2 + det A) - mu/2 L(i/4) + lambda/2 (J-1)^2,
//   P   = 3/4 mu (A + A^T - tr(A) I - cof A) + mu i / (4 (4 + i)) F + lambda (J-1) cof F,
// with L(x) = log1p(x) - x, cof(F) = I + tr(A) I - A^T + cof(A).
template <typename T>
__device__ __forceinline__ T snh_psi_P(const T* A, T mu, T lambda, T* P) {
    const T trA = A[0] + A[4] + A[8];
    T q = 0;
#pragma unroll
    for (int k = 0; k < 9; ++k) q += A[k] * A[k];
    const T m2 = A[0] * A[4] - A[1] * A[3] + A[0] * A[8] - A[2] * A[6] + A[4] * A[8] - A[5] * A[7];
    // cofactor matrix of A: columns a1 x a2, a2 x a0, a0 x a1 (a_b = column b)
    T cA[9];
    cA[0 * 3 + 0] = A[1 * 3 + 1] * A[2 * 3 + 2] - A[2 * 3 + 1] * A[1 * 3 + 2];
    cA[1 * 3 + 0] = A[2 * 3 + 1] * A[0 * 3 + 2] - A[0 * 3 + 1] * A[2 * 3 + 2];
    cA[2 * 3 + 0] = A[0 * 3 + 1] * A[1 * 3 + 2] - A[1 * 3 + 1] * A[0 * 3 + 2];
    cA[0 * 3 + 1] = A[1 * 3 + 2] * A[2 * 3 + 0] - A[2 * 3 + 2] * A[1 * 3 + 0];
    cA[1 * 3 + 1] = A[2 * 3 + 2] * A[0 * 3 + 0] - A[0 * 3 + 2] * A[2 * 3 + 0];
    cA[2 * 3 + 1] = A[0 * 3 + 2] * A[1 * 3 + 0] - A[1 * 3 + 2] * A[0 * 3 + 0];
    cA[0 * 3 + 2] = A[1 * 3 + 0] * A[2 * 3 + 1] - A[2 * 3 + 0] * A[1 * 3 + 1];
    cA[1 * 3 + 2] = A[2 * 3 + 0] * A[0 * 3 + 1] - A[0 * 3 + 0] * A[2 * 3 + 1];
    cA[2 * 3 + 2] = A[0 * 3 + 0] * A[1 * 3 + 1] - A[1 * 3 + 0] * A[0 * 3 + 1];
    const T detA = A[0] * cA[0] + A[3] * cA[3] + A[6] * cA[6];  // column-0 expansion
    const T jm1 = trA + m2 + detA;
    const T i_minus = T(2) * trA + q;
    const T x = i_minus * T(0.25);
    const T psi = T(0.375) * mu * q - T(0.75) * mu * (m2 + detA) - T(0.5) * mu * log1p_minus_x(x) +
                  T(0.5) * lambda * jm1 * jm1;
    const T c1 = T(0.75) * mu;
    const T c2 = mu * i_minus / (T(4) * (T(4) + i_minus));
    const T c3 = lambda * jm1;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const T Aab = A[a * 3 + b], Aba = A[b * 3 + a];
            const T id = (a == b) ? T(1) : T(0);
            const T cofF = id + trA * id - Aba + cA[a * 3 + b];
            const T F = id + Aab;
            P[a * 3 + b] = c1 * (Aab + Aba - trA * id - cA[a * 3 + b]) + c2 * F + c3 * cofF;
        }
    return psi;
}

}  // namespace lsb
