// Batched evaluation of E(z) and grad E(z) for many latent vectors (config 4),
// and the second-order path (subspace Hessians, Lipschitz loss; config 5).
//
// Layout per batch chunk of BC columns (fp32 storage, fp64 reductions):
//   Y_l, A_l  [h][BC]      hidden activations / pre-activations
//   U         [V][3][BC]   vertex displacements (pinned rows = pin displacement)
//   T         [n][BC]      s * (gathered elastic forces + inertia residual)
//   Ybar      [h][BC]      W_out^T T
// Element pass: contiguous tet blocks (host-precomputed block -> touched free
// vertices); one CTA per (block, 64-column tile); thread b owns column b and
// accumulates the block's vertex forces in shared memory in ascending tet order
// (deterministic, no atomics); block partials are combined per vertex in
// ascending block order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <tuple>
#include <vector>

#include "lsb_batched.hpp"
#include "lsb_tc.cuh"
#include "lsb_theta.cuh"

namespace lsb {

namespace {

constexpr int kBC = 256;       // batch columns per chunk (tcgen05 N)
constexpr int kEcols = 64;     // columns per element CTA
constexpr int kTB = 48;        // tets per element block (Hessian path; also the staging capacity)
#ifndef LSB_TBE
#define LSB_TBE 24
#endif
constexpr int kTBE = LSB_TBE;  // tets per element block of the batched evaluation (more CTAs resident)

__device__ __forceinline__ float act_f(int a, float x, int order) {
    return (float)act_eval(a, (double)x, order);
}

// ---------------------------------------------------------------- small GEMMs (hidden layers)
// C[M][N] = A[M][K] * B[K][N] (+ bias[M]); optional pre-activation store and activation.
// transA: A given as [K][M] (computes A^T B).  Tile 32x32, 256 threads, 2x2 per thread.
__global__ void __launch_bounds__(256) small_gemm_kernel(int M, int N, int K, const double* A, int transA,
                                                         const float* B, const double* bias, float* C,
                                                         float* pre, int act, const float* gate, int gate_act) {
    __shared__ float As[16][33];
    __shared__ float Bs[16][33];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
    float acc[2][2] = {{0, 0}, {0, 0}};
    for (int k0 = 0; k0 < K; k0 += 16) {
        for (int t = threadIdx.x; t < 16 * 32; t += 256) {
            const int kk = t / 32, mm = t % 32;
            const int m = m0 + mm, k = k0 + kk;
            As[kk][mm] = (m < M && k < K) ? (float)(transA ? A[(size_t)k * M + m] : A[(size_t)m * K + k]) : 0.f;
            const int n = n0 + mm;
            Bs[kk][mm] = (n < N && k < K) ? B[(size_t)k * N + n] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) acc[i][j] = fmaf(As[kk][ty * 2 + i], Bs[kk][tx * 2 + j], acc[i][j]);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int m = m0 + ty * 2 + i, n = n0 + tx * 2 + j;
            if (m < M && n < N) {
                float v = acc[i][j] + (bias ? (float)bias[m] : 0.f);
                if (pre) pre[(size_t)m * N + n] = v;
                if (gate) v *= act_f(gate_act, gate[(size_t)m * N + n], 1);  // backward: times phi'(pre)
                C[(size_t)m * N + n] = act >= 0 ? act_f(act, v, 0) : v;
            }
        }
}

// ---------------------------------------------------------------- output layer epilogue (CUDA-core path)
// Ubuf[n][BC] = W_out[n][h] * Y[h][BC] (fp32 SGEMM, 128x128 tiles, 8x8 per thread).
__global__ void __launch_bounds__(256) sgemm_nn_kernel(int M, int N, int K, const float* A, int lda, const float* B,
                                                       int ldb, float* C, int ldc) {
    __shared__ float As[16][128 + 4];
    __shared__ float Bs[16][128 + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.y * 128, n0 = blockIdx.x * 128;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    for (int k0 = 0; k0 < K; k0 += 16) {
        for (int t = threadIdx.x; t < 16 * 128; t += 256) {
            const int mm = t / 16, kk = t % 16;
            const int m = m0 + mm, k = k0 + kk;
            As[kk][mm] = (m < M && k < K) ? A[(size_t)m * lda + k] : 0.f;
            const int kb = t / 128, nn = t % 128;
            const int n = n0 + nn, k2 = k0 + kb;
            Bs[kb][nn] = (n < N && k2 < K) ? B[(size_t)k2 * ldb + n] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float a[8], b[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
            if (m < M && n < N) C[(size_t)m * ldc + n] = acc[i][j];
        }
}

// Split-K Ybar partials: P[kc][h][BC] = W_out[k-range]^T T[k-range][BC] (fp32).
__global__ void __launch_bounds__(256) sgemm_tn_splitk_kernel(int H, int N, int K, int kchunk, const float* W,
                                                              int ldw, const float* T, int ldt, float* P) {
    __shared__ float As[16][128 + 4];
    __shared__ float Bs[16][128 + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.y * 128, n0 = blockIdx.x * 128;
    const int kb0 = blockIdx.z * kchunk, kb1 = min(K, kb0 + kchunk);
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    for (int k0 = kb0; k0 < kb1; k0 += 16) {
        for (int t = threadIdx.x; t < 16 * 128; t += 256) {
            const int kk = t / 128, mm = t % 128;
            const int m = m0 + mm, k = k0 + kk;
            As[kk][mm] = (m < H && k < kb1) ? W[(size_t)k * ldw + m] : 0.f;
            const int n = n0 + mm;
            Bs[kk][mm] = (n < N && k < kb1) ? T[(size_t)k * ldt + n] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float a[8], b[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    float* out = P + (size_t)blockIdx.z * H * N;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
            if (m < H && n < N) out[(size_t)m * N + n] = acc[i][j];
        }
}

// Deterministic split-K reduction: Ybar[h][N] = sum_kc P[kc][h][N] (fp64 accumulate).
__global__ void splitk_reduce_kernel(int HN, int nk, const float* P, float* out, int N = 0, int ldo = 0) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < HN; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        int k = 0;
        for (; k + 8 <= nk; k += 8) {  // 8 loads in flight, summed in k order
            float v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = __ldg(P + (size_t)(k + q) * HN + i);
#pragma unroll
            for (int q = 0; q < 8; ++q) s += v[q];
        }
        for (; k < nk; ++k) s += P[(size_t)k * HN + i];
        out[ldo ? (size_t)(i / N) * ldo + i % N : (size_t)i] = (float)s;
    }
}

// u = s (C + b) + shift - X -> U[v][3][N]; inertia residual and energy partials per column.
__global__ void __launch_bounds__(256) out_epilogue_kernel(int n, int N, const float* C, const double* eprow,
                                                           const double* ut, int has_inertia, double inv_dt2,
                                                           float* U, float* rin, double* epart) {
    // block: 256 threads over (rows tile of 64) x (N columns), column-major partial sums
    const int col = threadIdx.x % 64 + 64 * blockIdx.y;
    const int rsub = threadIdx.x / 64;  // 4 row lanes
    __shared__ double red[4][64];
    double e = 0.0;
    if (col < N) {
        for (int row = blockIdx.x * 64 + rsub; row < min(n, (int)(blockIdx.x + 1) * 64); row += 4) {
            const double* e6 = eprow + (size_t)row * 6;
            const double u = e6[1] * ((double)C[(size_t)row * N + col] + e6[0]) + e6[2];
            const int slot = (int)e6[4];  // 4 v + c
            U[((size_t)(slot >> 2) * 3 + (slot & 3)) * N + col] = (float)u;
            if (has_inertia) {
                const double d = u - ut[row];
                rin[(size_t)row * N + col] = (float)(inv_dt2 * e6[3] * d);
                e += e6[3] * d * d;
            }
        }
    }
    red[rsub][threadIdx.x % 64] = e;
    __syncthreads();
    if (rsub == 0 && col < N)
        epart[(size_t)blockIdx.x * N + col] = 0.5 * inv_dt2 * (red[0][threadIdx.x] + red[1][threadIdx.x] +
                                                                red[2][threadIdx.x] + red[3][threadIdx.x]);
}

// Element pass per (block of kTB tets, kEcols columns), thread = column:
//  - the block's records (as fp32) and vertex slots are staged once in shared
//    memory (no per-thread record loads or conversions);
//  - displacements come through L1/L2 with the next tet's 12 values loaded while
//    the current tet computes (register double buffer);
//  - forces accumulate per (free vertex slot, column) in shared memory, tets in id
//    order -> deterministic.
template <typename TR>
__global__ void __launch_bounds__(kEcols) elem_batched2_kernel(const TR* rec, const int* blk_tet0,
                                                              const int* blk_vptr, const short* tet_loc,
                                                              const int4* tets, const float* U, int N,
                                                              float* partial, double* eblk) {
    extern __shared__ float sm[];
    const int blk = blockIdx.x, tid = threadIdx.x;
    const int col = blockIdx.y * kEcols + tid;
    const int e0 = blk_tet0[blk], ne = blk_tet0[blk + 1] - e0;
    const int v0 = blk_vptr[blk], nv = blk_vptr[blk + 1] - v0;
    float* acc = sm;                          // [(nv + 1) * 3][kEcols]; slot nv absorbs pinned corners
    float* rs = acc + (nv + 1) * 3 * kEcols;  // [kTB][12]
    int* vs = reinterpret_cast<int*>(rs + kTB * 12);  // [kTB][4] row offsets v * 3 * N
    int* los = vs + kTB * 4;                          // [kTB][4] accumulator offsets slot * 3 * kEcols
    for (int i = tid; i < nv * 3 * kEcols; i += kEcols) acc[i] = 0.f;
    for (int i = tid; i < ne * 12; i += kEcols) rs[i] = (float)rec[(size_t)e0 * 12 + i];
    for (int i = tid; i < ne * 4; i += kEcols) {
        const int4 t = __ldg(tets + e0 + (i >> 2));
        const int k = i & 3;
        vs[i] = (k == 0 ? t.x : k == 1 ? t.y : k == 2 ? t.z : t.w) * 3 * N;
        const int lv = tet_loc[(size_t)e0 * 4 + i];
        los[i] = (lv >= 0 ? lv : nv) * 3 * kEcols;
    }
    __syncthreads();
    double esum = 0.0;
    if (col < N) {
        const float* Uc = U + col;
        float un[12];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int c = 0; c < 3; ++c) un[k * 3 + c] = __ldg(Uc + vs[k] + c * N);
        for (int e = 0; e < ne; ++e) {
            float u[4][3];
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int c = 0; c < 3; ++c) u[k][c] = un[k * 3 + c];
            if (e + 1 < ne) {
                const int* vn = vs + (e + 1) * 4;
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int c = 0; c < 3; ++c) un[k * 3 + c] = __ldg(Uc + vn[k] + c * N);
            }
            float rc[12];
#pragma unroll
            for (int q = 0; q < 12; ++q) rc[q] = rs[e * 12 + q];
            float f[12];
            esum += (double)tet_energy_forces_t<float>(u[0], u[1], u[2], u[3], rc, f);
            // branch-free scatter: one 16-byte load of the 4 slot offsets (pinned -> slot nv)
            const int4 o4 = *reinterpret_cast<const int4*>(los + e * 4);
            const int off[4] = {o4.x, o4.y, o4.z, o4.w};
            float* at = acc + tid;
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int c = 0; c < 3; ++c) at[off[k] + c * kEcols] += f[k * 3 + c];
        }
        for (int i = 0; i < nv * 3; ++i) partial[((size_t)(v0 * 3) + i) * N + col] = acc[i * kEcols + tid];
        eblk[(size_t)blk * N + col] = esum;
    }
}

// ---- packed fp32x2 element pass (sm_100 FFMA2 / FMUL2 / FADD2): two latent columns per thread
// The scalar kernel above is issue-bound (~390 instructions per tet and column, 246 of them fp32
// arithmetic).  Here every arithmetic instruction works on the thread's two adjacent columns; operand
// negation rides on the FFMA2 / FADD2 source modifiers, per-tet constants are staged in shared memory
// as duplicated pairs (one 64-bit operand, no broadcast moves), the stress is regrouped as
//   P = (c1 + c2) A + (c1 - c3) (A^T - cof A) + (c2 + c3 - (c1 - c3) tr A) I
// (algebraically snh_psi_P's form) and the forces use vol Dm^-1 precomputed per tet:
// ~150 instructions per tet and column.  Forces accumulate per (vertex slot, column pair) in shared
// memory in tet order -- deterministic, as above.
__device__ __forceinline__ float2 p2neg(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 p2add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 p2sub(float2 a, float2 b) { return __fadd2_rn(a, p2neg(b)); }
__device__ __forceinline__ float2 p2mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 p2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 p2fms(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, p2neg(c)); }  // a b - c

constexpr int kP2Threads = 64;  // threads per CTA = column pairs: 128 columns per CTA
constexpr int kP2Consts = 26;   // per-tet constant pairs: Dm^-1 (9), vol Dm^-1 (9), energy / stress coefficients (8)

__global__ void __launch_bounds__(kP2Threads) elem_batched_p2_kernel(const float* rec, const int* blk_tet0,
                                                                     const int* blk_vptr, const short* tet_loc,
                                                                     const int4* tets, const float* U, int N,
                                                                     float* partial, double* eblk) {
    extern __shared__ __align__(16) float2 sm2[];
    const int blk = blockIdx.x, tid = threadIdx.x;
    const int col = blockIdx.y * (2 * kP2Threads) + 2 * tid;  // first of the two columns (N is even)
    const int e0 = blk_tet0[blk], ne = blk_tet0[blk + 1] - e0;
    const int v0 = blk_vptr[blk], nv = blk_vptr[blk + 1] - v0;
    float2* acc = sm2;                                  // [(nv + 1) * 3][kP2Threads]; slot nv absorbs pinned corners
    float2* cs = acc + (nv + 1) * 3 * kP2Threads;       // [kTBE][kP2Consts]
    int* vs = reinterpret_cast<int*>(cs + kTBE * kP2Consts);  // [kTBE][4] row offsets v * 3 * N
    int* los = vs + kTBE * 4;                           // [kTBE][4] accumulator offsets slot * 3 * kP2Threads
    for (int i = tid; i < (nv + 1) * 3 * kP2Threads; i += kP2Threads) acc[i] = make_float2(0.f, 0.f);
    for (int t = tid; t < ne; t += kP2Threads) {
        float rc[12];
#pragma unroll
        for (int q = 0; q < 12; ++q) rc[q] = rec[(size_t)(e0 + t) * 12 + q];
        float2* c = cs + t * kP2Consts;
        const float vol = rc[9], mu = rc[10], lam = rc[11];
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            c[q] = make_float2(rc[q], rc[q]);
            c[9 + q] = make_float2(vol * rc[q], vol * rc[q]);
        }
        const float k[8] = {0.375f * mu, -0.75f * mu, -0.5f * mu, 0.5f * lam, 0.75f * mu, 0.25f * mu, lam, vol};
#pragma unroll
        for (int q = 0; q < 8; ++q) c[18 + q] = make_float2(k[q], k[q]);
    }
    for (int i = tid; i < ne * 4; i += kP2Threads) {
        const int4 t = __ldg(tets + e0 + (i >> 2));
        const int kk = i & 3;
        vs[i] = (kk == 0 ? t.x : kk == 1 ? t.y : kk == 2 ? t.z : t.w) * 3 * N;
        const int lv = tet_loc[(size_t)e0 * 4 + i];
        los[i] = (lv >= 0 ? lv : nv) * 3 * kP2Threads;
    }
    __syncthreads();
    if (col >= N) return;
    const float* Uc[3] = {U + col, U + col + N, U + col + 2 * (size_t)N};  // per component: one 64-bit add per load
    float2 esum = make_float2(0.f, 0.f);
    float2 un[12];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int c = 0; c < 3; ++c) un[kk * 3 + c] = __ldg(reinterpret_cast<const float2*>(Uc[c] + vs[kk]));
    for (int e = 0; e < ne; ++e) {
        float2 u[12];
#pragma unroll
        for (int q = 0; q < 12; ++q) u[q] = un[q];
        if (e + 1 < ne) {
            const int4 vn = *reinterpret_cast<const int4*>(vs + (e + 1) * 4);
            const int vv[4] = {vn.x, vn.y, vn.z, vn.w};
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                for (int c = 0; c < 3; ++c) un[kk * 3 + c] = __ldg(reinterpret_cast<const float2*>(Uc[c] + vv[kk]));
        }
        const int4 o4 = *reinterpret_cast<const int4*>(los + e * 4);
        const int off[4] = {o4.x, o4.y, o4.z, o4.w};
        float2* at = acc + tid;
        float2 old[12];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int a = 0; a < 3; ++a) old[k * 3 + a] = at[off[k] + a * kP2Threads];
        float2 c[kP2Consts];  // the tet's constant pairs: 13 16-byte broadcast loads
#pragma unroll
        for (int k = 0; k < kP2Consts / 2; ++k) {
            const float4 t = *reinterpret_cast<const float4*>(cs + e * kP2Consts + 2 * k);
            c[2 * k] = make_float2(t.x, t.y);
            c[2 * k + 1] = make_float2(t.z, t.w);
        }
        // D = [u1 - u0, u2 - u0, u3 - u0] (row a = component), A = D Dm^-1
        float2 A[9];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float2 d0 = p2sub(u[3 + a], u[a]), d1 = p2sub(u[6 + a], u[a]), d2 = p2sub(u[9 + a], u[a]);
#pragma unroll
            for (int b = 0; b < 3; ++b) A[a * 3 + b] = p2fma(d2, c[6 + b], p2fma(d1, c[3 + b], p2mul(d0, c[b])));
        }
        const float2 trA = p2add(p2add(A[0], A[4]), A[8]);
        float2 q = p2mul(A[0], A[0]);
#pragma unroll
        for (int k = 1; k < 9; ++k) q = p2fma(A[k], A[k], q);
        float2 cA[9];  // cofactors of A
        cA[0] = p2fms(A[4], A[8], p2mul(A[7], A[5]));
        cA[3] = p2fms(A[7], A[2], p2mul(A[1], A[8]));
        cA[6] = p2fms(A[1], A[5], p2mul(A[4], A[2]));
        cA[1] = p2fms(A[5], A[6], p2mul(A[8], A[3]));
        cA[4] = p2fms(A[8], A[0], p2mul(A[2], A[6]));
        cA[7] = p2fms(A[2], A[3], p2mul(A[5], A[0]));
        cA[2] = p2fms(A[3], A[7], p2mul(A[6], A[4]));
        cA[5] = p2fms(A[6], A[1], p2mul(A[0], A[7]));
        cA[8] = p2fms(A[0], A[4], p2mul(A[3], A[1]));
        const float2 m2 = p2add(p2add(cA[0], cA[4]), cA[8]);  // sum of the principal 2 x 2 minors
        const float2 detA = p2fma(A[6], cA[6], p2fma(A[3], cA[3], p2mul(A[0], cA[0])));
        const float2 md = p2add(m2, detA);
        const float2 jm1 = p2add(trA, md);
        const float2 imin = p2fma(make_float2(2.f, 2.f), trA, q);  // I - 3
        // L(x) = log1p(x) - x at x = (I - 3) / 4: log1p_minus_x's series for both columns at once, its
        // log1pf branch per column beyond |x| = 0.05
        const float2 x = p2mul(make_float2(0.25f, 0.25f), imin);
        float2 L = p2fma(x, make_float2(1.0f / 7.0f, 1.0f / 7.0f), make_float2(-1.0f / 6.0f, -1.0f / 6.0f));
        L = p2fma(x, L, make_float2(0.2f, 0.2f));
        L = p2fma(x, L, make_float2(-0.25f, -0.25f));
        L = p2fma(x, L, make_float2(1.0f / 3.0f, 1.0f / 3.0f));
        L = p2fma(x, L, make_float2(-0.5f, -0.5f));
        L = p2mul(p2mul(x, x), L);
        if (fabsf(x.x) >= 5e-2f) L.x = log1pf(x.x) - x.x;
        if (fabsf(x.y) >= 5e-2f) L.y = log1pf(x.y) - x.y;
        // psi = 3/8 mu q - 3/4 mu (m2 + det A) - 1/2 mu L + 1/2 lambda (J - 1)^2
        float2 psi = p2mul(c[18], q);
        psi = p2fma(c[19], md, psi);
        psi = p2fma(c[20], L, psi);
        psi = p2fma(c[21], p2mul(jm1, jm1), psi);
        esum = p2fma(c[25], psi, esum);
        const float2 c2 = p2mul(c[23], make_float2(__fdividef(imin.x, 4.f + imin.x), __fdividef(imin.y, 4.f + imin.y)));
        const float2 c3 = p2mul(c[24], jm1);
        const float2 alpha = p2add(c[22], c2), beta = p2sub(c[22], c3);
        const float2 kappa = p2fms(p2neg(beta), trA, p2neg(p2add(c2, c3)));  // c2 + c3 - beta tr A
        float2 Pm[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                Pm[a * 3 + b] = p2fma(alpha, A[a * 3 + b], p2mul(beta, p2sub(A[b * 3 + a], cA[a * 3 + b])));
                if (a == b) Pm[a * 3 + b] = p2add(Pm[a * 3 + b], kappa);
            }
        // forces: vertex k + 1 gets P (vol Dm^-1)[k][:]^T, vertex 0 minus their sum.  The four corners of a
        // tet are distinct vertices, so the 12 accumulator entries are read up front (independent loads,
        // issued before the arithmetic above needs them) and written back together.
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float2 s0 = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float2 hv = p2fma(Pm[a * 3 + 2], c[9 + k * 3 + 2],
                                        p2fma(Pm[a * 3 + 1], c[9 + k * 3 + 1], p2mul(Pm[a * 3 + 0], c[9 + k * 3 + 0])));
                s0 = k == 0 ? hv : p2add(s0, hv);
                old[(k + 1) * 3 + a] = p2add(old[(k + 1) * 3 + a], hv);
            }
            old[a] = p2sub(old[a], s0);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int a = 0; a < 3; ++a) at[off[k] + a * kP2Threads] = old[k * 3 + a];
    }
    for (int i = 0; i < nv * 3; ++i)
        *reinterpret_cast<float2*>(partial + ((size_t)(v0 * 3) + i) * N + col) = acc[i * kP2Threads + tid];
    eblk[(size_t)blk * N + col] = (double)esum.x;
    eblk[(size_t)blk * N + col + 1] = (double)esum.y;
}

// T[row][N] = s (sum of the vertex's block partials in block order + inertia).
__global__ void combine_kernel(int n, int N, const int* vslot_ptr, const int* vslot, const float* partial,
                               const float* rin, int has_inertia, const double* eprow, float* T) {
    const size_t total = (size_t)n * N;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const int row = (int)(idx / N), col = (int)(idx % N);
        const int f = row / 3, c = row - 3 * f;
        double g = 0.0;
        for (int k = vslot_ptr[f]; k < vslot_ptr[f + 1]; ++k) g += partial[((size_t)vslot[k] * 3 + c) * N + col];
        if (has_inertia) g += rin[idx];
        T[idx] = (float)(g * eprow[(size_t)row * 6 + 1]);
    }
}

// combine_kernel with its output written straight into the tcgen05 VJP B operand: T[row][col]
// as a tf32 hi/lo pair in the K-major core-matrix tiles (B row = col, K = row; lsb_tc.cuh).
__global__ void combine_pack_kernel(int n, int N, const int* vslot_ptr, const int* vslot, const float* partial,
                                    const float* rin, int has_inertia, const double* eprow, float* B2) {
    // thread = (4 consecutive rows = one 16-byte core-matrix chunk, 4 consecutive columns): every
    // partial / inertia read is a 16-byte load (4 columns), so a warp moves 512 B per load; the
    // per-(row, column) sums keep the block order of combine_kernel
    const int nq = (n + 3) / 4, ncq = N / 4;  // N is a multiple of 4 (column chunks of 64 / 128 / 256)
    const size_t total = (size_t)nq * ncq;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const int q4 = (int)(idx / ncq), col0 = 4 * (int)(idx % ncq);
        float x[4][4];  // [row e][column j]
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int row = 4 * q4 + e;
#pragma unroll
            for (int j = 0; j < 4; ++j) x[e][j] = 0.f;
            if (row < n) {
                const int f = row / 3, c = row - 3 * f;
                double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
                const int kb = __ldg(vslot_ptr + f), ke = __ldg(vslot_ptr + f + 1);
                for (int k = kb; k < ke; ++k) {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(partial + ((size_t)__ldg(vslot + k) * 3 + c) * N + col0));
                    g0 += v.x;
                    g1 += v.y;
                    g2 += v.z;
                    g3 += v.w;
                }
                if (has_inertia) {
                    const float4 ri = __ldg(reinterpret_cast<const float4*>(rin + (size_t)row * N + col0));
                    g0 += ri.x;
                    g1 += ri.y;
                    g2 += ri.z;
                    g3 += ri.w;
                }
                const double sc = __ldg(eprow + (size_t)row * 6 + 1);
                x[e][0] = (float)(g0 * sc);
                x[e][1] = (float)(g1 * sc);
                x[e][2] = (float)(g2 * sc);
                x[e][3] = (float)(g3 * sc);
            }
        }
        const int row0 = 4 * q4;
        float* blk = B2 + (size_t)(row0 / tc::kSliceK) * tc::slice_floats(N);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float hi[4], lo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                hi[e] = tc::tf32_rna(x[e][j]);
                lo[e] = x[e][j] - hi[e];
            }
            const size_t o = tc::core_off(col0 + j, row0 % tc::kSliceK, N);  // 16-byte aligned chunk of 4 rows
            *reinterpret_cast<float4*>(blk + o) = make_float4(hi[0], hi[1], hi[2], hi[3]);
            *reinterpret_cast<float4*>(blk + (size_t)N * tc::kSliceK + o) = make_float4(lo[0], lo[1], lo[2], lo[3]);
        }
    }
}

// E[b] = sum of inertia partials + element block partials (fixed order, fp64):
// block = column; 256 threads stride the partial rows, fixed-tree block sum.
__global__ void __launch_bounds__(256) energy_reduce_kernel(int N, int nrow_tiles, const double* epart, int nblk,
                                                            const double* eblk, int has_inertia, double* E) {
    __shared__ double red[32];
    const int col = blockIdx.x;
    double s = 0.0;
    int b = threadIdx.x;
    for (; b + 7 * (int)blockDim.x < nblk; b += 8 * blockDim.x) {  // 8 loads in flight, same order
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldg(eblk + (size_t)(b + k * blockDim.x) * N + col);
#pragma unroll
        for (int k = 0; k < 8; ++k) s += v[k];
    }
    for (; b < nblk; b += blockDim.x) s += eblk[(size_t)b * N + col];
    if (has_inertia)
        for (int b = threadIdx.x; b < nrow_tiles; b += blockDim.x) s += epart[(size_t)b * N + col];
    const double tot = block_sum(s, red);
    if (threadIdx.x == 0) E[col] = tot;
}


// ================================================================ second order (config 5)
// Hidden forward with first and second tangents.  Per point p the column block
// of X is [y | P_1..P_r | S_(a,b), a <= b] (1 + r + r(r+1)/2 columns); after the
// GEMM Q = W X, this applies the activation rule per row:
//   y' = phi(a), P'_a = phi'(a) Q_a, S'_ab = phi''(a) Q_a Q_b + phi'(a) Q_ab.
__global__ void tangent_act_kernel(int R, int P, int r, int cols, const float* Q, const double* bias, int act,
                                   float* X) {
    const size_t total = (size_t)R * P * cols;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx % cols);
        const size_t ip = idx / cols;
        const int i = (int)(ip / P);
        const float* q = Q + ip * cols;
        const double a = (double)q[0] + bias[i];
        float v;
        if (j == 0) {
            v = (float)act_eval(act, a, 0);
        } else if (j <= r) {
            v = (float)act_eval(act, a, 1) * q[j];
        } else {
            int aa = 0, rem = j - 1 - r;
            while (rem >= r - aa) {
                rem -= r - aa;
                ++aa;
            }
            const int bb = aa + rem;
            v = (float)act_eval(act, a, 2) * q[1 + aa] * q[1 + bb] + (float)act_eval(act, a, 1) * q[j];
        }
        X[idx] = v;
    }
}

// X0 = [z | I | 0] per point.
__global__ void tangent_init_kernel(int r, int P, int cols, const float* Zt /*[r][P]*/, float* X) {
    const int total = r * P * cols;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int i = idx / (P * cols), rem = idx % (P * cols), p = rem / cols, j = rem % cols;
        float v = 0.f;
        if (j == 0) v = Zt[(size_t)i * P + p];
        else if (j == 1 + i) v = 1.f;
        X[idx] = v;
    }
}

// B operand of the output GEMM: [h][P*(1+r)] = the y and P columns of X_L.
__global__ void tangent_pack_kernel(int h, int P, int r, int cols, const float* X, float* B) {
    const int w = 1 + r;
    const int total = h * P * w;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        // column order [y (P) | tangents (P x r)]: the J part of an output row is one contiguous run of Jv
        const int i = idx / (P * w), rem = idx % (P * w);
        const int p = rem < P ? rem : (rem - P) / r, j = rem < P ? 0 : 1 + (rem - P) % r;
        B[idx] = X[(size_t)i * P * cols + (size_t)p * cols + j];
    }
}

// Pinned rows of the chunk buffers for chunks of P points: U = pin displacement, J = 0.
__global__ void pinned_rows_kernel(int np, int P, int r, const int* pin_v, const float* pin_d, float* U, float* Jv) {
    const size_t total = (size_t)np * 3 * P;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx / (3 * (size_t)P)), k = (int)((idx / P) % 3), p = (int)(idx % P);
        const size_t row = ((size_t)pin_v[i] * 3 + k) * P + p;
        U[row] = pin_d[3 * i + k];
        if (Jv)
            for (int a = 0; a < r; ++a) Jv[row * r + a] = 0.f;
    }
}

// u -> U[v][3][P]; J_ia = s_i C_ia -> Jv[v][3][P][r] (pinned rows: pin displacement, zero J).
// With inertia (objective Hessian): rin[row][p] = m (u - (qbar - X)) / h^2, the inertia part
// of the full-space residual whose contraction with the decoder curvature enters H.
__global__ void tangent_out_kernel(int n, int P, int r, const float* C, const double* eprow, float* U, float* Jv,
                                   int inertia, double inv_dt2, float* rin) {
    const int w = 1 + r;
    const int total = n * P;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int row = idx / P, p = idx % P;
        const double* e6 = eprow + (size_t)row * 6;
        const float* crow = C + (size_t)row * P * w;   // [u (P) | J (P x r)] (tangent_pack_kernel)
        const float* c = crow + P + (size_t)p * r - 1;  // c[1 + a] = J column a of point p
        const int slot = (int)e6[4];
        const size_t vc = (size_t)(slot >> 2) * 3 + (slot & 3);
        const double u = e6[1] * ((double)crow[p] + e6[0]) + e6[2];
        U[vc * P + p] = (float)u;
        if (inertia) rin[(size_t)row * P + p] = (float)(inv_dt2 * e6[3] * (u - e6[5]));
        float* jo = Jv + (vc * P + p) * r;
        if ((r & 3) == 0) {  // 16-byte stores (rows of r floats are 16-byte aligned)
            const double sc = e6[1];
            for (int a = 0; a < r; a += 4)
                *reinterpret_cast<float4*>(jo + a) = make_float4((float)(sc * c[1 + a]), (float)(sc * c[2 + a]),
                                                                 (float)(sc * c[3 + a]), (float)(sc * c[4 + a]));
        } else {
            for (int a = 0; a < r; ++a) jo[a] = (float)(e6[1] * c[1 + a]);
        }
    }
}

// Inertia block of the objective Hessian (reduced_solver.cpp:218-221):
//   C[p][ab] += sum_rows (m / h^2) J_a J_b,  a <= b.
// CTA per point, thread per pair; rows streamed through shared-memory tiles of J (row
// order fixed -> deterministic).
__global__ void __launch_bounds__(256) inertia_hess_kernel(int n, int P, int r, const double* eprow, const float* Jv,
                                                           double inv_dt2, double* C) {
    constexpr int TRW = 64;
    __shared__ float Js[TRW][33];
    __shared__ float ms[TRW];
    const int p = blockIdx.x, tid = threadIdx.x;
    const int npair = r * (r + 1) / 2;
    int a = 0, bb = 0;
    if (tid < npair) {
        int rem = tid;
        while (rem >= r - a) {
            rem -= r - a;
            ++a;
        }
        bb = a + rem;
    }
    double acc = 0.0;
    for (int r0 = 0; r0 < n; r0 += TRW) {
        const int nr = min(TRW, n - r0);
        __syncthreads();
        for (int i = tid; i < nr * r; i += blockDim.x) {
            const int rr = i / r, k = i % r;
            const int row = r0 + rr;
            const int slot = (int)eprow[(size_t)row * 6 + 4];
            const size_t vc = (size_t)(slot >> 2) * 3 + (slot & 3);
            Js[rr][k] = Jv[(vc * P + p) * r + k];
            if (k == 0) ms[rr] = (float)eprow[(size_t)row * 6 + 3];
        }
        __syncthreads();
        if (tid < npair) {
            float s = 0.f;
            for (int rr = 0; rr < nr; ++rr) s = fmaf(ms[rr] * Js[rr][a], Js[rr][bb], s);
            acc += (double)s;
        }
    }
    if (tid < npair) C[(size_t)p * npair + tid] += inv_dt2 * acc;
}

// Order-2 Lipschitz loss backward on the device (losses.cpp:196-213 through scale / dot / sub, then
// symmetric_from_entries, tape.cpp:212-222): per pair q (points 2q, 2q + 1, factor f = 2 / (P |dz|^2)),
// Hbar = +-f (H1 - H2) as fp32 rows, ebar_ab = Hbar_ab + Hbar_ba (a < b) / Hbar_aa, and the pair's
// |H1 - H2|^2 (fixed-order block sum) for the loss.  One CTA per pair.  With hb = eb = null only the
// |H1 - H2|^2 (the loss-only path uses the same reduction, so loss and loss + gradient agree bitwise).
__global__ void __launch_bounds__(256) lipschitz_dldh_kernel(int npairs, int r, const double* H, const double* fac,
                                                             float* hb, float* eb, double* d2out) {
    __shared__ double red[32];
    const int q = blockIdx.x;
    if (q >= npairs) return;
    const int rr = r * r, npair = r * (r + 1) / 2;
    const double* H1 = H + (size_t)(2 * q) * rr;
    const double* H2 = H1 + rr;
    const double f = fac ? fac[q] : 0.0;
    double d2 = 0.0;
    for (int k = threadIdx.x; k < rr; k += blockDim.x) {
        const double d = H1[k] - H2[k];
        d2 += d * d;
        if (hb) {
            hb[(size_t)(2 * q) * rr + k] = (float)(f * d);
            hb[(size_t)(2 * q + 1) * rr + k] = (float)(-f * d);
        }
    }
    for (int sidx = threadIdx.x; eb && sidx < npair; sidx += blockDim.x) {
        int a = 0, rem = sidx;
        while (rem >= r - a) {
            rem -= r - a;
            ++a;
        }
        const int b = a + rem;
        const double hab = f * (H1[a * r + b] - H2[a * r + b]);
        const double v = a != b ? hab + f * (H1[b * r + a] - H2[b * r + a]) : hab;
        eb[(size_t)(2 * q) * npair + sidx] = (float)v;
        eb[(size_t)(2 * q + 1) * npair + sidx] = (float)(-v);
    }
    const double t = block_sum(d2, red);
    if (threadIdx.x == 0) d2out[q] = t;
}

// Element Hessian contraction.  CTA = (block of kTB tets, GP = 128/R points).  Tets go
// in batches of R: first thread (point pl, t) forms, once per (tet, point), F, cof(F),
// the SNH derivatives and the element's elastic forces vol B^T P(F) into shared memory;
// then per tet thread (pl, direction b) forms the K = 11 rows of its column of
//   D  = [dF_b (9), alpha_b = gI.dF_b, beta_b = gJ.dF_b]
//   M' = vol [2 psi_I dF_b + psi_J dcof[dF_b], psi_II alpha_b, lambda beta_b]
// (double-buffered, one barrier per tet) and lanes own local dofs b, b + R, ... (< 12)
// of the force accumulation (tet order, as the reference's assemble).  The contraction
//   C_ab += sum_k D[k][a] M'[k][b]
//         = vol (dF_a : M_b) + vol psi_II alpha_a alpha_b + vol lambda beta_a beta_b
// runs on the tensor cores as mma.sync m16n8k8 TF32 with 3xTF32 splitting (fp32-level
// accuracy), fragments read straight from the [dir][12] rows (conflict-free); each warp
// owns GP / 4 points; the a <= b entries are written out.
__device__ __forceinline__ uint32_t tf32_bits(float x) {
    uint32_t u;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
    return u;
}
// 3xTF32 operand split by truncation: hi keeps the top 10 mantissa bits (one LOP3), lo = x - hi
// is exact in fp32 and the MMA reads its top bits; hi lo' + lo hi' + hi hi' then carries ~22
// bits (~2.4e-7 relative), against the 1e-4 bar of the Hessian path.  cvt.rna.tf32 (the
// round-to-nearest form) lowers to an FSETP / SEL / integer sequence per conversion: with 64
// conversions per tet it was the largest instruction block of the contraction (c5 107 -> 96 ms).
// Staging the block's Jacobian rows in shared memory instead of the one-tet-ahead L2 prefetch
// was measured slower (99 ms: two CTAs per SM instead of four).
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    hi = __float_as_uint(x) & 0xffffe000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_tf32_16x8x8(float* c, const uint32_t* a, const uint32_t* b) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int R>
__global__ void __launch_bounds__(128) elem_hess2_kernel(const int4* tets, const float* rec, const int* blk_tet0,
                                                        const int* blk_vptr, const short* tet_loc,
                                                        const int* blk_aptr, const int* blk_avert,
                                                        const short* tet_aloc, const float* U, const float* Jv,
                                                        int P, float* Cpart, float* gpart) {
    constexpr int GP = 128 / R;               // points per CTA
    constexpr int NPAIR = R * (R + 1) / 2;
    constexpr int NH = 33;                    // batch record: F 9, cof 9, psiI, psiII, psiJ, forces 12
    constexpr int PPW = GP / 4;               // points per warp (tensor-core contraction)
    constexpr int MT = R >= 16 ? R / 16 : 1;  // 16-row m tiles (R = 8: rows 8..15 are zero)
    constexpr int NT = R / 8;                 // 8-column n tiles
    __shared__ __align__(16) float sh_dF[2][GP][R][12];  // D rows per direction (k 0..11)
    __shared__ __align__(16) float sh_M[2][GP][R][12];   // M' rows per direction
    __shared__ __align__(16) float sh_rec[kTB][12];   // the block's records
    __shared__ int sh_off[kTB][8];  // accg offsets of the free slots (pinned -> scratch slot nv) (4), Us offsets of the touched slots (4)
    __shared__ int4 sh_tq[kTB];     // the block's vertex ids: the one-tet-ahead J prefetch reads them from here
    __shared__ float sh_b[R][GP][NH];
    extern __shared__ __align__(16) float dyn[];
    const int tid = threadIdx.x;
    const int pl = tid / R, b = tid % R;
    const int p0 = blockIdx.y * GP;
    const int blk = blockIdx.x;
    const int e0 = blk_tet0[blk], e1 = blk_tet0[blk + 1];
    const int v0 = blk_vptr[blk], nv = blk_vptr[blk + 1] - v0;
    const int a0 = blk_aptr[blk], nva = blk_aptr[blk + 1] - a0;
    float* Us = dyn;                            // [nva][3][GP]
    float* accg = Us + (size_t)nva * 3 * GP;    // [nv][3][GP]
    static_assert(GP % 4 == 0, "16-byte staging of U");
    for (int i = tid; i < nva * 3 * (GP / 4); i += 128) {
        const int vcl = i / (GP / 4), k4 = i % (GP / 4);
        const int va = __ldg(blk_avert + a0 + vcl / 3), c = vcl % 3;
        cp_async16(Us + (size_t)vcl * GP + 4 * k4, U + ((size_t)va * 3 + c) * P + p0 + 4 * k4);
    }
    for (int i = tid; i < (nv + 1) * 3 * GP; i += 128) accg[i] = 0.f;
    for (int i = tid; i < (e1 - e0) * 12; i += 128) sh_rec[i / 12][i % 12] = rec[(size_t)e0 * 12 + i];
    for (int i = tid; i < (e1 - e0) * 4; i += 128) {
        const int lv = tet_loc[(size_t)e0 * 4 + i];
        sh_off[i >> 2][i & 3] = (lv >= 0 ? lv : nv) * 3 * GP;
        sh_off[i >> 2][4 + (i & 3)] = tet_aloc[(size_t)e0 * 4 + i] * 3 * GP;
    }
    for (int i = tid; i < e1 - e0; i += 128) sh_tq[i] = __ldg(tets + e0 + i);
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    float cacc[PPW][MT][NT][4];
#pragma unroll
    for (int pp = 0; pp < PPW; ++pp)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int q = 0; q < 4; ++q) cacc[pp][mt][nt][q] = 0.f;
    cp_async_wait_all();
    __syncthreads();
    const bool live = p0 + pl < P;
    // this thread's Jacobian column (point pl, direction b) of the current tet's 12 dofs,
    // read from L2 one tet ahead (coalesced over the CTA's points x directions)
    const float* Jp = Jv + ((size_t)(p0 + pl)) * R + b;
    const size_t jstride = (size_t)P * R;  // per (vertex, component) row
    // two-deep register ring: dun for tet e + 1, dun2 for tet e + 2 (L2 / DRAM latency exceeds
    // one tet's work)
    float dun[12], dun2[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) dun[q] = dun2[q] = 0.f;
    if (live && e0 < e1) {
        const int4 t = sh_tq[0];
        const int vv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int a = 0; a < 3; ++a) dun[k * 3 + a] = __ldg(Jp + ((size_t)vv[k] * 3 + a) * jstride);
    }
    if (live && e0 + 1 < e1) {
        const int4 t = sh_tq[1];
        const int vv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int a = 0; a < 3; ++a) dun2[k * 3 + a] = __ldg(Jp + ((size_t)vv[k] * 3 + a) * jstride);
    }
    for (int eb = e0; eb < e1; eb += R) {
        // ---- batch phase: thread (pl, t = b) forms the per-(tet, point) quantities of tet eb + b
        {
            const int e = eb + b;
            if (live && e < e1) {
                float rc[12], uu[12];
#pragma unroll
                for (int qq = 0; qq < 12; ++qq) rc[qq] = sh_rec[e - e0][qq];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int uo = sh_off[e - e0][4 + k] + pl;
#pragma unroll
                    for (int a = 0; a < 3; ++a) uu[k * 3 + a] = Us[uo + a * GP];
                }
                float A[9];
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int c2 = 0; c2 < 3; ++c2)
                        A[a * 3 + c2] = (uu[3 + a] - uu[a]) * rc[c2] + (uu[6 + a] - uu[a]) * rc[3 + c2] +
                                        (uu[9 + a] - uu[a]) * rc[6 + c2];
                float F[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) F[k] = A[k] + ((k % 4) == 0 ? 1.f : 0.f);
                float cof[9];
                cof[0] = F[4] * F[8] - F[7] * F[5];
                cof[3] = F[7] * F[2] - F[1] * F[8];
                cof[6] = F[1] * F[5] - F[4] * F[2];
                cof[1] = F[5] * F[6] - F[8] * F[3];
                cof[4] = F[8] * F[0] - F[2] * F[6];
                cof[7] = F[2] * F[3] - F[5] * F[0];
                cof[2] = F[3] * F[7] - F[6] * F[4];
                cof[5] = F[6] * F[1] - F[0] * F[7];
                cof[8] = F[0] * F[4] - F[3] * F[1];
                const float vol = rc[9], mu = rc[10], lam = rc[11];
                const float trA = A[0] + A[4] + A[8];
                float q = 0.f;
#pragma unroll
                for (int k = 0; k < 9; ++k) q += A[k] * A[k];
                const float m2 = A[0] * A[4] - A[1] * A[3] + A[0] * A[8] - A[2] * A[6] + A[4] * A[8] - A[5] * A[7];
                const float detA = A[0] * (A[4] * A[8] - A[7] * A[5]) - A[3] * (A[1] * A[8] - A[7] * A[2]) +
                                   A[6] * (A[1] * A[5] - A[4] * A[2]);
                const float jm1 = trA + m2 + detA;
                const float uI = 4.f + 2.f * trA + q;  // I + 1
                float* o = sh_b[b][pl];
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    o[k] = F[k];
                    o[9 + k] = cof[k];
                }
                o[18] = 0.5f * mu * (1.f - 1.f / uI);
                o[19] = 0.5f * mu / (uI * uI);
                o[20] = lam * jm1 - 0.75f * mu;
                // elastic forces vol B^T P (cancellation-free first Piola stress)
                float cA[9];
                cA[0] = A[4] * A[8] - A[7] * A[5];
                cA[3] = A[7] * A[2] - A[1] * A[8];
                cA[6] = A[1] * A[5] - A[4] * A[2];
                cA[1] = A[5] * A[6] - A[8] * A[3];
                cA[4] = A[8] * A[0] - A[2] * A[6];
                cA[7] = A[2] * A[3] - A[5] * A[0];
                cA[2] = A[3] * A[7] - A[6] * A[4];
                cA[5] = A[6] * A[1] - A[0] * A[7];
                cA[8] = A[0] * A[4] - A[3] * A[1];
                const float c1 = 0.75f * mu, c2 = mu * (2.f * trA + q) / (4.f * uI), c3 = lam * jm1;
#pragma unroll
                for (int aa = 0; aa < 3; ++aa) {
                    float Pa[3];
#pragma unroll
                    for (int bb = 0; bb < 3; ++bb) {
                        const float id = aa == bb ? 1.f : 0.f;
                        Pa[bb] = c1 * (A[aa * 3 + bb] + A[bb * 3 + aa] - trA * id - cA[aa * 3 + bb]) +
                                 c2 * F[aa * 3 + bb] + c3 * cof[aa * 3 + bb];
                    }
                    float hc[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        hc[c] = vol * (Pa[0] * rc[c * 3 + 0] + Pa[1] * rc[c * 3 + 1] + Pa[2] * rc[c * 3 + 2]);
                    float s0 = 0.f;
                    s0 += hc[0];
                    s0 += hc[1];
                    s0 += hc[2];
                    o[21 + aa] = -s0;
#pragma unroll
                    for (int c = 0; c < 3; ++c) o[21 + (c + 1) * 3 + aa] = hc[c];
                }
            }
        }
        __syncthreads();
        const int nbt = min(R, e1 - eb);
        for (int tb = 0; tb < nbt; ++tb) {
            const int e = eb + tb;
            const int buf = (e - e0) & 1;
            if (live) {
                const float* bq = sh_b[tb][pl];
                float rc[9];
#pragma unroll
                for (int qq = 0; qq < 9; ++qq) rc[qq] = sh_rec[e - e0][qq];
                float duc[12];
#pragma unroll
                for (int q = 0; q < 12; ++q) {
                    duc[q] = dun[q];
                    dun[q] = dun2[q];
                }
                if (e + 2 < e1) {
                    const int4 t = sh_tq[e + 2 - e0];
                    const int vv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int a = 0; a < 3; ++a) dun2[k * 3 + a] = __ldg(Jp + ((size_t)vv[k] * 3 + a) * jstride);
                }
                float dA[9];
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int c2 = 0; c2 < 3; ++c2)
                        dA[a * 3 + c2] = (duc[3 + a] - duc[a]) * rc[c2] + (duc[6 + a] - duc[a]) * rc[3 + c2] +
                                         (duc[9 + a] - duc[a]) * rc[6 + c2];
                float F[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) F[k] = bq[k];
                float alpha = 0.f, beta = 0.f;
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    alpha += 2.f * F[k] * dA[k];
                    beta += bq[9 + k] * dA[k];
                }
                const float psiI = bq[18], psiJ = bq[20];
                float dc[9];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int ci = (c + 1) % 3, cj = (c + 2) % 3;
                    const float a1[3] = {F[ci], F[3 + ci], F[6 + ci]}, a2[3] = {F[cj], F[3 + cj], F[6 + cj]};
                    const float d1[3] = {dA[ci], dA[3 + ci], dA[6 + ci]}, d2[3] = {dA[cj], dA[3 + cj], dA[6 + cj]};
                    dc[0 * 3 + c] = d1[1] * a2[2] - d1[2] * a2[1] + a1[1] * d2[2] - a1[2] * d2[1];
                    dc[1 * 3 + c] = d1[2] * a2[0] - d1[0] * a2[2] + a1[2] * d2[0] - a1[0] * d2[2];
                    dc[2 * 3 + c] = d1[0] * a2[1] - d1[1] * a2[0] + a1[0] * d2[1] - a1[1] * d2[0];
                }
                const float vol = sh_rec[e - e0][9], lam = sh_rec[e - e0][11];
                float4* dFo = reinterpret_cast<float4*>(sh_dF[buf][pl][b]);
                float4* Mo = reinterpret_cast<float4*>(sh_M[buf][pl][b]);
                float Mv[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) Mv[k] = vol * (2.f * psiI * dA[k] + psiJ * dc[k]);
                dFo[0] = make_float4(dA[0], dA[1], dA[2], dA[3]);
                dFo[1] = make_float4(dA[4], dA[5], dA[6], dA[7]);
                dFo[2] = make_float4(dA[8], alpha, beta, 0.f);
                Mo[0] = make_float4(Mv[0], Mv[1], Mv[2], Mv[3]);
                Mo[1] = make_float4(Mv[4], Mv[5], Mv[6], Mv[7]);
                Mo[2] = make_float4(Mv[8], vol * bq[19] * alpha, vol * lam * beta, 0.f);
                // elastic forces: lanes own local dofs b, b + R, ... (< 12), tet order
#pragma unroll
                for (int d0 = 0; d0 < 12; d0 += R) {
                    const int d = d0 + b;
                    if (d < 12) accg[sh_off[e - e0][d / 3] + (d % 3) * GP + pl] += bq[21 + d];
                }
            }
            __syncthreads();
            // tensor-core contraction: warp owns points warp * PPW + pp; A = D^T (dir x k),
            // B = M' (k x dir); k-step 1 = rows 0..7, k-step 2 = rows 8..11 (12..15 zero)
#pragma unroll
            for (int pp = 0; pp < PPW; ++pp) {
                const int pc = warp * PPW + pp;
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const int k0 = ks * 8;
                    uint32_t ah[MT][4], al[MT][4], bh[NT][2], bl[NT][2];
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const float* r0 = sh_dF[buf][pc][mt * 16 + g];
                        const float x0 = r0[k0 + t4];
                        const float x2 = ks == 0 ? r0[k0 + 4 + t4] : 0.f;
                        float x1 = 0.f, x3 = 0.f;
                        if (R >= 16) {
                            const float* r1 = sh_dF[buf][pc][mt * 16 + 8 + g];
                            x1 = r1[k0 + t4];
                            x3 = ks == 0 ? r1[k0 + 4 + t4] : 0.f;
                        }
                        split_tf32(x0, ah[mt][0], al[mt][0]);
                        split_tf32(x1, ah[mt][1], al[mt][1]);
                        split_tf32(x2, ah[mt][2], al[mt][2]);
                        split_tf32(x3, ah[mt][3], al[mt][3]);
                    }
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        const float* rb = sh_M[buf][pc][nt * 8 + g];
                        const float y0 = rb[k0 + t4];
                        const float y1 = ks == 0 ? rb[k0 + 4 + t4] : 0.f;
                        split_tf32(y0, bh[nt][0], bl[nt][0]);
                        split_tf32(y1, bh[nt][1], bl[nt][1]);
                    }
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) {
                            mma_tf32_16x8x8(cacc[pp][mt][nt], al[mt], bh[nt]);
                            mma_tf32_16x8x8(cacc[pp][mt][nt], ah[mt], bl[nt]);
                            mma_tf32_16x8x8(cacc[pp][mt][nt], ah[mt], bh[nt]);
                        }
                }
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int pp = 0; pp < PPW; ++pp) {
        const int pc = warp * PPW + pp;
        if (p0 + pc >= P) continue;
        float* Co = Cpart + ((size_t)blk * P + p0 + pc) * NPAIR;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int a = mt * 16 + g + (q >= 2 ? 8 : 0), bb = nt * 8 + 2 * t4 + (q & 1);
                    if (a < R && a <= bb) Co[a * R - a * (a - 1) / 2 + (bb - a)] = cacc[pp][mt][nt][q];
                }
    }
    for (int i = tid; i < nv * 3 * GP; i += 128) {
        const int pp = i % GP;
        if (p0 + pp < P) gpart[((size_t)(v0 * 3) + i / GP) * P + p0 + pp] = accg[i];
    }
}

// ---- Element Hessian contraction, edge-space form (default; elem_hess2_kernel is the A/B fallback)
// For one (tet, point) the reduced Hessian block is a quadratic form in the EDGE differences of the
// Jacobian columns, E[b][(e, a)] = J[v_{e+1}, a][b] - J[v_0, a][b] (R directions x 9):
//     C_ab += sum_{kk, kk'} E[a][kk] H_E[kk][kk'] E[b][kk'],     H_E = Bd H_F Bd^T   (9 x 9, symmetric)
// with Bd the block-diagonal Dm^-1 map (dF[a][c] = sum_e E[(e, a)] Dm^-1[e][c]) and
//     H_F = vol (2 psi_I I + psi_J dcof/dF + 4 psi_II f f^T + lambda c c^T),  f = vec F, c = vec cof F
// -- the same contraction as D^T M' above (alpha = 2 f.dF, beta = c.dF), regrouped so that everything
// that depends on the direction is tensor-core work.  H_E is formed once per (tet, point) in fp32 by one
// thread (batch phase: thread = (point, tet of the batch)) and stored as its upper triangle; then per
// (tet, point) one warp runs two chained mma.sync m16n8k8 TF32 stages entirely in registers:
//     X = E H_E        (A = E from the fp32 edge differences of the L2-prefetched Jacobian rows, B = H_E)
//     C += E X^T       (A = E again; B = the accumulator fragments of X, reused directly: lane (g, t4) of
//                       an accumulator holds columns 2 t4, 2 t4 + 1, so every stage orders its K index as
//                       position t4 <-> kk = 2 t4, position t4 + 4 <-> kk = 2 t4 + 1 and no shuffle is needed)
// Every product is a 3xTF32 sum (hi lo' + lo hi' + hi hi', operands split by truncation: fp32-level accuracy).
// One TF32 pass is not enough: on a smooth (trained) decoder neighbouring tets carry nearly the same E and
// H_E, so their rounding errors are correlated and do not average out over the mesh (7.5e-4 against the
// oracle, tests/test_gpu_hessian.py::test_edge_space_hessian_smooth_decoder).  The ninth K component (one slot
// of a second k step) stays off the tensor cores: its rank-one terms X += e8 H_E[6][:] and C += e8 X[:, 6]^T
// are fp32 FMAs on the accumulator fragments (e8 and X[:, 6] reach the lanes by shuffles), which halves the
// MMA count (12 m16n8k8 per (tet, point) at r = 16).
// Forces are accumulated per warp for its own points in tet order (deterministic).
__device__ __forceinline__ uint32_t rn_tf32(float x) { return (__float_as_uint(x) + 0x1000u) & 0xffffe000u; }
__device__ __forceinline__ void mma_tf32_u(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                           uint32_t b1) {
    asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// N consecutive floats (N = 1, 2, 4; N-float aligned) through the read-only path
template <int N>
__device__ __forceinline__ void ldg_vec(float* o, const float* p) {
    if constexpr (N == 1) {
        o[0] = __ldg(p);
    } else if constexpr (N == 2) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(p));
        o[0] = v.x;
        o[1] = v.y;
    } else {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p));
        o[0] = v.x;
        o[1] = v.y;
        o[2] = v.z;
        o[3] = v.w;
    }
}

#ifndef LSB_H3_MINB
#define LSB_H3_MINB 4
#endif
template <int R>
__global__ void __launch_bounds__(128, LSB_H3_MINB) elem_hess3_kernel(const int4* tets, const float* rec, const int* blk_tet0,
                                                        const int* blk_vptr, const short* tet_loc,
                                                        const int* blk_aptr, const int* blk_avert,
                                                        const short* tet_aloc, const float* U, const float* Jv,
                                                        int P, float* Cpart, float* gpart) {
    constexpr int GP = 128 / R;               // points per CTA
    constexpr int NPAIR = R * (R + 1) / 2;
    constexpr int PPW = GP / 4;               // points per warp
    constexpr int MT = R >= 16 ? R / 16 : 1;  // 16-row m tiles (R = 8: rows 8..15 are zero)
    constexpr int NT = R / 8;                 // 8-column n tiles
    constexpr int NR = R >= 16 ? R / 8 : 1;   // 8-direction row groups a lane loads
    constexpr int HS = 60;  // floats per (tet, point) record: H_E upper triangle 45 (tf32), pad 3, forces 12
    __shared__ __align__(16) float sh_h[128][HS];    // [point * R + tet of the batch]: consecutive lanes of the batch
                                                     // phase write consecutive records (60-word stride: conflict-free)
    __shared__ __align__(16) float sh_rec[kTB][12];  // the block's records
    __shared__ int sh_off[kTB][8];  // accg offsets of the free slots (pinned -> scratch slot nv) (4), Us offsets (4)
    __shared__ int4 sh_tq[kTB];     // the block's vertex ids
    extern __shared__ __align__(16) float dyn[];
    const int tid = threadIdx.x;
    const int pl = tid / R, tb = tid % R;
    const int p0 = blockIdx.y * GP;
    const int blk = blockIdx.x;
    const int e0 = blk_tet0[blk], ne = blk_tet0[blk + 1] - e0;
    const int v0 = blk_vptr[blk], nv = blk_vptr[blk + 1] - v0;
    const int a0 = blk_aptr[blk], nva = blk_aptr[blk + 1] - a0;
    float* Us = dyn;                            // [nva][3][GP]
    float* accg = Us + (size_t)nva * 3 * GP;    // [nv + 1][3][GP]
    static_assert(GP % 4 == 0, "16-byte staging of U");
    for (int i = tid; i < nva * 3 * (GP / 4); i += 128) {
        const int vcl = i / (GP / 4), k4 = i % (GP / 4);
        const int va = __ldg(blk_avert + a0 + vcl / 3), c = vcl % 3;
        cp_async16(Us + (size_t)vcl * GP + 4 * k4, U + ((size_t)va * 3 + c) * P + p0 + 4 * k4);
    }
    for (int i = tid; i < (nv + 1) * 3 * GP; i += 128) accg[i] = 0.f;
    for (int i = tid; i < ne * 12; i += 128) sh_rec[i / 12][i % 12] = rec[(size_t)e0 * 12 + i];
    for (int i = tid; i < ne * 4; i += 128) {
        const int lv = tet_loc[(size_t)e0 * 4 + i];
        sh_off[i >> 2][i & 3] = (lv >= 0 ? lv : nv) * 3 * GP;
        sh_off[i >> 2][4 + (i & 3)] = tet_aloc[(size_t)e0 * 4 + i] * 3 * GP;
    }
    for (int i = tid; i < ne; i += 128) sh_tq[i] = __ldg(tets + e0 + i);
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    float cacc[PPW][MT][NT][4];
#pragma unroll
    for (int pp = 0; pp < PPW; ++pp)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int q = 0; q < 4; ++q) cacc[pp][mt][nt][q] = 0.f;
    cp_async_wait_all();
    __syncthreads();
    // ---- lane constants of the tensor-core phase
    // K slots (kk = 3 e + a: edge e, component a) are dealt to the four t4 lanes so that a lane's slots
    // share Jacobian rows -- lanes 0..2 take component a = t4 of edges 0 and 1 (lane 0 also edge 2, its k-step-1
    // slot), lane 3 takes edge 2 of components 1 and 2: 14 row loads per quad instead of 18.  Any assignment
    // works as long as the H_E operand is permuted the same way (its offsets are per-lane constants) and the
    // accumulator column order matches: column 2 t4 <-> slot 0 of lane t4, 2 t4 + 1 <-> slot 1, column 8 <->
    // lane 0's slot 2.
    //   rows loaded per lane (vertex of the tet, component):        slots
    //   t4 = 0: R0 (1, 0)  R1 (2, 0)  R2 (3, 0)  R3 (0, 0)          R0 - R3, R1 - R3, R2 - R3
    //   t4 = 1: R0 (1, 1)  R1 (2, 1)             R3 (0, 1)          R0 - R3, R1 - R3
    //   t4 = 2: R0 (1, 2)  R1 (2, 2)             R3 (0, 2)          R0 - R3, R1 - R3
    //   t4 = 3: R0 (3, 1)  R1 (3, 2)  R2 (0, 2)  R3 (0, 1)          R0 - R3, R1 - R2
    const bool is3 = t4 == 3, slot2 = t4 == 0, has_r2 = slot2 || is3;
    const int kks[3] = {is3 ? 7 : t4, is3 ? 8 : 3 + t4, 6};   // kk of slots 0, 1 and (lane 0) 2
    const int rv[4] = {is3 ? 3 : 1, is3 ? 3 : 2, is3 ? 0 : 3, 0};           // vertex of the tet per row
    const int ra[4] = {is3 ? 1 : t4, is3 ? 2 : t4, is3 ? 2 : 0, is3 ? 1 : t4};  // component per row
    const size_t PR = (size_t)P * R;
    const float* jb[4];   // Jv + a PR + (first point of the warp) R + first direction of the lane
#pragma unroll
    for (int s = 0; s < 4; ++s) jb[s] = Jv + (size_t)ra[s] * PR + (size_t)(p0 + warp * PPW) * R + g * NR;
    const unsigned vstrideB = 3u * (unsigned)PR * (unsigned)sizeof(float);  // bytes per vertex of Jv
    // H_E upper-triangle offsets of this lane's B fragments; accumulator column c holds kk = colk(c)
    auto tri = [](int i, int j) {
        const int lo = i < j ? i : j, hi = i < j ? j : i;
        return lo * 9 - lo * (lo - 1) / 2 + (hi - lo);
    };
    auto colk = [](int c) { return c == 8 ? 6 : c == 6 ? 7 : c == 7 ? 8 : (c & 1) * 3 + (c >> 1); };
    const int hb00 = tri(kks[0], colk(g)), hb01 = tri(kks[1], colk(g));  // n tile 0 (column g), k step 0
    const int hb10 = tri(kks[0], colk(8)), hb11 = tri(kks[1], colk(8));  // n tile 1 (column 8: g == 0 only), k step 0
    // the ninth K component (kk = 6, lane 0's slot 2) stays off the tensor cores: its rank-one terms are fp32
    // FMAs on the accumulators (H_E row 6 at this lane's accumulator columns 2 t4, 2 t4 + 1 and at column 8)
    const int ht0 = tri(6, colk(2 * t4)), ht1 = tri(6, colk(2 * t4 + 1)), ht8 = tri(6, colk(8));
    const bool n8 = g == 0;
    bool livep[PPW];
#pragma unroll
    for (int pp = 0; pp < PPW; ++pp) livep[pp] = p0 + warp * PPW + pp < P;
    // raw Jacobian entries of one tet for this lane: [point][row R0..R3][direction of the lane]
    float rawA[PPW][4][NR], rawB[PPW][4][NR];
#pragma unroll
    for (int pp = 0; pp < PPW; ++pp)
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
            for (int q = 0; q < NR; ++q) rawA[pp][s][q] = rawB[pp][s][q] = 0.f;
    auto load_raw = [&](float (&raw)[PPW][4][NR], int el) {
        const int4 tq = sh_tq[el];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            if (s == 2 && !has_r2) continue;
            const unsigned v = (unsigned)(rv[s] == 0 ? tq.x : rv[s] == 1 ? tq.y : rv[s] == 2 ? tq.z : tq.w);
            const float* pr = reinterpret_cast<const float*>(reinterpret_cast<const char*>(jb[s]) + (unsigned long long)v * vstrideB);
#pragma unroll
            for (int pp = 0; pp < PPW; ++pp) {
                if (!livep[pp]) continue;
                ldg_vec<NR>(raw[pp][s], pr + pp * R);
            }
        }
    };
    auto process = [&](const float (&raw)[PPW][4][NR], int el, int tbl) {
        // forces of this tet: lanes own (point of the warp, local dof), tet order
        for (int i = lane; i < 12 * PPW; i += 32) {
            const int pp = i / 12, d = i % 12, pc = warp * PPW + pp;
            if (p0 + pc < P) accg[sh_off[el][d / 3] + (d % 3) * GP + pc] += sh_h[pc * R + tbl][48 + d];
        }
        __syncwarp();
#pragma unroll
        for (int pp = 0; pp < PPW; ++pp) {  // points beyond P run on zero Jacobian entries; their block is never stored
            const float* hr = sh_h[(warp * PPW + pp) * R + tbl];
            // B fragments of H_E (fp32 in the record), split hi + lo: every product below is the 3xTF32 sum
            // lo hi' + hi lo' + hi hi' (split_tf32), i.e. fp32-level accuracy.  A single TF32 pass is NOT enough:
            // with a smooth (trained) decoder neighbouring tets carry nearly the same E and H_E, their
            // rounding errors are correlated and do not average out over the mesh (7.5e-4 against the oracle on
            // tests/test_gpu_hessian.py::test_edge_space_hessian_smooth_decoder; 1.2e-5 only on the random
            // decoders of the configs).
            uint32_t bh[4], bl[4];
            split_tf32(hr[hb00], bh[0], bl[0]);
            split_tf32(hr[hb01], bh[1], bl[1]);
            split_tf32(n8 ? hr[hb10] : 0.f, bh[2], bl[2]);
            split_tf32(n8 ? hr[hb11] : 0.f, bh[3], bl[3]);
            const float hk0 = hr[ht0], hk1 = hr[ht1], hk8 = slot2 ? hr[ht8] : 0.f;
            uint32_t eh[MT][4], el2[MT][4];  // a0..a3 of the one k step (hi / lo)
            float e8[MT][2];                  // E[row][kk = 6] for rows g, g + 8 of every m tile (from lane t4 = 0)
            float X[MT][2][4];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const int q0 = R >= 16 ? 2 * mt : 0, q1 = NR > 1 ? q0 + 1 : 0;
                // slot 0 = R0 - R3, slot 1 = R1 - (lane 3: R2, else R3), slot 2 (lane 0) = R2 - R3
                float ev[4];
                ev[0] = raw[pp][0][q0] - raw[pp][3][q0];
                ev[2] = raw[pp][1][q0] - (is3 ? raw[pp][2][q0] : raw[pp][3][q0]);
                e8[mt][0] = __shfl_sync(0xffffffffu, raw[pp][2][q0] - raw[pp][3][q0], lane & ~3);
                if (R >= 16) {
                    ev[1] = raw[pp][0][q1] - raw[pp][3][q1];
                    ev[3] = raw[pp][1][q1] - (is3 ? raw[pp][2][q1] : raw[pp][3][q1]);
                    e8[mt][1] = __shfl_sync(0xffffffffu, raw[pp][2][q1] - raw[pp][3][q1], lane & ~3);
                } else {
                    ev[1] = ev[3] = 0.f;
                    e8[mt][1] = 0.f;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) split_tf32(ev[q], eh[mt][q], el2[mt][q]);
#pragma unroll
                for (int q = 0; q < 4; ++q) X[mt][0][q] = X[mt][1][q] = 0.f;
                // X = E H_E over the eight tensor-core K slots: n tile 0 (columns 0..7), n tile 1 (column 8);
                // small terms first
                mma_tf32_u(X[mt][0], el2[mt][0], el2[mt][1], el2[mt][2], el2[mt][3], bh[0], bh[1]);
                mma_tf32_u(X[mt][0], eh[mt][0], eh[mt][1], eh[mt][2], eh[mt][3], bl[0], bl[1]);
                mma_tf32_u(X[mt][0], eh[mt][0], eh[mt][1], eh[mt][2], eh[mt][3], bh[0], bh[1]);
                mma_tf32_u(X[mt][1], el2[mt][0], el2[mt][1], el2[mt][2], el2[mt][3], bh[2], bh[3]);
                mma_tf32_u(X[mt][1], eh[mt][0], eh[mt][1], eh[mt][2], eh[mt][3], bl[2], bl[3]);
                mma_tf32_u(X[mt][1], eh[mt][0], eh[mt][1], eh[mt][2], eh[mt][3], bh[2], bh[3]);
                // ninth K component: X[row][c] += E[row][6] H_E[6][c]
                X[mt][0][0] = fmaf(e8[mt][0], hk0, X[mt][0][0]);
                X[mt][0][1] = fmaf(e8[mt][0], hk1, X[mt][0][1]);
                X[mt][0][2] = fmaf(e8[mt][1], hk0, X[mt][0][2]);
                X[mt][0][3] = fmaf(e8[mt][1], hk1, X[mt][0][3]);
                X[mt][1][0] = fmaf(e8[mt][0], hk8, X[mt][1][0]);  // column 8 lives on the t4 = 0 lanes (hk8 = 0 elsewhere)
                X[mt][1][2] = fmaf(e8[mt][1], hk8, X[mt][1][2]);
            }
            // C += E X^T: n tile j = directions 8 j + g = rows of X (m tile j / 2, half j % 2)
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int mj = j >> 1, hj = (j & 1) * 2;
                uint32_t xh[2], xl[2];
                split_tf32(X[mj][0][hj], xh[0], xl[0]);
                split_tf32(X[mj][0][hj + 1], xh[1], xl[1]);
                // ninth K component: C[a][b] += E[a][6] X[b][6]; X[b][6] (accumulator column 8) of the rows
                // b = 8 j + 2 t4 + {0, 1} sits on the t4 = 0 lanes of those rows
                const float x80 = __shfl_sync(0xffffffffu, X[mj][1][hj], (2 * t4) * 4);
                const float x81 = __shfl_sync(0xffffffffu, X[mj][1][hj], (2 * t4 + 1) * 4);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    mma_tf32_u(cacc[pp][mt][j], el2[mt][0], el2[mt][1], el2[mt][2], el2[mt][3], xh[0], xh[1]);
                    mma_tf32_u(cacc[pp][mt][j], eh[mt][0], eh[mt][1], eh[mt][2], eh[mt][3], xl[0], xl[1]);
                    mma_tf32_u(cacc[pp][mt][j], eh[mt][0], eh[mt][1], eh[mt][2], eh[mt][3], xh[0], xh[1]);
                    cacc[pp][mt][j][0] = fmaf(e8[mt][0], x80, cacc[pp][mt][j][0]);
                    cacc[pp][mt][j][1] = fmaf(e8[mt][0], x81, cacc[pp][mt][j][1]);
                    cacc[pp][mt][j][2] = fmaf(e8[mt][1], x80, cacc[pp][mt][j][2]);
                    cacc[pp][mt][j][3] = fmaf(e8[mt][1], x81, cacc[pp][mt][j][3]);
                }
            }
        }
    };
    if (ne > 0) load_raw(rawA, 0);
    for (int eb = 0; eb < ne; eb += R) {
        __syncthreads();  // the previous batch's records are no longer read
        // ---- batch phase: thread (pl, tb) forms H_E and the forces of tet eb + tb at point pl
        {
            const int el = eb + tb;
            if (p0 + pl < P && el < ne) {
                float rc[12], uu[12];
#pragma unroll
                for (int qq = 0; qq < 12; ++qq) rc[qq] = sh_rec[el][qq];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int uo = sh_off[el][4 + k] + pl;
#pragma unroll
                    for (int a = 0; a < 3; ++a) uu[k * 3 + a] = Us[uo + a * GP];
                }
                float A[9];
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int c2 = 0; c2 < 3; ++c2)
                        A[a * 3 + c2] = (uu[3 + a] - uu[a]) * rc[c2] + (uu[6 + a] - uu[a]) * rc[3 + c2] +
                                        (uu[9 + a] - uu[a]) * rc[6 + c2];
                float F[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) F[k] = A[k] + ((k % 4) == 0 ? 1.f : 0.f);
                float cof[9];
                cof[0] = F[4] * F[8] - F[7] * F[5];
                cof[3] = F[7] * F[2] - F[1] * F[8];
                cof[6] = F[1] * F[5] - F[4] * F[2];
                cof[1] = F[5] * F[6] - F[8] * F[3];
                cof[4] = F[8] * F[0] - F[2] * F[6];
                cof[7] = F[2] * F[3] - F[5] * F[0];
                cof[2] = F[3] * F[7] - F[6] * F[4];
                cof[5] = F[6] * F[1] - F[0] * F[7];
                cof[8] = F[0] * F[4] - F[3] * F[1];
                const float vol = rc[9], mu = rc[10], lam = rc[11];
                const float trA = A[0] + A[4] + A[8];
                float q = 0.f;
#pragma unroll
                for (int k = 0; k < 9; ++k) q += A[k] * A[k];
                const float m2 = A[0] * A[4] - A[1] * A[3] + A[0] * A[8] - A[2] * A[6] + A[4] * A[8] - A[5] * A[7];
                const float detA = A[0] * (A[4] * A[8] - A[7] * A[5]) - A[3] * (A[1] * A[8] - A[7] * A[2]) +
                                   A[6] * (A[1] * A[5] - A[4] * A[2]);
                const float jm1 = trA + m2 + detA;
                const float uI = 4.f + 2.f * trA + q;  // I + 1
                const float inv_uI = 1.f / uI;
                float* o = sh_h[pl * R + tb];
                // elastic forces vol B^T P (cancellation-free first Piola stress)
                float cA[9];
                cA[0] = A[4] * A[8] - A[7] * A[5];
                cA[3] = A[7] * A[2] - A[1] * A[8];
                cA[6] = A[1] * A[5] - A[4] * A[2];
                cA[1] = A[5] * A[6] - A[8] * A[3];
                cA[4] = A[8] * A[0] - A[2] * A[6];
                cA[7] = A[2] * A[3] - A[5] * A[0];
                cA[2] = A[3] * A[7] - A[6] * A[4];
                cA[5] = A[6] * A[1] - A[0] * A[7];
                cA[8] = A[0] * A[4] - A[3] * A[1];
                const float c1 = 0.75f * mu, c2 = mu * (2.f * trA + q) * 0.25f * inv_uI, c3 = lam * jm1;
                float fo[12];
#pragma unroll
                for (int aa = 0; aa < 3; ++aa) {
                    float Pa[3];
#pragma unroll
                    for (int bb = 0; bb < 3; ++bb) {
                        const float id = aa == bb ? 1.f : 0.f;
                        Pa[bb] = c1 * (A[aa * 3 + bb] + A[bb * 3 + aa] - trA * id - cA[aa * 3 + bb]) +
                                 c2 * F[aa * 3 + bb] + c3 * cof[aa * 3 + bb];
                    }
                    float hc[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        hc[c] = vol * (Pa[0] * rc[c * 3 + 0] + Pa[1] * rc[c * 3 + 1] + Pa[2] * rc[c * 3 + 2]);
                    float s0 = 0.f;
                    s0 += hc[0];
                    s0 += hc[1];
                    s0 += hc[2];
                    fo[aa] = -s0;
#pragma unroll
                    for (int c = 0; c < 3; ++c) fo[(c + 1) * 3 + aa] = hc[c];
                }
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    reinterpret_cast<float4*>(o + 48)[k] = make_float4(fo[4 * k], fo[4 * k + 1], fo[4 * k + 2], fo[4 * k + 3]);
                // edge-space Hessian H_E[(e, a)][(e', a')], index 3 e + a, upper triangle
                const float k1 = 2.f * vol * (0.5f * mu * (1.f - inv_uI));   // 2 vol psi_I
                const float k2 = vol * (lam * jm1 - 0.75f * mu);              // vol psi_J
                const float k3 = 4.f * vol * (0.5f * mu * inv_uI * inv_uI);   // 4 vol psi_II
                const float k4 = vol * lam;
                float Fe[9], Ce[9], Fs[9], Cs[9];  // [a][e]
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int e = 0; e < 3; ++e) {
                        Fe[a * 3 + e] = F[a * 3] * rc[e * 3] + F[a * 3 + 1] * rc[e * 3 + 1] + F[a * 3 + 2] * rc[e * 3 + 2];
                        Ce[a * 3 + e] = cof[a * 3] * rc[e * 3] + cof[a * 3 + 1] * rc[e * 3 + 1] + cof[a * 3 + 2] * rc[e * 3 + 2];
                        Fs[a * 3 + e] = k3 * Fe[a * 3 + e];
                        Cs[a * 3 + e] = k4 * Ce[a * 3 + e];
                    }
                float Gm[9];  // k1 Dm^-1 Dm^-T
#pragma unroll
                for (int e = 0; e < 3; ++e)
#pragma unroll
                    for (int f = 0; f < 3; ++f)
                        Gm[e * 3 + f] = k1 * (rc[e * 3] * rc[f * 3] + rc[e * 3 + 1] * rc[f * 3 + 1] + rc[e * 3 + 2] * rc[f * 3 + 2]);
                // Sx[t][pair] = k2 F[t][:] . (row e x row e') of Dm^-1, pairs (0,1), (0,2), (1,2)
                float Sx[9];
#pragma unroll
                for (int pq = 0; pq < 3; ++pq) {
                    const int e = pq == 2 ? 1 : 0, f = pq == 0 ? 1 : 2;
                    const float x0 = rc[e * 3 + 1] * rc[f * 3 + 2] - rc[e * 3 + 2] * rc[f * 3 + 1];
                    const float x1 = rc[e * 3 + 2] * rc[f * 3 + 0] - rc[e * 3 + 0] * rc[f * 3 + 2];
                    const float x2 = rc[e * 3 + 0] * rc[f * 3 + 1] - rc[e * 3 + 1] * rc[f * 3 + 0];
#pragma unroll
                    for (int t = 0; t < 3; ++t) Sx[t * 3 + pq] = k2 * (F[t * 3] * x0 + F[t * 3 + 1] * x1 + F[t * 3 + 2] * x2);
                }
                float H[48];
#pragma unroll
                for (int i = 0; i < 9; ++i) {
                    const int e = i / 3, a = i % 3;
#pragma unroll
                    for (int j = i; j < 9; ++j) {
                        const int f = j / 3, b = j % 3;
                        float v = Fs[a * 3 + e] * Fe[b * 3 + f] + Cs[a * 3 + e] * Ce[b * 3 + f];
                        if (a == b) {
                            v += Gm[e * 3 + f];
                        } else if (e != f) {
                            const int t = 3 - a - b;
                            const float sx = Sx[t * 3 + (e + f - 1)];
                            v = ((b - a + 3) % 3 == 1) ? v + sx : v - sx;
                        }
                        H[i * 9 - i * (i - 1) / 2 + (j - i)] = v;
                    }
                }
                H[45] = H[46] = H[47] = 0.f;
#pragma unroll
                for (int k = 0; k < 12; ++k)
                    reinterpret_cast<float4*>(o)[k] = make_float4(H[4 * k], H[4 * k + 1], H[4 * k + 2], H[4 * k + 3]);
            }
        }
        __syncthreads();
        const int nbt = min(R, ne - eb);
        for (int t2 = 0; t2 < nbt; t2 += 2) {
            const int el = eb + t2;
            if (el + 1 < ne) load_raw(rawB, el + 1);
            process(rawA, el, t2);
            if (t2 + 1 < nbt) {
                if (el + 2 < ne) load_raw(rawA, el + 2);
                process(rawB, el + 1, t2 + 1);
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int pp = 0; pp < PPW; ++pp) {
        const int pc = warp * PPW + pp;
        if (p0 + pc >= P) continue;
        float* Co = Cpart + ((size_t)blk * P + p0 + pc) * NPAIR;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    // tile position 8 q + g holds direction g NR + q (the lanes load NR consecutive directions)
                    const int ap = mt * 16 + g + (q >= 2 ? 8 : 0), bp = nt * 8 + 2 * t4 + (q & 1);
                    const int a = (ap & 7) * NR + (ap >> 3), bb = (bp & 7) * NR + (bp >> 3);
                    if (ap < R && a <= bb) Co[a * R - a * (a - 1) / 2 + (bb - a)] = cacc[pp][mt][nt][q];
                }
    }
    for (int i = tid; i < nv * 3 * GP; i += 128) {
        const int pp = i % GP;
        if (p0 + pp < P) gpart[((size_t)(v0 * 3) + i / GP) * P + p0 + pp] = accg[i];
    }
}

// C[p][pair] = sum over blocks (fixed order, fp64): CTA per 32 (p, pair) entries,
// 8 warps stride the blocks, fixed combine order.
__global__ void __launch_bounds__(256) hess_reduce_kernel(int nblk, int P, int npair, const float* Cpart, double* C) {
    __shared__ double red[8][33];
    const int total = P * npair;
    const int idx = blockIdx.x * 32 + (threadIdx.x & 31);
    const int w = threadIdx.x >> 5;
    double s = 0.0;
    if (idx < total) {
        // 8 independent loads in flight per thread, summed in the same (block) order
        int b = w;
        for (; b + 56 < nblk; b += 64) {
            float v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __ldg(Cpart + (size_t)(b + 8 * k) * total + idx);
#pragma unroll
            for (int k = 0; k < 8; ++k) s += v[k];
        }
        for (; b < nblk; b += 8) s += Cpart[(size_t)b * total + idx];
    }
    red[w][threadIdx.x & 31] = s;
    __syncthreads();
    if (w == 0 && idx < total) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k][threadIdx.x];
        C[idx] = t;
    }
}

// H[p][a][b] = C_ab + sum_j ybar[j][p] S_L[j][p, ab]  (symmetric fill).
__global__ void hess_final_kernel(int h, int P, int r, int cols, const double* C, const float* Ybar, const float* X,
                                  double* H) {
    const int npair = r * (r + 1) / 2;
    const int total = P * npair;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int p = idx / npair, pr = idx % npair;
        double s = C[idx];
        const float* xp = X + (size_t)p * cols + 1 + r + pr;
        int j = 0;
        for (; j + 8 <= h; j += 8) {  // 8 independent load pairs in flight, summed in j order
            float yv[8], xv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                yv[k] = __ldg(Ybar + (size_t)(j + k) * P + p);
                xv[k] = __ldg(xp + (size_t)(j + k) * P * cols);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) s += (double)yv[k] * (double)xv[k];
        }
        for (; j < h; ++j) s += (double)Ybar[(size_t)j * P + p] * (double)xp[(size_t)j * P * cols];
        int a = 0, rem = pr;
        while (rem >= r - a) {
            rem -= r - a;
            ++a;
        }
        const int b = a + rem;
        H[((size_t)p * r + a) * r + b] = s;
        H[((size_t)p * r + b) * r + a] = s;
    }
}

}  // namespace

// ---------------------------------------------------------------- engine
struct BatchedEngine : BatchedBase {
    int BC = kBC;
    // tet blocks
    int nblk = 0, nslots = 0;
    int *d_blk_tet0 = nullptr, *d_blk_vptr = nullptr, *d_vslot_ptr = nullptr, *d_vslot = nullptr;
    short* d_tet_loc = nullptr;
    int max_nv = 0;
    // all touched vertices (free and pinned) per block, for shared-memory staging
    int *d_blk_aptr = nullptr, *d_blk_avert = nullptr;
    short* d_tet_aloc = nullptr;
    int max_nva = 0;
    size_t esmem2 = 0, esmem_f2 = 0;
    bool use_f2 = true;
    // buffers
    float *d_W = nullptr;  // W_out fp32 [n][h] (unpadded)
    float *d_Z = nullptr, *d_Y[kMaxLayers + 1] = {}, *d_A[kMaxLayers] = {};
    // group buffers: the hidden layers run once over a group of up to kGroup columns
    static constexpr int kGroup = 4096;
    float *d_Zg = nullptr, *d_Yg[kMaxLayers + 1] = {}, *d_Ag[kMaxLayers] = {}, *d_Ybg = nullptr, *d_Gbg[2] = {};
    double* d_Eg = nullptr;
    float *d_C = nullptr, *d_U = nullptr, *d_rin = nullptr, *d_T = nullptr, *d_part = nullptr, *d_P = nullptr;
    float *d_Ybar = nullptr, *d_Gb[2] = {};
    double *d_epart = nullptr, *d_eblk = nullptr, *d_E = nullptr;
    int nk = 1, kchunk = 1, nrow_tiles = 1;
    std::vector<void*> allocs;
    TcGemm tc;  // tcgen05 GEMM engine (lsb_tc.cuh)
    // second order (config 5)
    static constexpr int PH = 64;  // points per chunk of the theta-gradient path (and the minimum allocation width)
    int PHmax = PH;                // allocation width of the Hessian buffers: up to 256 points per chunk when they fit
    int Pcur = 0;                  // chunk width the pinned rows of d_Uh / d_Jv are laid out for
    int* d_pin_v = nullptr;        // pinned vertex ids and pin displacements (upload_pin_rows)
    float* d_pin_d = nullptr;
    int pins_uploaded = -1, pins_hess = -1, pins_eval = 0;  // Context::pins_version last applied
    bool hess_ready = false;
    float *d_Whf = nullptr;  // hidden weights fp32 (concatenated, row-major)
    float *d_Xl[kMaxLayers + 1] = {}, *d_Ql[kMaxLayers] = {}, *d_Bt = nullptr, *d_Ct = nullptr, *d_Uh = nullptr, *d_Jv = nullptr;
    float *d_Cpart = nullptr, *d_gpart = nullptr, *d_Th = nullptr, *d_Yh = nullptr, *d_Ph = nullptr, *d_Zh = nullptr;
    double *d_Ch = nullptr, *d_H = nullptr;
    float* d_rinh = nullptr;  // inertia residual of the objective Hessian (n x PH)
    int hcols = 0;
    struct PackedLayer {
        float* A = nullptr;
        int tiles = 0, S = 0;
    };
    std::vector<PackedLayer> hA;  // hidden weights as tcgen05 A tiles (tangent GEMMs)

    ~BatchedEngine() override {
        tc.release();
        for (void* p : allocs) cudaFree(p);
    }
    template <typename X>
    X* alloc(size_t count) {
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, std::max<size_t>(count * sizeof(X), 16)), "batched malloc");
        allocs.push_back(p);
        return static_cast<X*>(p);
    }

    // Blocks of tb consecutive tets with their touched free vertices (slots), local slot of
    // every tet corner, and per free vertex its slots in ascending block order.
    struct FreeBlocks {
        int nblk = 0, nslots = 0, max_nv = 0, max_nva = 0;
        int *tet0 = nullptr, *vptr = nullptr, *vslot_ptr = nullptr, *vslot = nullptr;
        short* loc = nullptr;
        // with_all: every touched vertex (free and pinned) per block, for shared-memory staging
        int *aptr = nullptr, *avert = nullptr;
        short* aloc = nullptr;
    };
    FreeBlocks build_free_blocks(Context& c, int tb, bool with_all = false) {
        const HostMesh& m = c.mesh;
        FreeBlocks fb;
        fb.nblk = (m.E + tb - 1) / tb;
        std::vector<int> tet0(fb.nblk + 1), vptr(fb.nblk + 1, 0);
        std::vector<short> loc(4 * (size_t)m.E, -1);
        std::vector<int> slot_vertex;
        for (int bk = 0; bk < fb.nblk; ++bk) {
            tet0[bk] = bk * tb;
            const int e1 = std::min(m.E, (bk + 1) * tb);
            std::vector<int> verts;
            for (int e = bk * tb; e < e1; ++e)
                for (int k = 0; k < 4; ++k) {
                    const int f = m.free_index[m.T[4 * (size_t)e + k]];
                    if (f >= 0) verts.push_back(f);
                }
            std::sort(verts.begin(), verts.end());
            verts.erase(std::unique(verts.begin(), verts.end()), verts.end());
            for (int e = bk * tb; e < e1; ++e)
                for (int k = 0; k < 4; ++k) {
                    const int f = m.free_index[m.T[4 * (size_t)e + k]];
                    if (f >= 0)
                        loc[4 * (size_t)e + k] =
                            (short)(std::lower_bound(verts.begin(), verts.end(), f) - verts.begin());
                }
            vptr[bk + 1] = vptr[bk] + (int)verts.size();
            fb.max_nv = std::max(fb.max_nv, (int)verts.size());
            slot_vertex.insert(slot_vertex.end(), verts.begin(), verts.end());
        }
        tet0[fb.nblk] = m.E;
        fb.nslots = vptr[fb.nblk];
        std::vector<int> cnt(m.n_free + 1, 0);
        for (int s = 0; s < fb.nslots; ++s) cnt[slot_vertex[s] + 1]++;
        std::vector<int> sptr(m.n_free + 1, 0);
        for (int f = 0; f < m.n_free; ++f) sptr[f + 1] = sptr[f] + cnt[f + 1];
        std::vector<int> slots(fb.nslots), fill(sptr.begin(), sptr.end() - 1);
        for (int s = 0; s < fb.nslots; ++s) slots[fill[slot_vertex[s]]++] = s;
        fb.tet0 = alloc<int>(fb.nblk + 1);
        fb.vptr = alloc<int>(fb.nblk + 1);
        fb.loc = alloc<short>(4 * (size_t)m.E);
        fb.vslot_ptr = alloc<int>(m.n_free + 1);
        fb.vslot = alloc<int>(fb.nslots);
        c.copy(fb.tet0, tet0.data(), 4 * tet0.size(), cudaMemcpyHostToDevice, "blk");
        c.copy(fb.vptr, vptr.data(), 4 * vptr.size(), cudaMemcpyHostToDevice, "blk");
        c.copy(fb.loc, loc.data(), 2 * loc.size(), cudaMemcpyHostToDevice, "blk");
        c.copy(fb.vslot_ptr, sptr.data(), 4 * sptr.size(), cudaMemcpyHostToDevice, "blk");
        c.copy(fb.vslot, slots.data(), 4 * slots.size(), cudaMemcpyHostToDevice, "blk");
        if (with_all) {
            std::vector<int> aptr(fb.nblk + 1, 0), avert;
            std::vector<short> aloc(4 * (size_t)m.E, -1);
            for (int bk = 0; bk < fb.nblk; ++bk) {
                const int e1 = std::min(m.E, (bk + 1) * tb);
                std::vector<int> verts;
                for (int e = bk * tb; e < e1; ++e)
                    for (int k = 0; k < 4; ++k) verts.push_back(m.T[4 * (size_t)e + k]);
                std::sort(verts.begin(), verts.end());
                verts.erase(std::unique(verts.begin(), verts.end()), verts.end());
                for (int e = bk * tb; e < e1; ++e)
                    for (int k = 0; k < 4; ++k)
                        aloc[4 * (size_t)e + k] = (short)(std::lower_bound(verts.begin(), verts.end(),
                                                                           m.T[4 * (size_t)e + k]) - verts.begin());
                aptr[bk + 1] = aptr[bk] + (int)verts.size();
                fb.max_nva = std::max(fb.max_nva, (int)verts.size());
                avert.insert(avert.end(), verts.begin(), verts.end());
            }
            fb.aptr = alloc<int>(fb.nblk + 1);
            fb.avert = alloc<int>(avert.size());
            fb.aloc = alloc<short>(aloc.size());
            c.copy(fb.aptr, aptr.data(), 4 * aptr.size(), cudaMemcpyHostToDevice, "blk");
            c.copy(fb.avert, avert.data(), 4 * avert.size(), cudaMemcpyHostToDevice, "blk");
            c.copy(fb.aloc, aloc.data(), 2 * aloc.size(), cudaMemcpyHostToDevice, "blk");
        }
        return fb;
    }
    FreeBlocks eb;  // the batched evaluation's (smaller) element blocks

    void init(Context& c) {
        const HostMesh& m = c.mesh;
        // --- tet blocks of kTB consecutive tets; touched free vertices, local indices
        nblk = (m.E + kTB - 1) / kTB;
        std::vector<int> tet0(nblk + 1), vptr(nblk + 1, 0);
        std::vector<short> loc(4 * (size_t)m.E, -1);
        std::vector<int> slot_vertex;  // global slot -> free vertex slot f
        for (int b = 0; b < nblk; ++b) {
            tet0[b] = b * kTB;
            const int e1 = std::min(m.E, (b + 1) * kTB);
            std::vector<int> verts;
            for (int e = b * kTB; e < e1; ++e)
                for (int k = 0; k < 4; ++k) {
                    const int f = m.free_index[m.T[4 * (size_t)e + k]];
                    if (f >= 0) verts.push_back(f);
                }
            std::sort(verts.begin(), verts.end());
            verts.erase(std::unique(verts.begin(), verts.end()), verts.end());
            for (int e = b * kTB; e < e1; ++e)
                for (int k = 0; k < 4; ++k) {
                    const int f = m.free_index[m.T[4 * (size_t)e + k]];
                    if (f >= 0)
                        loc[4 * (size_t)e + k] =
                            (short)(std::lower_bound(verts.begin(), verts.end(), f) - verts.begin());
                }
            vptr[b + 1] = vptr[b] + (int)verts.size();
            max_nv = std::max(max_nv, (int)verts.size());
            slot_vertex.insert(slot_vertex.end(), verts.begin(), verts.end());
        }
        tet0[nblk] = m.E;
        nslots = vptr[nblk];
        {
            std::vector<int> aptr(nblk + 1, 0), avert;
            std::vector<short> aloc(4 * (size_t)m.E, -1);
            for (int bk = 0; bk < nblk; ++bk) {
                const int e1 = std::min(m.E, (bk + 1) * kTB);
                std::vector<int> verts;
                for (int e = bk * kTB; e < e1; ++e)
                    for (int k = 0; k < 4; ++k) verts.push_back(m.T[4 * (size_t)e + k]);
                std::sort(verts.begin(), verts.end());
                verts.erase(std::unique(verts.begin(), verts.end()), verts.end());
                for (int e = bk * kTB; e < e1; ++e)
                    for (int k = 0; k < 4; ++k)
                        aloc[4 * (size_t)e + k] = (short)(std::lower_bound(verts.begin(), verts.end(),
                                                                           m.T[4 * (size_t)e + k]) - verts.begin());
                aptr[bk + 1] = aptr[bk] + (int)verts.size();
                max_nva = std::max(max_nva, (int)verts.size());
                avert.insert(avert.end(), verts.begin(), verts.end());
            }
            d_blk_aptr = alloc<int>(nblk + 1);
            d_blk_avert = alloc<int>(avert.size());
            d_tet_aloc = alloc<short>(aloc.size());
            c.copy(d_blk_aptr, aptr.data(), 4 * aptr.size(), cudaMemcpyHostToDevice, "blk");
            c.copy(d_blk_avert, avert.data(), 4 * avert.size(), cudaMemcpyHostToDevice, "blk");
            c.copy(d_tet_aloc, aloc.data(), 2 * aloc.size(), cudaMemcpyHostToDevice, "blk");
        }
        // vertex -> slots (ascending block order)
        std::vector<int> cnt(m.n_free + 1, 0);
        for (int s = 0; s < nslots; ++s) cnt[slot_vertex[s] + 1]++;
        std::vector<int> sptr(m.n_free + 1, 0);
        for (int f = 0; f < m.n_free; ++f) sptr[f + 1] = sptr[f] + cnt[f + 1];
        std::vector<int> slots(nslots), fill(sptr.begin(), sptr.end() - 1);
        for (int s = 0; s < nslots; ++s) slots[fill[slot_vertex[s]]++] = s;
        d_blk_tet0 = alloc<int>(nblk + 1);
        d_blk_vptr = alloc<int>(nblk + 1);
        d_tet_loc = alloc<short>(4 * (size_t)m.E);
        d_vslot_ptr = alloc<int>(m.n_free + 1);
        d_vslot = alloc<int>(nslots);
        c.copy(d_blk_tet0, tet0.data(), 4 * tet0.size(), cudaMemcpyHostToDevice, "blk");
        c.copy(d_blk_vptr, vptr.data(), 4 * vptr.size(), cudaMemcpyHostToDevice, "blk");
        c.copy(d_tet_loc, loc.data(), 2 * loc.size(), cudaMemcpyHostToDevice, "blk");
        c.copy(d_vslot_ptr, sptr.data(), 4 * sptr.size(), cudaMemcpyHostToDevice, "blk");
        c.copy(d_vslot, slots.data(), 4 * slots.size(), cudaMemcpyHostToDevice, "blk");
        // --- decoder output layer (fp32, unpadded [n][h])
        const HostLayer& o = c.layers[c.nhid];
        std::vector<float> W(o.W.size());
        for (size_t i = 0; i < W.size(); ++i) W[i] = (float)o.W[i];
        d_W = alloc<float>(W.size());
        c.copy(d_W, W.data(), 4 * W.size(), cudaMemcpyHostToDevice, "batched W");
        // --- chunk buffers
        const int n = c.n, h = c.h, V = m.V;
        int hmax = c.r;
        for (int l = 0; l < c.nhid; ++l) hmax = std::max(hmax, c.hrows[l]);
        d_Zg = alloc<float>((size_t)c.r * kGroup);
        for (int l = 0; l < c.nhid; ++l) {
            d_Yg[l + 1] = alloc<float>((size_t)c.hrows[l] * kGroup);
            d_Ag[l] = alloc<float>((size_t)c.hrows[l] * kGroup);
        }
        d_Yg[0] = d_Zg;
        d_Ybg = alloc<float>((size_t)h * kGroup);
        d_Gbg[0] = alloc<float>((size_t)hmax * kGroup);
        d_Gbg[1] = alloc<float>((size_t)hmax * kGroup);
        d_Eg = alloc<double>(kGroup);
        d_Z = alloc<float>((size_t)c.r * BC);
        for (int l = 0; l < c.nhid; ++l) {
            d_Y[l + 1] = alloc<float>((size_t)c.hrows[l] * BC);
            d_A[l] = alloc<float>((size_t)c.hrows[l] * BC);
        }
        d_Y[0] = d_Z;
        d_C = alloc<float>((size_t)n * BC);
        d_U = alloc<float>((size_t)V * 3 * BC);
        d_rin = alloc<float>((size_t)n * BC);
        d_T = alloc<float>((size_t)n * BC);
        eb = build_free_blocks(c, kTBE);
        d_part = alloc<float>((size_t)std::max(nslots, eb.nslots) * 3 * BC);
        kchunk = 256;
        nk = (n + kchunk - 1) / kchunk;
        d_P = alloc<float>((size_t)nk * h * BC);
        d_Ybar = alloc<float>((size_t)h * BC);
        d_Gb[0] = alloc<float>((size_t)hmax * BC);
        d_Gb[1] = alloc<float>((size_t)hmax * BC);
        nrow_tiles = (n + 63) / 64;
        d_epart = alloc<double>((size_t)nrow_tiles * BC);
        d_eblk = alloc<double>((size_t)std::max(nblk, eb.nblk) * BC);
        d_E = alloc<double>(BC);
        // pinned rows of U: pin displacement, constant across columns
        std::vector<float> U0((size_t)V * 3 * BC, 0.f);
        for (int v : m.pinned)
            for (int k = 0; k < 3; ++k) {
                const float d = (float)(c.pin_positions[3 * (size_t)v + k] - m.X[3 * (size_t)v + k]);
                for (int b = 0; b < BC; ++b) U0[((size_t)v * 3 + k) * BC + b] = d;
            }
        c.copy(d_U, U0.data(), 4 * U0.size(), cudaMemcpyHostToDevice, "U pins");
        pins_eval = c.pins_version;
        esmem2 = (size_t)(eb.max_nv + 1) * 3 * kEcols * sizeof(float) + kTB * 12 * sizeof(float) +
                 kTB * 4 * sizeof(int) + kTB * 4 * sizeof(int);
        esmem_f2 = (size_t)(eb.max_nv + 1) * 3 * kP2Threads * sizeof(float2) + (size_t)kTBE * kP2Consts * sizeof(float2) +
                   kTBE * 4 * sizeof(int) + kTBE * 4 * sizeof(int);
        cuda_check(cudaFuncSetAttribute(elem_batched_p2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)esmem_f2), "elem p2 smem");
        // packed fp32x2 element kernel (fp32 contexts; LSB_ELEM_F2=0 selects the scalar kernel)
        use_f2 = c.dev.elem_f2 && BC % (2 * kP2Threads) == 0;
        cuda_check(cudaFuncSetAttribute(elem_batched2_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)esmem2), "elem2 smem");
        cuda_check(cudaFuncSetAttribute(elem_batched2_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)esmem2), "elem2 smem");
        if (c.dev.tc) tc.init(c.stream, d_W, n, h, BC, c.num_sms);
    }

    // One group of N <= kGroup columns; Z (N x r, host) -> E (N), G (N x r or null).
    // Hidden layers (forward and backward) run once over the whole group; the output
    // layer, element pass and VJP run per chunk of BC columns.
    void run_group(Context& c, int N, const double* Z, double* E, double* G) {
        cudaStream_t s = c.stream;
        const int n = c.n, h = c.h, r = c.r;
        const int Np = (N + BC - 1) / BC * BC;  // padded to whole chunks (zero columns)
        if (pins_eval != c.pins_version) {  // lsb_set_pin_positions since the last call: pinned rows of U
            upload_pin_rows(c);
            const int np = (int)c.mesh.pinned.size();
            if (np) pinned_rows_kernel<<<c.num_sms * 4, 256, 0, s>>>(np, BC, 0, d_pin_v, d_pin_d, d_U, nullptr);
            cuda_check(cudaGetLastError(), "pinned rows");
            pins_eval = c.pins_version;
        }
        DevState* hs = c.h_state;
        cuda_check(cudaMemcpyAsync(hs, c.d_state, sizeof(DevState), cudaMemcpyDeviceToHost, s), "state");
        cuda_check(cudaStreamSynchronize(s), "sync");
        const int has_inertia = hs->has_inertia;
        const double inv_dt2 = hs->inv_dt2;
        // Z^T -> [r][Np]
        std::vector<float> zt((size_t)r * Np, 0.f);
        for (int b = 0; b < N; ++b)
            for (int k = 0; k < r; ++k) zt[(size_t)k * Np + b] = (float)Z[(size_t)b * r + k];
        cuda_check(cudaMemcpyAsync(d_Zg, zt.data(), 4 * zt.size(), cudaMemcpyHostToDevice, s), "Z");
        // hidden forward over the group
        for (int l = 0; l < c.nhid; ++l) {
            const int M = c.hrows[l], K = c.hcols[l];
            dim3 grid((Np + 31) / 32, (M + 31) / 32);
            small_gemm_kernel<<<grid, 256, 0, s>>>(M, Np, K, c.d_Wh + c.hoff[l], 0, d_Yg[l], c.d_bh + c.boff[l],
                                                   d_Yg[l + 1], d_Ag[l], c.hact[l], nullptr, 0);
        }
        c.batched_launches += c.nhid;
        for (int c0 = 0; c0 < Np; c0 += BC) {
            const float* Yc = d_Yg[c.nhid] + c0;  // h x BC slice, row stride Np
            // output layer u = s (W_out Y_L + b) + shift - X: tcgen05 GEMM with the epilogue fused
            // (U, inertia residual, energy partials per 128-row tile); else SGEMM + epilogue kernel
            int e_tiles = nrow_tiles;
            if (tc.gemm_out_fused(s, Yc, Np, c.d_eprow, d_U, d_rin, d_epart, has_inertia, inv_dt2)) {
                e_tiles = tc.tiles1;
            } else {
                dim3 g1((BC + 127) / 128, (n + 127) / 128);
                sgemm_nn_kernel<<<g1, 256, 0, s>>>(n, BC, h, d_W, h, Yc, Np, d_C, BC);
                dim3 g((n + 63) / 64, (BC + 63) / 64);
                out_epilogue_kernel<<<g, 256, 0, s>>>(n, BC, d_C, c.d_eprow, c.d_ut, has_inertia, inv_dt2, d_U,
                                                      d_rin, d_epart);
                c.batched_launches += 2;
            }
            if (use_f2 && c.precision != LSB_FP64) {
                // packed fp32x2: thread = two adjacent columns, 2 kEcols columns per CTA
                dim3 g(eb.nblk, (BC + 2 * kP2Threads - 1) / (2 * kP2Threads));
                elem_batched_p2_kernel<<<g, kP2Threads, esmem_f2, s>>>(
                    static_cast<const float*>(c.d_rec), eb.tet0, eb.vptr, eb.loc,
                    reinterpret_cast<const int4*>(c.d_tets), d_U, BC, d_part, d_eblk);
            } else {
                dim3 g(eb.nblk, (BC + kEcols - 1) / kEcols);
                if (c.precision == LSB_FP64)
                    elem_batched2_kernel<double><<<g, kEcols, esmem2, s>>>(
                        static_cast<const double*>(c.d_rec), eb.tet0, eb.vptr, eb.loc,
                        reinterpret_cast<const int4*>(c.d_tets), d_U, BC, d_part, d_eblk);
                else
                    elem_batched2_kernel<float><<<g, kEcols, esmem2, s>>>(
                        static_cast<const float*>(c.d_rec), eb.tet0, eb.vptr, eb.loc,
                        reinterpret_cast<const int4*>(c.d_tets), d_U, BC, d_part, d_eblk);
            }
            energy_reduce_kernel<<<BC, 256, 0, s>>>(BC, e_tiles, d_epart, eb.nblk, d_eblk, has_inertia, d_Eg + c0);
            c.batched_launches += 2;
            if (G) {
                // Ybar[:, c0:c0+BC] = W_out^T T: tcgen05 with T packed by the combine, else SGEMM
                if (tc.enabled) {
                    combine_pack_kernel<<<c.num_sms * 8, 256, 0, s>>>(n, BC, eb.vslot_ptr, eb.vslot, d_part, d_rin,
                                                                      has_inertia, c.d_eprow, tc.B2);
                    tc.gemm_vjp_prepacked(s, d_Ybg + c0, Np);
                    c.batched_launches += 1;
                } else {
                    combine_kernel<<<c.num_sms * 8, 256, 0, s>>>(n, BC, eb.vslot_ptr, eb.vslot, d_part, d_rin,
                                                                 has_inertia, c.d_eprow, d_T);
                    c.batched_launches += 1;
                    dim3 g2((BC + 127) / 128, (h + 127) / 128, nk);
                    sgemm_tn_splitk_kernel<<<g2, 256, 0, s>>>(h, BC, n, kchunk, d_W, h, d_T, BC, d_P);
                    splitk_reduce_kernel<<<c.num_sms, 256, 0, s>>>(h * BC, nk, d_P, d_Ybg + c0, BC, Np);
                    c.batched_launches += 2;
                }
            }
            c.batched_launches += tc.launches;
            tc.launches = 0;
        }
        std::vector<double> e(Np);
        if (G) {
            // hidden backward over the group: g_{l-1} = W_l^T (g_l * phi'(A_l))
            const float* gin = d_Ybg;
            int buf = 0;
            for (int l = c.nhid - 1; l >= 0; --l) {
                const int R = c.hrows[l], C = c.hcols[l];
                dim3 grid((Np + 31) / 32, (C + 31) / 32);
                gate_mul(s, R * Np, gin, d_Ag[l], c.hact[l], d_Gbg[buf]);
                small_gemm_kernel<<<grid, 256, 0, s>>>(C, Np, R, c.d_Wh + c.hoff[l], 1, d_Gbg[buf], nullptr,
                                                       d_Gbg[buf ^ 1], nullptr, -1, nullptr, 0);
                gin = d_Gbg[buf ^ 1];
                buf ^= 1;
                c.batched_launches += 2;
            }
            std::vector<float> gz((size_t)r * Np);
            cuda_check(cudaMemcpyAsync(gz.data(), gin, 4 * gz.size(), cudaMemcpyDeviceToHost, s), "G");
            cuda_check(cudaMemcpyAsync(e.data(), d_Eg, 8 * Np, cudaMemcpyDeviceToHost, s), "E");
            cuda_check(cudaStreamSynchronize(s), "sync");
            for (int b = 0; b < N; ++b)
                for (int k = 0; k < r; ++k) G[(size_t)b * r + k] = gz[(size_t)k * Np + b];
        } else {
            cuda_check(cudaMemcpyAsync(e.data(), d_Eg, 8 * Np, cudaMemcpyDeviceToHost, s), "E");
            cuda_check(cudaStreamSynchronize(s), "sync");
        }
        for (int b = 0; b < N; ++b) E[b] = e[b];
    }

    static void gate_mul(cudaStream_t s, int total, const float* g, const float* A, int act, float* out);

    void init_hessian(Context& c) {
        const int r = c.r, h = c.h, n = c.n;
        if (c.out_act != kIdentity) throw LsbError(LSB_EINVAL, "hessian: device path requires an identity output layer");
        if (r != 8 && r != 16 && r != 32)
            throw LsbError(LSB_EINVAL, "hessian: device path supports latent dims 8, 16, 32");
        const int npair = r * (r + 1) / 2;
        hcols = 1 + r + npair;
        int hmax = r;
        for (int l = 0; l < c.nhid; ++l) hmax = std::max(hmax, c.hrows[l]);
        size_t wtot = 0;
        for (int l = 0; l < c.nhid; ++l) wtot += (size_t)c.hrows[l] * c.hcols[l];
        std::vector<float> wf(wtot);
        size_t off = 0;
        for (int l = 0; l < c.nhid; ++l)
            for (double v : c.layers[l].W) wf[off++] = (float)v;
        d_Whf = alloc<float>(std::max<size_t>(1, wtot));
        if (wtot) c.copy(d_Whf, wf.data(), 4 * wtot, cudaMemcpyHostToDevice, "Whf");
        if (tc.enabled) {
            size_t wo = 0;
            hA.resize(c.nhid);
            for (int l = 0; l < c.nhid; ++l) {
                const int R = c.hrows[l], K = c.hcols[l];
                hA[l].A = alloc<float>(TcGemm::packed_a_floats(R, K));
                tc.pack_a(c.stream, d_Whf + wo, R, K, hA[l].A, hA[l].tiles, hA[l].S);
                wo += (size_t)R * K;
            }
            cuda_check(cudaGetLastError(), "pack hidden");
        }
        // chunk width: wide chunks amortise the small hidden-layer GEMMs and launches (config 5: 64 -> 256
        // points per chunk); bounded by ~4 GB of chunk buffers (a config-3-sized mesh stays at 64)
        {
            const double per_point = 4.0 * ((double)n * (3 + r) + (double)c.mesh.V * 3 * (1 + r) + (double)nblk * npair +
                                            (double)hmax * hcols * (2 * c.nhid + 1));
            PHmax = PH;
            while (PHmax < 256 && per_point * (2 * PHmax) <= 4.0e9) PHmax *= 2;
        }
        for (int l = 0; l <= c.nhid; ++l) d_Xl[l] = alloc<float>((size_t)hmax * PHmax * hcols);
        for (int l = 0; l < c.nhid; ++l) d_Ql[l] = alloc<float>((size_t)hmax * PHmax * hcols);
        d_Bt = alloc<float>((size_t)h * PHmax * (1 + r));
        d_Ct = alloc<float>((size_t)n * PHmax * (1 + r));
        d_Uh = alloc<float>((size_t)c.mesh.V * 3 * PHmax);
        d_Jv = alloc<float>((size_t)c.mesh.V * 3 * PHmax * r);
        d_Cpart = alloc<float>((size_t)nblk * PHmax * npair);
        d_rinh = alloc<float>((size_t)c.n * PHmax);
        d_gpart = alloc<float>((size_t)nslots * 3 * PHmax);
        d_Th = alloc<float>((size_t)n * PHmax);
        d_Yh = alloc<float>((size_t)h * PHmax);
        d_Ph = alloc<float>((size_t)nk * h * PHmax);
        d_Zh = alloc<float>((size_t)r * PHmax);
        d_Ch = alloc<double>((size_t)PHmax * npair);
        d_H = alloc<double>((size_t)PHmax * r * r);
        Pcur = 0;  // pinned rows of U (pin displacement) and J (zero) are laid out per chunk width: prepare_width
        const size_t gsmem = hess_smem(r);
        if (r == 8) cuda_check(cudaFuncSetAttribute(elem_hess2_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem), "smem");
        if (r == 16) cuda_check(cudaFuncSetAttribute(elem_hess2_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem), "smem");
        if (r == 32) cuda_check(cudaFuncSetAttribute(elem_hess2_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem), "smem");
        if (r == 8) cuda_check(cudaFuncSetAttribute(elem_hess3_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem), "smem");
        if (r == 16) cuda_check(cudaFuncSetAttribute(elem_hess3_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem), "smem");
        if (r == 32) cuda_check(cudaFuncSetAttribute(elem_hess3_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem), "smem");
        hess_ready = true;
    }

    // ---------------------------------------------------------------- theta-gradient (lsb_theta.cuh)
    bool theta_ready = false;
    float *d_Hbf = nullptr, *d_ebf = nullptr, *d_Bt2 = nullptr, *d_Bfwd = nullptr, *d_Ct2 = nullptr;
    double* d_fac = nullptr;  // per-pair factors 2 / (P |dz|^2) of a chunk
    float *d_Wv = nullptr, *d_gbar = nullptr, *d_partJ = nullptr, *d_partq = nullptr, *d_Abar = nullptr;
    float *d_XbL = nullptr, *d_Xbar[2] = {}, *d_Abl = nullptr, *d_spart = nullptr;
    double *d_gW = nullptr, *d_gb = nullptr;
    size_t gw_total = 0, gb_total = 0, spart_floats = 0, tsmem = 0;
    std::vector<size_t> gw_off, gb_off, hw_off;  // per layer (hidden..., output); fp32 hidden weight offsets

    FreeBlocks tbk;  // the theta pass's element blocks (LSB_THETA_TB tets, default 24)
    static constexpr int kSplitOut = 64;  // split-K of W_out^T Abar (K = n)
    static constexpr int kSplitHid = 32;  // split-K of Abar_l X_l^T (K = PH * cols)

    void init_theta(Context& c) {
        if (!hess_ready) init_hessian(c);
        const int r = c.r, h = c.h, n = c.n, P = PH, npair = r * (r + 1) / 2, V = c.mesh.V;
        int hmax = r;
        for (int l = 0; l < c.nhid; ++l) hmax = std::max(hmax, c.hrows[l]);
        d_Hbf = alloc<float>((size_t)P * r * r);
        d_ebf = alloc<float>((size_t)P * npair);
        d_fac = alloc<double>((size_t)P / 2 + 1);
        d_Bt2 = alloc<float>((size_t)h * P * (r + 1));
        d_Bfwd = alloc<float>((size_t)P * (r + 2) * h);
        d_Ct2 = alloc<float>((size_t)n * P * (r + 1));
        d_Wv = alloc<float>((size_t)V * 3 * P * r);
        d_gbar = alloc<float>((size_t)V * 3 * P);
        cuda_check(cudaMemsetAsync(d_Wv, 0, 4 * (size_t)V * 3 * P * r, c.stream), "Wv");
        cuda_check(cudaMemsetAsync(d_gbar, 0, 4 * (size_t)V * 3 * P, c.stream), "Gb");
        tbk = build_free_blocks(c, c.dev.theta_tb, true);
        d_partJ = alloc<float>((size_t)tbk.nslots * 3 * P * r);
        d_partq = alloc<float>((size_t)tbk.nslots * 3 * P);
        d_Abar = alloc<float>((size_t)n * P * (r + 2));
        d_XbL = alloc<float>((size_t)h * P * (r + 2));
        d_Xbar[0] = alloc<float>((size_t)hmax * P * hcols);
        d_Xbar[1] = alloc<float>((size_t)hmax * P * hcols);
        d_Abl = alloc<float>((size_t)hmax * P * hcols);
        gw_off.assign(c.nhid + 1, 0);
        gb_off.assign(c.nhid + 1, 0);
        hw_off.assign(c.nhid, 0);
        size_t hw = 0;
        spart_floats = std::max((size_t)n * h, (size_t)h * P * (r + 2) * kSplitOut);
        for (int l = 0; l <= c.nhid; ++l) {
            const size_t rows = l < c.nhid ? c.hrows[l] : n, cols = l < c.nhid ? c.hcols[l] : h;
            gw_off[l] = gw_total;
            gb_off[l] = gb_total;
            gw_total += rows * cols;
            gb_total += rows;
            if (l < c.nhid) {
                hw_off[l] = hw;
                hw += rows * cols;
                spart_floats = std::max(spart_floats, rows * cols * kSplitHid);
                spart_floats = std::max(spart_floats, cols * P * hcols);
            }
        }
        d_spart = alloc<float>(spart_floats);
        d_gW = alloc<double>(gw_total);
        d_gb = alloc<double>(gb_total);
        const int gp = 128 / r;
        tsmem = ((size_t)tbk.max_nva * 3 * gp + (size_t)tbk.max_nv * 3 * gp * r + (size_t)tbk.max_nv * 3 * gp) *
                    sizeof(float) + 64;
        if (tsmem > 227 * 1024 - 4096)
            throw LsbError(LSB_EINVAL, "lipschitz grad: element blocks too large for shared memory");
        if (r == 8) cuda_check(cudaFuncSetAttribute(theta::elem_theta_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem), "smem");
        if (r == 16) cuda_check(cudaFuncSetAttribute(theta::elem_theta_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem), "smem");
        if (r == 32) cuda_check(cudaFuncSetAttribute(theta::elem_theta_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem), "smem");
        cuda_check(cudaStreamSynchronize(c.stream), "theta init");
        theta_ready = true;
    }

    // C[M][N] (fp32 store and/or fp64 accumulate) = sum_k A[m*sam + k*sak] B[k*sbk + n*sbn]
    void gemm_strided(cudaStream_t s, int M, int N, int K, int nz, const float* A, long long sam, long long sak,
                      const float* B, long long sbk, long long sbn, float* out32, double* acc64, int sms) {
        int kchunk = (K + nz - 1) / nz;
        kchunk = (kchunk + 15) / 16 * 16;
        nz = (K + kchunk - 1) / kchunk;
        dim3 g((N + 127) / 128, (M + 127) / 128, nz);
        theta::sgemm_strided_kernel<<<g, 256, 0, s>>>(M, N, K, kchunk, A, sam, sak, B, sbk, sbn, d_spart);
        theta::splitk_out_kernel<<<sms * 4, 256, 0, s>>>((long long)M * N, nz, d_spart, out32, acc64);
    }

    template <int R>
    void launch_theta_elem(Context& c, int P) {
        constexpr int GP = 128 / R;
        dim3 g(tbk.nblk, (P + GP - 1) / GP);
        const float* recf = static_cast<const float*>(rec_f32(c));
        const int4* tt = reinterpret_cast<const int4*>(c.d_tets);
        theta::elem_theta_kernel<R><<<g, 128, tsmem, c.stream>>>(tt, recf, tbk.tet0, tbk.vptr, tbk.loc, tbk.aptr,
                                                                 tbk.avert, tbk.aloc, d_Uh, d_Jv, d_Wv, d_gbar, P,
                                                                 d_partJ, d_partq);
    }
    template <int R>
    void launch_theta_small(Context& c, int which, int rows, int l, int cur) {
        const int P = PH, cols = hcols;
        cudaStream_t s = c.stream;
        if (which == 0)
            theta::theta_prep_kernel<R><<<c.num_sms * 4, 256, 0, s>>>(c.h, P, cols, d_Xl[c.nhid], d_Hbf, d_ebf, d_Bt2,
                                                                      d_Bfwd);
        else if (which == 1)
            theta::theta_top_kernel<R><<<c.num_sms * 8, 256, 0, s>>>(c.h, P, cols, d_XbL, d_ebf, d_Xbar[0]);
        else
            theta::tangent_act_bwd_kernel<R><<<(rows * P + 127) / 128, 128, 0, s>>>(
                rows, P, cols, d_Ql[l], c.d_bh + c.boff[l], c.hact[l], d_Xbar[cur], d_Abl);
    }
    void theta_small(Context& c, int which, int rows = 0, int l = 0, int cur = 0) {
        if (c.r == 8) launch_theta_small<8>(c, which, rows, l, cur);
        else if (c.r == 16) launch_theta_small<16>(c, which, rows, l, cur);
        else launch_theta_small<32>(c, which, rows, l, cur);
    }

    // One chunk of N <= PH points (pairs interleaved z1, z2): H via run_hessian_chunk, the
    // loss terms and dL/dH on the host (fp64), then the device reverse sweep accumulating
    // dL/dtheta into d_gW / d_gb.  inv_P = 1 / (number of pairs in the whole loss).
    // One chunk of N (even) points = N / 2 pairs: Hessians into the device buffer, dL/dH on the device
    // (lipschitz_dldh_kernel) with the pair factors f = 2 inv_P / |dz|^2 from the host, |H1 - H2|^2
    // into d2_out (device, N / 2); no host round trip inside the chunk.
    void run_theta_chunk(Context& c, int N, const double* Z, double inv_P, double* d2_out) {
        if (!theta_ready) init_theta(c);
        const int r = c.r, h = c.h, n = c.n, P = PH, cols = hcols;
        cudaStream_t s = c.stream;
        double* d_Hc = hess_all(c, (size_t)P * r * r);
        run_hessian_chunk(c, N, Z, nullptr, false, d_Hc);
        std::vector<double> fac(N / 2);
        for (int q = 0; q < N / 2; ++q) {
            const double* z1 = Z + (size_t)(2 * q) * r;
            const double* z2 = z1 + r;
            double dz2 = 0.0;
            for (int k = 0; k < r; ++k) dz2 += (z1[k] - z2[k]) * (z1[k] - z2[k]);
            fac[q] = 2.0 * inv_P / dz2;
        }
        cuda_check(cudaMemcpyAsync(d_fac, fac.data(), 8 * fac.size(), cudaMemcpyHostToDevice, s), "pair factors");
        cuda_check(cudaMemsetAsync(d_Hbf, 0, 4 * (size_t)P * r * r, s), "Hbar");
        cuda_check(cudaMemsetAsync(d_ebf, 0, 4 * (size_t)P * (r * (r + 1) / 2), s), "ebar");
        lipschitz_dldh_kernel<<<N / 2, 256, 0, s>>>(N / 2, r, d_Hc, d_fac, d_Hbf, d_ebf, d2_out);
        // h-level operands, output GEMM -> W = J Hbar and gbar in the vertex layout
        theta_small(c, 0);
        if (!tc.enabled ||
            !tc.gemm_general(s, tc.A1, tc.tiles1, tc.S1, n, d_Bt2, P * (r + 1), h, P * (r + 1), d_Ct2, P * (r + 1))) {
            dim3 g((P * (r + 1) + 127) / 128, (n + 127) / 128);
            sgemm_nn_kernel<<<g, 256, 0, s>>>(n, P * (r + 1), h, d_W, h, d_Bt2, P * (r + 1), d_Ct2, P * (r + 1));
        }
        theta::theta_out_kernel<<<c.num_sms * 4, 256, 0, s>>>(n, P, r, d_Ct2, c.d_eprow, d_Wv, d_gbar);
        // element pass: Jbar = 2 K W, qbar = T[J, W] + K gbar (block partials), then per row
        if (r == 8) launch_theta_elem<8>(c, P);
        else if (r == 16) launch_theta_elem<16>(c, P);
        else launch_theta_elem<32>(c, P);
        theta::theta_combine_kernel<<<c.num_sms * 4, 256, 0, s>>>(n, P, r, tbk.vslot_ptr, tbk.vslot, d_partJ, d_partq,
                                                                   c.d_eprow, d_Th, d_Abar);
        const int w2 = P * (r + 2);
        // output layer: dW_out += Abar Bfwd, db_out += sum_p s qbar
        gemm_strided(s, n, h, w2, 1, d_Abar, w2, 1, d_Bfwd, h, 1, nullptr, d_gW + gw_off[c.nhid], c.num_sms);
        theta::rowsum_acc_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, P, w2, r + 2, d_Abar, d_gb + gb_off[c.nhid]);
        // adjoint of the top hidden block: W_out^T Abar, then S-bar = ebar rho
        gemm_strided(s, h, w2, n, kSplitOut, d_W, 1, h, d_Abar, w2, 1, d_XbL, nullptr, c.num_sms);
        theta_small(c, 1);
        int cur = 0;
        for (int l = c.nhid - 1; l >= 0; --l) {
            const int R = c.hrows[l], K = c.hcols[l];
            theta_small(c, 2, R, l, cur);
            gemm_strided(s, R, K, P * cols, kSplitHid, d_Abl, (long long)P * cols, 1, d_Xl[l], 1, (long long)P * cols,
                         nullptr, d_gW + gw_off[l], c.num_sms);
            theta::rowsum_acc_kernel<<<(R + 127) / 128, 128, 0, s>>>(R, P, (long long)P * cols, cols, d_Abl,
                                                                     d_gb + gb_off[l]);
            if (l > 0) {
                gemm_strided(s, K, P * cols, R, 1, d_Whf + hw_off[l], 1, K, d_Abl, (long long)P * cols, 1,
                             d_Xbar[cur ^ 1], nullptr, c.num_sms);
                cur ^= 1;
            }
        }
        cuda_check(cudaGetLastError(), "theta chunk");
        c.batched_launches += 12 + 5 * c.nhid;
    }

    // Lay the constant rows of the chunk buffers out for chunks of P points: pinned rows hold the pin
    // displacement in U and zero in J (tangent_out_kernel writes the free rows only).
    // device copies of the pinned vertex ids and pin displacements (current pins_version)
    void upload_pin_rows(Context& c) {
        if (pins_uploaded == c.pins_version) return;
        const size_t np = c.mesh.pinned.size();
        std::vector<int> pv(c.mesh.pinned.begin(), c.mesh.pinned.end());
        std::vector<float> pd(3 * np);
        for (size_t i = 0; i < np; ++i)
            for (int k = 0; k < 3; ++k)
                pd[3 * i + k] = (float)(c.pin_positions[3 * (size_t)pv[i] + k] - c.mesh.X[3 * (size_t)pv[i] + k]);
        if (!d_pin_v) {
            d_pin_v = alloc<int>(std::max<size_t>(1, np));
            d_pin_d = alloc<float>(std::max<size_t>(1, 3 * np));
        }
        if (np) {
            c.copy(d_pin_v, pv.data(), 4 * np, cudaMemcpyHostToDevice, "pinned ids");
            c.copy(d_pin_d, pd.data(), 12 * np, cudaMemcpyHostToDevice, "pin displacements");
        }
        pins_uploaded = c.pins_version;
    }
    void prepare_width(Context& c, int P) {
        if (P == Pcur && pins_hess == c.pins_version) return;
        if (P > PHmax || P % 16 != 0) throw LsbError(LSB_EINVAL, "hessian: bad chunk width");
        // only the pinned rows are constant (tangent_out_kernel rewrites every free row of a chunk)
        upload_pin_rows(c);
        const int np = (int)c.mesh.pinned.size();
        if (np) pinned_rows_kernel<<<c.num_sms * 4, 256, 0, c.stream>>>(np, P, c.r, d_pin_v, d_pin_d, d_Uh, d_Jv);
        cuda_check(cudaGetLastError(), "pinned rows");
        Pcur = P;
        pins_hess = c.pins_version;
    }
    // chunk width for a call over `total` points
    int pick_width(Context& c, int total) {
        if (!hess_ready) init_hessian(c);
        return std::min(PHmax, std::max(16, (total + 15) / 16 * 16));
    }

    size_t hess_smem(int r) const {
        const int gp = 128 / r;
        return ((size_t)max_nva * 3 * gp + (size_t)(max_nv + 1) * 3 * gp) * sizeof(float) + 64;  // Us + accg (elem_hess2)
    }

    // Hessians of the elastic potential for N <= PH points Z (N x r) -> H (N x r x r).
    // Hout_dev (device, N x r x r) instead of Hout: no host copy and no stream synchronisation, so
    // consecutive chunks queue back to back.
    void run_hessian_chunk(Context& c, int N, const double* Z, double* Hout, bool with_inertia = false,
                           double* Hout_dev = nullptr, int Pw = PH) {
        if (!hess_ready) init_hessian(c);
        prepare_width(c, Pw);
        cudaStream_t s = c.stream;
        int inertia = 0;
        double inv_dt2 = 0.0;
        if (with_inertia) {
            DevState* hs = c.h_state;
            cuda_check(cudaMemcpyAsync(hs, c.d_state, sizeof(DevState), cudaMemcpyDeviceToHost, s), "state");
            cuda_check(cudaStreamSynchronize(s), "sync");
            inertia = hs->has_inertia;
            inv_dt2 = hs->inv_dt2;
        }
        const int r = c.r, h = c.h, n = c.n, P = Pw, cols = hcols, npair = r * (r + 1) / 2;
        std::vector<float> zt((size_t)r * P, 0.f);
        for (int p = 0; p < N; ++p)
            for (int k = 0; k < r; ++k) zt[(size_t)k * P + p] = (float)Z[(size_t)p * r + k];
        cuda_check(cudaMemcpyAsync(d_Zh, zt.data(), 4 * zt.size(), cudaMemcpyHostToDevice, s), "Zh");
        tangent_init_kernel<<<c.num_sms, 256, 0, s>>>(r, P, cols, d_Zh, d_Xl[0]);
        size_t woff = 0;
        for (int l = 0; l < c.nhid; ++l) {
            const int R = c.hrows[l], K = c.hcols[l];
            if (!tc.enabled ||
                !tc.gemm_general(s, hA[l].A, hA[l].tiles, hA[l].S, R, d_Xl[l], P * cols, K, P * cols, d_Ql[l], P * cols)) {
                dim3 g((P * cols + 127) / 128, (R + 127) / 128);
                sgemm_nn_kernel<<<g, 256, 0, s>>>(R, P * cols, K, d_Whf + woff, K, d_Xl[l], P * cols, d_Ql[l], P * cols);
            }
            tangent_act_kernel<<<c.num_sms * 8, 256, 0, s>>>(R, P, r, cols, d_Ql[l], c.d_bh + c.boff[l], c.hact[l],
                                                             d_Xl[l + 1]);
            woff += (size_t)R * K;
        }
        const float* XL = d_Xl[c.nhid];
        tangent_pack_kernel<<<c.num_sms, 256, 0, s>>>(h, P, r, cols, XL, d_Bt);
        // output layer with the tangent-output epilogue fused into the tcgen05 GEMM (U, Jv, inertia residual
        // straight from TMEM: no n x P (1 + r) product written and re-read); else SGEMM + tangent_out_kernel
        if (!c.dev.fuse_tangent_out ||
            !tc.gemm_tangent_out(s, d_Bt, h, P, r, c.d_eprow, d_Uh, d_Jv, d_rinh, inertia, inv_dt2)) {
            if (!tc.enabled ||
                !tc.gemm_general(s, tc.A1, tc.tiles1, tc.S1, n, d_Bt, P * (1 + r), h, P * (1 + r), d_Ct, P * (1 + r))) {
                dim3 g((P * (1 + r) + 127) / 128, (n + 127) / 128);
                sgemm_nn_kernel<<<g, 256, 0, s>>>(n, P * (1 + r), h, d_W, h, d_Bt, P * (1 + r), d_Ct, P * (1 + r));
            }
            tangent_out_kernel<<<c.num_sms * 4, 256, 0, s>>>(n, P, r, d_Ct, c.d_eprow, d_Uh, d_Jv, inertia, inv_dt2,
                                                             d_rinh);
        }
        {
            const int gp = 128 / r;
            dim3 g(nblk, (P + gp - 1) / gp);
            const size_t gsmem = hess_smem(r);
            const float* recf = static_cast<const float*>(rec_f32(c));
            const int4* tt = reinterpret_cast<const int4*>(c.d_tets);
            // edge-space form: two chained 3xTF32 MMA stages per (tet, point); LSB_HESS3=0 selects the D^T M' kernel
            if (c.dev.hess3) {
                if (r == 8)
                    elem_hess3_kernel<8><<<g, 128, gsmem, s>>>(tt, recf, d_blk_tet0, d_blk_vptr, d_tet_loc, d_blk_aptr,
                                                             d_blk_avert, d_tet_aloc, d_Uh, d_Jv, P, d_Cpart, d_gpart);
                else if (r == 16)
                    elem_hess3_kernel<16><<<g, 128, gsmem, s>>>(tt, recf, d_blk_tet0, d_blk_vptr, d_tet_loc,
                                                              d_blk_aptr, d_blk_avert, d_tet_aloc, d_Uh, d_Jv, P,
                                                              d_Cpart, d_gpart);
                else
                    elem_hess3_kernel<32><<<g, 128, gsmem, s>>>(tt, recf, d_blk_tet0, d_blk_vptr, d_tet_loc,
                                                              d_blk_aptr, d_blk_avert, d_tet_aloc, d_Uh, d_Jv, P,
                                                              d_Cpart, d_gpart);
            } else if (r == 8)
                elem_hess2_kernel<8><<<g, 128, gsmem, s>>>(tt, recf, d_blk_tet0, d_blk_vptr, d_tet_loc, d_blk_aptr,
                                                         d_blk_avert, d_tet_aloc, d_Uh, d_Jv, P, d_Cpart, d_gpart);
            else if (r == 16)
                elem_hess2_kernel<16><<<g, 128, gsmem, s>>>(tt, recf, d_blk_tet0, d_blk_vptr, d_tet_loc, d_blk_aptr,
                                                          d_blk_avert, d_tet_aloc, d_Uh, d_Jv, P, d_Cpart, d_gpart);
            else
                elem_hess2_kernel<32><<<g, 128, gsmem, s>>>(tt, recf, d_blk_tet0, d_blk_vptr, d_tet_loc, d_blk_aptr,
                                                          d_blk_avert, d_tet_aloc, d_Uh, d_Jv, P, d_Cpart, d_gpart);
        }
        hess_reduce_kernel<<<(P * npair + 31) / 32, 256, 0, s>>>(nblk, P, npair, d_Cpart, d_Ch);
        if (inertia) inertia_hess_kernel<<<P, 256, 0, s>>>(n, P, r, c.d_eprow, d_Jv, inv_dt2, d_Ch);
        // full-space residual (elastic gradient [+ inertia]), times s
        combine_kernel<<<c.num_sms * 4, 256, 0, s>>>(n, P, d_vslot_ptr, d_vslot, d_gpart, d_rinh, inertia, c.d_eprow,
                                                     d_Th);
        {
            dim3 g2((P + 127) / 128, (h + 127) / 128, nk);
            sgemm_tn_splitk_kernel<<<g2, 256, 0, s>>>(h, P, n, kchunk, d_W, h, d_Th, P, d_Ph);
            splitk_reduce_kernel<<<c.num_sms, 256, 0, s>>>(h * P, nk, d_Ph, d_Yh);
        }
        hess_final_kernel<<<c.num_sms, 256, 0, s>>>(h, P, r, cols, d_Ch, d_Yh, XL, d_H);
        c.batched_launches += 10 + 2 * c.nhid;
        if (Hout_dev) {
            cuda_check(cudaMemcpyAsync(Hout_dev, d_H, 8 * (size_t)N * r * r, cudaMemcpyDeviceToDevice, s), "H d2d");
            return;
        }
        std::vector<double> Hh((size_t)P * r * r);
        cuda_check(cudaMemcpyAsync(Hh.data(), d_H, 8 * Hh.size(), cudaMemcpyDeviceToHost, s), "H");
        cuda_check(cudaStreamSynchronize(s), "sync");
        std::memcpy(Hout, Hh.data(), 8 * (size_t)N * r * r);
    }

    // device buffer of a whole batch's Hessians (grown on demand, owned by the context)
    double* d_hall = nullptr;
    size_t hall_cap = 0;
    double* hess_all(Context& c, size_t count) {
        if (count > hall_cap) {
            if (d_hall) c.dfree(d_hall);
            d_hall = static_cast<double*>(c.dmalloc(8 * count));
            hall_cap = count;
        }
        return d_hall;
    }

    // fp32 copy of the element records (the fp64 context stores them in fp64)
    float* d_recf = nullptr;
    const void* rec_f32(Context& c) {
        if (c.precision == LSB_FP32) return c.d_rec;
        if (!d_recf) {
            const HostMesh& m = c.mesh;
            std::vector<float> rec(12 * (size_t)m.E);
            for (int e = 0; e < m.E; ++e) {
                for (int k = 0; k < 9; ++k) rec[12 * (size_t)e + k] = (float)m.Dminv[9 * (size_t)e + k];
                rec[12 * (size_t)e + 9] = (float)m.vol[e];
                rec[12 * (size_t)e + 10] = (float)c.mu[e];
                rec[12 * (size_t)e + 11] = (float)c.lambda[e];
            }
            d_recf = alloc<float>(rec.size());
            c.copy(d_recf, rec.data(), 4 * rec.size(), cudaMemcpyHostToDevice, "recf");
        }
        return d_recf;
    }
};

namespace {
__global__ void gate_kernel(int total, const float* g, const float* A, int act, float* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x)
        out[i] = g[i] * act_f(act, A[i], 1);
}
}  // namespace

void BatchedEngine::gate_mul(cudaStream_t s, int total, const float* g, const float* A, int act, float* out) {
    gate_kernel<<<(total + 255) / 256, 256, 0, s>>>(total, g, A, act, out);
}

static BatchedEngine& engine(Context& c) {
    if (!c.batched) {
        auto* e = new BatchedEngine();
        c.batched.reset(e);
        e->init(c);
    }
    return *static_cast<BatchedEngine*>(c.batched.get());
}

void batched_eval(Context& c, int B, const double* Z, double* E, double* G) {
    BatchedEngine& eng = engine(c);
    for (int b0 = 0; b0 < B; b0 += BatchedEngine::kGroup) {
        const int N = std::min(BatchedEngine::kGroup, B - b0);
        eng.run_group(c, N, Z + (size_t)b0 * c.r, E + b0, G ? G + (size_t)b0 * c.r : nullptr);
    }
}

// ReducedObjective::hessian (reduced_solver.cpp:204-229) at B points: the elastic Hessian plus,
// when the context has inertia set, the M / h^2 block and the inertia residual's curvature.
void batched_objective_hessian(Context& c, int B, const double* Z, double* H) {
    BatchedEngine& eng = engine(c);
    const int r = c.r;
    const int W = eng.pick_width(c, B);
    for (int b0 = 0; b0 < B; b0 += W) {
        const int N = std::min(W, B - b0);
        eng.run_hessian_chunk(c, N, Z + (size_t)b0 * r, H + (size_t)b0 * r * r, true, nullptr, W);
    }
}

void batched_hessian(Context& c, int B, const double* Z, double* H) {
    BatchedEngine& eng = engine(c);
    const int r = c.r;
    // all chunks write into one device buffer; a single copy and synchronisation at the end
    double* d_all = eng.hess_all(c, (size_t)B * r * r);
    const int W = eng.pick_width(c, B);
    for (int b0 = 0; b0 < B; b0 += W) {
        const int N = std::min(W, B - b0);
        eng.run_hessian_chunk(c, N, Z + (size_t)b0 * r, nullptr, false, d_all + (size_t)b0 * r * r, W);
    }
    c.copy(H, d_all, 8 * (size_t)B * r * r, cudaMemcpyDeviceToHost, "hessians");
}

// mean_p |H(z1_p) - H(z2_p)|_F^2 / |z1_p - z2_p|^2 (losses.cpp:196-213, order 2), fp64 combine:
// the Hessians stay on the device, |H1 - H2|^2 per pair comes from lipschitz_dldh_kernel (the
// reduction the gradient path uses), and the host sums d2 / |dz|^2 in pair order.
double lipschitz_loss(Context& c, int P, const double* Z1, const double* Z2) {
    BatchedEngine& eng = engine(c);
    const int r = c.r;
    std::vector<double> Z(2 * (size_t)P * r);
    for (int p = 0; p < P; ++p) {  // interleave z1, z2 so both Hessians of a pair share a chunk
        std::memcpy(&Z[(2 * (size_t)p) * r], Z1 + (size_t)p * r, 8 * r);
        std::memcpy(&Z[(2 * (size_t)p + 1) * r], Z2 + (size_t)p * r, 8 * r);
    }
    double* d_all = eng.hess_all(c, 2 * (size_t)P * r * r + P);
    double* d_d2 = d_all + 2 * (size_t)P * r * r;
    const int W = eng.pick_width(c, 2 * P);  // a multiple of 16: both points of a pair share a chunk
    for (int b0 = 0; b0 < 2 * P; b0 += W) {
        const int N = std::min(W, 2 * P - b0);
        eng.run_hessian_chunk(c, N, Z.data() + (size_t)b0 * r, nullptr, false, d_all + (size_t)b0 * r * r, W);
    }
    lipschitz_dldh_kernel<<<P, 256, 0, c.stream>>>(P, r, d_all, nullptr, nullptr, nullptr, d_d2);
    cuda_check(cudaGetLastError(), "pair losses");
    std::vector<double> d2(P);
    c.copy(d2.data(), d_d2, 8 * (size_t)P, cudaMemcpyDeviceToHost, "pair losses");
    double total = 0.0;
    for (int p = 0; p < P; ++p) {
        double dz2 = 0.0;
        for (int k = 0; k < r; ++k) dz2 += (Z1[(size_t)p * r + k] - Z2[(size_t)p * r + k]) * (Z1[(size_t)p * r + k] - Z2[(size_t)p * r + k]);
        total += d2[p] / dz2;
    }
    return total / P;
}

// Order-2 Lipschitz loss and dL/dtheta: grad holds, per decoder
// layer in order (hidden layers, then the output layer), W row-major then b.
double lipschitz_loss_grad(Context& c, int P, const double* Z1, const double* Z2, double* grad) {
    BatchedEngine& eng = engine(c);
    if (!eng.theta_ready) eng.init_theta(c);
    cuda_check(cudaMemsetAsync(eng.d_gW, 0, 8 * eng.gw_total, c.stream), "gW");
    cuda_check(cudaMemsetAsync(eng.d_gb, 0, 8 * eng.gb_total, c.stream), "gb");
    const int r = c.r;
    std::vector<double> Z(2 * (size_t)P * r);
    for (int p = 0; p < P; ++p) {
        std::memcpy(&Z[(2 * (size_t)p) * r], Z1 + (size_t)p * r, 8 * r);
        std::memcpy(&Z[(2 * (size_t)p + 1) * r], Z2 + (size_t)p * r, 8 * r);
    }
    double* d_d2 = static_cast<double*>(c.dmalloc(8 * (size_t)P));
    for (int b0 = 0; b0 < 2 * P; b0 += BatchedEngine::PH) {
        const int N = std::min(BatchedEngine::PH, 2 * P - b0);
        eng.run_theta_chunk(c, N, Z.data() + (size_t)b0 * r, 1.0 / P, d_d2 + b0 / 2);
    }
    std::vector<double> d2(P);
    c.copy(d2.data(), d_d2, 8 * (size_t)P, cudaMemcpyDeviceToHost, "pair losses");
    c.dfree(d_d2);
    double total = 0.0;  // losses.cpp:208-211: pair order
    for (int p = 0; p < P; ++p) {
        double dz2 = 0.0;
        for (int k = 0; k < r; ++k) dz2 += (Z1[p * r + k] - Z2[p * r + k]) * (Z1[p * r + k] - Z2[p * r + k]);
        total += d2[p] / dz2;
    }
    std::vector<double> gW(eng.gw_total), gb(eng.gb_total);
    c.copy(gW.data(), eng.d_gW, 8 * gW.size(), cudaMemcpyDeviceToHost, "gW");
    c.copy(gb.data(), eng.d_gb, 8 * gb.size(), cudaMemcpyDeviceToHost, "gb");
    size_t o = 0;
    for (int l = 0; l <= c.nhid; ++l) {
        const size_t nw = (l < c.nhid ? eng.gb_off[l + 1] : eng.gb_total) - eng.gb_off[l];
        const size_t ww = (l < c.nhid ? eng.gw_off[l + 1] : eng.gw_total) - eng.gw_off[l];
        std::memcpy(grad + o, gW.data() + eng.gw_off[l], 8 * ww);
        o += ww;
        std::memcpy(grad + o, gb.data() + eng.gb_off[l], 8 * nw);
        o += nw;
    }
    return total / P;
}

}  // namespace lsb
