// tcgen05 (5th-generation tensor core) GEMMs of the batched path (config 4 and the
// config-5 tangent VJP): the output layer's forward C = W_out Y and its VJP
// Ybar = W_out^T T over a batch of latent columns.
//
// Both are D(128 x N) = sum over 32-wide K slices of A_s (128 x 32) . B_s (N x 32)^T,
// computed as 3xTF32 (hi.hi + hi.lo + lo.hi, fixed order) for ~fp32 accuracy:
// tf32 keeps 10 mantissa bits, x = hi + lo with hi = rna_tf32(x) and lo = x - hi.
//
// Operand layout: every slice is pre-tiled into the canonical SWIZZLE_NONE
// K-major UMMA layout (8-row x 16-byte core matrices; core (chunk c, row group g)
// at ((c * R/8) + g) * 128 B, so SBO = 128 B between row groups and LBO = R * 16 B
// between the two 16-byte K chunks one MMA consumes), hi block then lo block,
// contiguous -- one 1-D bulk copy (TMA) per operand per slice.
//
// Kernel roles (192 threads): warps 0-3 epilogue (TMEM lane quarter = warp),
// warp 4 lane 0 TMA producer, warp 5 lane 0 MMA issuer.  A 3-stage smem ring
// (full/empty mbarriers; the MMA frees a stage with tcgen05.commit), and two TMEM
// accumulators (acc_full/acc_empty) so the epilogue of job j overlaps the MMAs of j+1.
//
//   mode 0 (forward): job = 128-row tile of W_out, its S slices against the same
//                     B slices (Y^T); rows written to C (row-major, ldc).
//   mode 1 (VJP):     one 128-row A (W_out^T, h <= 128), job = contiguous slice range
//                     (split-K); 128 x N partial per job, reduced in job order.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lsb_common.cuh"

namespace lsb {
namespace tc {

constexpr int kSliceK = 32;  // K elements (fp32 / tf32) per slice
constexpr int kTileM = 128;
constexpr int kStages = 3;  // maximum ring depth (N = 256 tiles fit 2)
constexpr int kThreads = 192;

__host__ __device__ constexpr size_t slice_floats(int rows) { return 2 * (size_t)rows * kSliceK; }  // hi + lo

// element (row, kk) of one hi-or-lo block with R rows (kk < 32)
__host__ __device__ inline size_t core_off(int row, int kk, int R) {
    const int c = kk >> 2, e = kk & 3, g = row >> 3, r = row & 7;
    return (((size_t)c * (R >> 3) + g) * 8 + r) * 4 + e;
}

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t u;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
    return __uint_as_float(u);
}

// Pack a strided fp32 matrix (element (row, k) = src[row * srs + k * sks], rows x K)
// into tiles of R rows x S slices: block (tile t, slice s) at ((t * S) + s) * 2R*32.
// Rows >= rows and k >= K are zero.
__global__ void pack_kernel(const float* __restrict__ src, long long srs, long long sks, int rows, int K, int R,
                            int tiles, int S, float* __restrict__ dst) {
    const long long total = (long long)tiles * R * S * kSliceK;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        // i enumerates (tile, slice, row, kk): kk fastest when k is the contiguous source
        // dimension (sks == 1), row fastest otherwise -- coalesced reads either way
        int kk, row;
        long long q;
        if (sks == 1) {
            kk = (int)(i % kSliceK);
            q = i / kSliceK;
            row = (int)(q % R);
            q /= R;
        } else {
            row = (int)(i % R);
            q = i / R;
            kk = (int)(q % kSliceK);
            q /= kSliceK;
        }
        const int s = (int)(q % S);
        const int t = (int)(q / S);
        const int grow = t * R + row, k = s * kSliceK + kk;
        const float x = (grow < rows && k < K) ? src[(long long)grow * srs + (long long)k * sks] : 0.f;
        const float hi = tf32_rna(x);
        float* blk = dst + ((size_t)t * S + s) * slice_floats(R);
        const size_t o = core_off(row, kk, R);
        blk[o] = hi;
        blk[(size_t)R * kSliceK + o] = x - hi;
    }
}

// ---- PTX wrappers -------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    // base_offset 0, lbo_mode 0, layout_type 0 = SWIZZLE_NONE
    return d;
}
// kind::tf32, D f32, A/B tf32, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t make_idesc(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct GemmArgs {
    const float* A;  // pre-tiled A slices (128 rows each)
    const float* B;  // pre-tiled B slices (N rows each)
    float* out;
    int mode;        // 0 forward (jobs = A tiles), 1 split-K partials
    int njobs;
    int S;           // mode 0: slices per job; mode 1: total slices
    int N;           // batch columns (multiple of 32, <= 256)
    int ldc;         // mode 0: row stride of out
    int m_valid;     // mode 0: valid rows of out
    uint32_t tmem_cols;
    int stages;  // ring depth (<= kStages, by shared memory)
    int ntn;     // mode 3: N tiles per M tile (job j -> M tile j / ntn, N tile j % ntn)
    int ncols;   // mode 3: valid output columns
    // mode 2 (forward with the output-layer epilogue fused): u = s (C + b) + shift - X ->
    // U[slot][col]; inertia residual rin[row][col]; per-column energy partial per 128-row tile
    const double* eprow;  // n x 6 {b, s, shift - X, m, U slot, qbar - X}
    const double* ut;     // q-bar - X (unused: taken from eprow col 5)
    float* U;
    float* rin;
    double* epart;        // [tiles][N]
    int has_inertia;
    double inv_dt2;
    // mode 4 (general tile grid with the tangent-output epilogue fused): output columns are
    // [u (P) | J (P x r)] per row; u = s (C + b) + shift - X -> U[slot][p], J = s C -> Jv[slot][p][a]
    // (one contiguous run per row), inertia residual rin[row][p]
    float* Jv = nullptr;
    int P = 0, r = 0;
};

__device__ __forceinline__ void job_slices(const GemmArgs& g, int j, int& s0, int& s1) {
    if (g.mode != 1) {
        s0 = 0;
        s1 = g.S;
    } else {
        s0 = (int)((long long)g.S * j / g.njobs);
        s1 = (int)((long long)g.S * (j + 1) / g.njobs);
    }
}

__global__ void __launch_bounds__(kThreads, 1) gemm3_kernel(const GemmArgs g) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_base_s;
    __shared__ double esum_s[4][256];  // mode 2: per-warp column energy partials
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int N = g.N;
    const uint32_t a_bytes = (uint32_t)(slice_floats(kTileM) * 4), b_bytes = (uint32_t)(slice_floats(N) * 4);
    const uint32_t stage_bytes = a_bytes + b_bytes;
    if (tid == 0) {
        for (int s = 0; s < g.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], 128);
        }
        mbar_fence_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                     "r"(g.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;

    if (warp == 4) {
        // ---- TMA producer
        if (lane == 0) {
            const uint64_t pol_b = l2_policy(1);  // B slices: shared by every CTA
            uint64_t pol_a;
            asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_a));
            int it = 0;
            for (int j = blockIdx.x; j < g.njobs; j += gridDim.x) {
                int s0, s1;
                job_slices(g, j, s0, s1);
                for (int s = s0; s < s1; ++s, ++it) {
                    const int st = it % g.stages, u = it / g.stages;
                    if (u > 0) mbar_wait(&empty[st], (u - 1) & 1);
                    unsigned char* sa = smem + (size_t)st * stage_bytes;
                    const bool grid2d = g.mode == 3 || g.mode == 4;  // job = (M tile, N tile)
                    const size_t a_slice = grid2d ? (size_t)(j / g.ntn) * g.S + s
                                                  : (g.mode != 1 ? (size_t)j * g.S + s : (size_t)s);
                    const size_t b_slice = grid2d ? (size_t)(j % g.ntn) * g.S + s : (size_t)s;
                    mbar_expect_tx(&full[st], stage_bytes);
                    tma_load_1d(sa, g.A + a_slice * slice_floats(kTileM), a_bytes, &full[st], pol_a);
                    tma_load_1d(sa + a_bytes, g.B + b_slice * slice_floats(N), b_bytes, &full[st], pol_b);
                }
            }
        }
    } else if (warp == 5) {
        // ---- MMA issuer (single thread)
        if (lane == 0) {
            const uint32_t idesc = make_idesc(N);
            int it = 0, jl = 0;
            for (int j = blockIdx.x; j < g.njobs; j += gridDim.x, ++jl) {
                const int acc = jl & 1, u = jl >> 1;
                if (u > 0) mbar_wait(&acc_empty[acc], (u - 1) & 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * N);
                int s0, s1;
                job_slices(g, j, s0, s1);
                for (int s = s0; s < s1; ++s, ++it) {
                    const int st = it % g.stages;
                    mbar_wait(&full[st], (it / g.stages) & 1);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + (size_t)st * stage_bytes);
                    const uint32_t sb = sa + a_bytes;
                    const uint32_t a_lo = (uint32_t)(kTileM * kSliceK * 4), b_lo = (uint32_t)(N * kSliceK * 4);
#pragma unroll
                    for (int ks = 0; ks < kSliceK / 8; ++ks) {
                        // one MMA consumes K = 8 tf32 = two 16-byte chunks
                        const uint32_t ao = (uint32_t)ks * 2 * (kTileM / 8) * 128, bo = (uint32_t)ks * 2 * (N / 8) * 128;
                        const uint64_t ahi = make_desc(sa + ao, kTileM * 16, 128);
                        const uint64_t alo = make_desc(sa + a_lo + ao, kTileM * 16, 128);
                        const uint64_t bhi = make_desc(sb + bo, (uint32_t)N * 16, 128);
                        const uint64_t blo = make_desc(sb + b_lo + bo, (uint32_t)N * 16, 128);
                        mma_tf32(d, ahi, bhi, idesc, (s > s0 || ks > 0) ? 1u : 0u);
                        mma_tf32(d, ahi, blo, idesc, 1u);
                        mma_tf32(d, alo, bhi, idesc, 1u);
                    }
                    mma_commit(&empty[st]);  // stage reusable once these MMAs have read it
                }
                // (an empty job issues no MMA; its epilogue writes zeros)
                mma_commit(&acc_full[acc]);
            }
        }
    } else {
        // ---- epilogue: warps 0-3, thread = accumulator row
        const int row = warp * 32 + lane;
        int jl = 0;
        for (int j = blockIdx.x; j < g.njobs; j += gridDim.x, ++jl) {
            const int acc = jl & 1, u = jl >> 1;
            mbar_wait(&acc_full[acc], u & 1);
            tc_fence_after();
            int s0, s1;
            job_slices(g, j, s0, s1);
            const bool empty_job = s1 == s0;
            for (int c0 = 0; c0 < N; c0 += 32) {
                float v[32];
                tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * N + c0), v);
                if (empty_job) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = 0.f;
                }
                if (g.mode == 2) {
                    // fused output-layer epilogue for row grow, columns c0..c0+31
                    const int grow = j * kTileM + row;
                    double e[32];
                    if (grow < g.m_valid) {
                        const double* e6 = g.eprow + (size_t)grow * 6;
                        const double b = e6[0], s = e6[1], sh = e6[2], m = e6[3], qb = e6[5];
                        const int slot = (int)e6[4];
                        float* Ur = g.U + ((size_t)(slot >> 2) * 3 + (slot & 3)) * N + c0;
                        float* Rr = g.rin + (size_t)grow * N + c0;
#pragma unroll
                        for (int i = 0; i < 32; i += 4) {
                            float4 uo, ro;
                            float* up = &uo.x;
                            float* rp = &ro.x;
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const double u = s * ((double)v[i + q] + b) + sh;
                                up[q] = (float)u;
                                const double d = u - qb;
                                rp[q] = (float)(g.inv_dt2 * m * d);
                                e[i + q] = g.has_inertia ? m * d * d : 0.0;
                            }
                            *reinterpret_cast<float4*>(Ur + i) = uo;
                            if (g.has_inertia) *reinterpret_cast<float4*>(Rr + i) = ro;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) e[i] = 0.0;
                    }
                    // per-column sums over the warp's 32 rows: recursive halving, lane c ends with
                    // column c0 + c (fixed order)
#pragma unroll
                    for (int o = 16, nn = 32; o > 0; o >>= 1) {
                        nn >>= 1;
                        const bool up = (lane & o) != 0;
#pragma unroll
                        for (int k = 0; k < nn; ++k) {
                            const double give = up ? e[k] : e[k + nn];
                            const double keep = up ? e[k + nn] : e[k];
                            e[k] = keep + __shfl_xor_sync(0xffffffffu, give, o);
                        }
                    }
                    // lane l holds column c0 + bitrev-free index: lanes with bit o set kept the upper
                    // half at each step -> column = lane
                    esum_s[warp][c0 + lane] = e[0];
                    continue;
                }
                if (g.mode == 4) {  // tangent output: columns [u (P) | J (P r)], 4-column groups never straddle P
                    const int grow = (j / g.ntn) * kTileM + row;
                    const int col0 = (j % g.ntn) * N + c0;
                    if (grow < g.m_valid) {
                        const double* e6 = g.eprow + (size_t)grow * 6;
                        const double b = e6[0], sc = e6[1], sh = e6[2], m = e6[3], qb = e6[5];
                        const int slot = (int)e6[4];
                        const size_t vc = (size_t)(slot >> 2) * 3 + (slot & 3);
                        float* Ur = g.U + vc * g.P;
                        float* Jr = g.Jv + vc * g.P * g.r;
#pragma unroll
                        for (int i = 0; i < 32; i += 4) {
                            const int col = col0 + i;
                            if (col >= g.ncols) break;
                            if (col < g.P) {
                                float4 uo, ro;
                                float* up = &uo.x;
                                float* rp = &ro.x;
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    const double u = sc * ((double)v[i + q] + b) + sh;
                                    up[q] = (float)u;
                                    rp[q] = (float)(g.inv_dt2 * m * (u - qb));
                                }
                                *reinterpret_cast<float4*>(Ur + col) = uo;
                                if (g.has_inertia) *reinterpret_cast<float4*>(g.rin + (size_t)grow * g.P + col) = ro;
                            } else {
                                *reinterpret_cast<float4*>(Jr + (col - g.P)) =
                                    make_float4((float)(sc * v[i]), (float)(sc * v[i + 1]), (float)(sc * v[i + 2]),
                                                (float)(sc * v[i + 3]));
                            }
                        }
                    }
                    continue;
                }
                if (g.mode == 3) {  // general tile grid, masked columns
                    const int grow = (j / g.ntn) * kTileM + row;
                    const int col0 = (j % g.ntn) * N + c0;
                    if (grow < g.m_valid) {
                        float* d3 = g.out + (size_t)grow * g.ldc + col0;
                        if (col0 + 32 <= g.ncols && (g.ldc & 3) == 0) {
#pragma unroll
                            for (int i = 0; i < 32; i += 4)
                                *reinterpret_cast<float4*>(d3 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                        } else {
                            for (int i = 0; i < 32 && col0 + i < g.ncols; ++i) d3[i] = v[i];
                        }
                    }
                    continue;
                }
                float* dst;
                if (g.mode == 0) {
                    const int grow = j * kTileM + row;
                    if (grow >= g.m_valid) continue;
                    dst = g.out + (size_t)grow * g.ldc + c0;
                } else {
                    dst = g.out + ((size_t)j * kTileM + row) * N + c0;
                }
#pragma unroll
                for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            }
            tc_fence_before();
            mbar_arrive(&acc_empty[acc]);
            if (g.mode == 2) {
                named_bar_sync(1, 128);  // the 4 epilogue warps' column partials are in esum_s
                for (int c = threadIdx.x; c < N; c += 128)
                    g.epart[(size_t)j * N + c] =
                        0.5 * g.inv_dt2 * ((esum_s[0][c] + esum_s[1][c]) + (esum_s[2][c] + esum_s[3][c]));
                named_bar_sync(1, 128);  // esum_s reusable for the next job
            }
        }
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(g.tmem_cols) : "memory");
    }
}

// Ybar[m][b] = sum_j part[j][m][b] (job order), m < h
__global__ void reduce_parts_kernel(const float* __restrict__ part, int njobs, int h, int N, float* __restrict__ out,
                                    int ldo) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < h * N; i += gridDim.x * blockDim.x) {
        // 8 independent loads in flight, summed in job order
        float s = 0.f;
        int j = 0;
        for (; j + 8 <= njobs; j += 8) {
            float v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __ldg(part + (size_t)(j + k) * kTileM * N + i);
#pragma unroll
            for (int k = 0; k < 8; ++k) s += v[k];
        }
        for (; j < njobs; ++j) s += __ldg(part + (size_t)j * kTileM * N + i);
        out[(size_t)(i / N) * ldo + i % N] = s;
    }
}

}  // namespace tc

// Host side: owns the pre-tiled W_out operands and the per-call B / partial buffers.
struct TcGemm {
    bool enabled = false;
    int n = 0, h = 0, N = 0, S1 = 0, S2 = 0, tiles1 = 0, jobs2 = 0, sms = 0;
    float *A1 = nullptr, *A2 = nullptr, *B1 = nullptr, *B2 = nullptr, *part = nullptr;
    size_t smem = 0;
    uint32_t tmem_cols = 0;
    int stages = tc::kStages;
    long long launches = 0;

    static void* dalloc(size_t bytes) {
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, bytes), "tc malloc");
        return p;
    }

    // W: device fp32 n x h row-major.  N = batch columns per call.
    void init(cudaStream_t s, const float* W, int n_, int h_, int N_, int num_sms) {
        if (h_ > tc::kTileM || N_ % 32 != 0 || N_ > 256 || N_ < 32) return;
        n = n_;
        h = h_;
        N = N_;
        sms = num_sms;
        S1 = (h + tc::kSliceK - 1) / tc::kSliceK;
        S2 = (n + tc::kSliceK - 1) / tc::kSliceK;
        tiles1 = (n + tc::kTileM - 1) / tc::kTileM;
        jobs2 = std::min(S2, num_sms);
        A1 = static_cast<float*>(dalloc(sizeof(float) * tc::slice_floats(tc::kTileM) * (size_t)tiles1 * S1));
        A2 = static_cast<float*>(dalloc(sizeof(float) * tc::slice_floats(tc::kTileM) * (size_t)S2));
        B1 = static_cast<float*>(dalloc(sizeof(float) * tc::slice_floats(N) * (size_t)S1));
        B2 = static_cast<float*>(dalloc(sizeof(float) * tc::slice_floats(N) * (size_t)S2));
        cuda_check(cudaMemsetAsync(B2, 0, sizeof(float) * tc::slice_floats(N) * (size_t)S2, s), "tc B2");  // K padding
        part = static_cast<float*>(dalloc(sizeof(float) * (size_t)jobs2 * tc::kTileM * N));
        // A1: W rows x h (K); A2: W^T = h rows x n (K)
        tc::pack_kernel<<<num_sms * 8, 256, 0, s>>>(W, h, 1, n, h, tc::kTileM, tiles1, S1, A1);
        tc::pack_kernel<<<num_sms * 8, 256, 0, s>>>(W, 1, h, h, n, tc::kTileM, 1, S2, A2);
        cuda_check(cudaGetLastError(), "tc pack W");
        stages = tc::kStages;
        while (stages > 1 && (size_t)stages * (tc::slice_floats(tc::kTileM) + tc::slice_floats(N)) * 4 > 220 * 1024)
            --stages;
        smem = (size_t)stages * (tc::slice_floats(tc::kTileM) + tc::slice_floats(N)) * 4;
        if (stages < 2) {
            release();
            return;
        }
        tmem_cols = 32;
        while (tmem_cols < (uint32_t)(2 * N)) tmem_cols <<= 1;
        cuda_check(cudaFuncSetAttribute(tc::gemm3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                   "tc smem");
        cuda_check(cudaStreamSynchronize(s), "tc init");
        enabled = true;
    }
    void release() {
        if (Bg) cudaFree(Bg);
        Bg = nullptr;
        Bg_floats = 0;
        for (float* p : {A1, A2, B1, B2, part})
            if (p) cudaFree(p);
        A1 = A2 = B1 = B2 = part = nullptr;
        enabled = false;
    }

    // C (n x N, row-major, ldc = N) = W Y, Y: h x N (feature-major, row stride ldy)
    bool gemm_out(cudaStream_t s, const float* Y, int ldy, float* C) {
        if (!enabled) return false;
        tc::pack_kernel<<<sms * 2, 256, 0, s>>>(Y, 1, ldy, N, h, N, 1, S1, B1);
        tc::GemmArgs a{A1, B1, C, 0, tiles1, S1, N, N, n, tmem_cols, stages, 1, N, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0.0};
        tc::gemm3_kernel<<<std::min(tiles1, sms), tc::kThreads, smem, s>>>(a);
        launches += 2;
        return true;
    }
    // Forward with the output-layer epilogue fused (mode 2): U, rin and per-128-row-tile
    // energy partials epart[tiles1][N] straight from TMEM.
    bool gemm_out_fused(cudaStream_t s, const float* Y, int ldy, const double* eprow, float* U, float* rin,
                        double* epart, int has_inertia, double inv_dt2) {
        if (!enabled) return false;
        tc::pack_kernel<<<sms * 2, 256, 0, s>>>(Y, 1, ldy, N, h, N, 1, S1, B1);
        tc::GemmArgs a{A1, B1, nullptr, 2, tiles1, S1, N, N, n, tmem_cols, stages, 1, N, eprow, nullptr, U,
                       rin, epart, has_inertia, inv_dt2};
        tc::gemm3_kernel<<<std::min(tiles1, sms), tc::kThreads, smem, s>>>(a);
        launches += 2;
        return true;
    }

    // General C (M x ncols, row stride ldc) = A B on a tile grid: A pre-tiled (tiles_m x S slices,
    // pack_rows), B feature-major (K x ncols, row stride ldb) packed here into 256-column tiles.
    float* Bg = nullptr;
    size_t Bg_floats = 0;
    bool gemm_general(cudaStream_t s, const float* Apacked, int tiles_m, int S, int m_valid, const float* B, int ldb,
                      int K, int ncols, float* C, int ldc) {
        if (!enabled || N != 256) return false;
        const int ntn = (ncols + N - 1) / N;
        const size_t need = (size_t)ntn * S * tc::slice_floats(N);
        if (need > Bg_floats) {
            if (Bg) cudaFree(Bg);
            Bg = static_cast<float*>(dalloc(sizeof(float) * need));
            Bg_floats = need;
        }
        tc::pack_kernel<<<sms * 8, 256, 0, s>>>(B, 1, ldb, ncols, K, N, ntn, S, Bg);
        tc::GemmArgs a{Apacked, Bg, C, 3, tiles_m * ntn, S, N, ldc, m_valid, tmem_cols, stages, ntn, ncols,
                       nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0.0};
        tc::gemm3_kernel<<<std::min(tiles_m * ntn, sms), tc::kThreads, smem, s>>>(a);
        launches += 2;
        return true;
    }
    // gemm_general on the output layer with the tangent-output epilogue fused (mode 4): B holds the columns
    // [y (P) | tangents (P x r)] feature-major; writes U, Jv (and rin with inertia) instead of C.
    bool gemm_tangent_out(cudaStream_t s, const float* B, int K, int P, int r, const double* eprow, float* U, float* Jv,
                          float* rin, int has_inertia, double inv_dt2) {
        if (!enabled || N != 256 || (P & 3)) return false;
        const int ncols = P * (1 + r);
        const int ntn = (ncols + N - 1) / N;
        const size_t need = (size_t)ntn * S1 * tc::slice_floats(N);
        if (need > Bg_floats) {
            if (Bg) cudaFree(Bg);
            Bg = static_cast<float*>(dalloc(sizeof(float) * need));
            Bg_floats = need;
        }
        tc::pack_kernel<<<sms * 8, 256, 0, s>>>(B, 1, ncols, ncols, K, N, ntn, S1, Bg);
        tc::GemmArgs a{A1, Bg, nullptr, 4, tiles1 * ntn, S1, N, 0, n, tmem_cols, stages, ntn, ncols,
                       eprow, nullptr, U, rin, nullptr, has_inertia, inv_dt2};
        a.Jv = Jv;
        a.P = P;
        a.r = r;
        tc::gemm3_kernel<<<std::min(tiles1 * ntn, sms), tc::kThreads, smem, s>>>(a);
        launches += 2;
        return true;
    }
    // Pack a row-major fp32 matrix (rows x K) as A tiles (128-row tiles, S = ceil(K / 32)
    // slices) into dst, which holds packed_a_floats(rows, K) floats.
    static size_t packed_a_floats(int rows, int K) {
        return tc::slice_floats(tc::kTileM) * (size_t)((rows + tc::kTileM - 1) / tc::kTileM) *
               ((K + tc::kSliceK - 1) / tc::kSliceK);
    }
    void pack_a(cudaStream_t s, const float* W, int rows, int K, float* dst, int& tiles_m, int& S) const {
        tiles_m = (rows + tc::kTileM - 1) / tc::kTileM;
        S = (K + tc::kSliceK - 1) / tc::kSliceK;
        tc::pack_kernel<<<sms * 4, 256, 0, s>>>(W, K, 1, rows, K, tc::kTileM, tiles_m, S, dst);
    }

    // VJP with B already packed into B2 by the caller (combine_pack_kernel)
    bool gemm_vjp_prepacked(cudaStream_t s, float* Ybar, int ldo) {
        if (!enabled) return false;
        tc::GemmArgs a{A2, B2, part, 1, jobs2, S2, N, 0, 0, tmem_cols, stages, 1, N, nullptr, nullptr, nullptr, nullptr, nullptr,
                       0, 0.0};
        tc::gemm3_kernel<<<jobs2, tc::kThreads, smem, s>>>(a);
        tc::reduce_parts_kernel<<<sms * 2, 256, 0, s>>>(part, jobs2, h, N, Ybar, ldo);
        launches += 2;
        return true;
    }

    // Ybar (h x N, row stride ldo) = W^T T, T: n x N (row-major)
    bool gemm_vjp(cudaStream_t s, const float* T, float* Ybar, int ldo) {
        if (!enabled) return false;
        tc::pack_kernel<<<sms * 8, 256, 0, s>>>(T, 1, N, N, n, N, 1, S2, B2);
        tc::GemmArgs a{A2, B2, part, 1, jobs2, S2, N, 0, 0, tmem_cols, stages, 1, N, nullptr, nullptr, nullptr, nullptr, nullptr,
                       0, 0.0};
        tc::gemm3_kernel<<<jobs2, tc::kThreads, smem, s>>>(a);
        tc::reduce_parts_kernel<<<sms * 2, 256, 0, s>>>(part, jobs2, h, N, Ybar, ldo);
        launches += 3;
        return true;
    }
};

}  // namespace lsb
