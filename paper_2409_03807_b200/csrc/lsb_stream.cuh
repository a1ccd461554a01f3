// TMA-pipelined streaming of the decoder output layer W_out (n x hp, row-major).
//
// Both passes over W_out per evaluation (forward u = W y and the VJP
// ybar = W^T (s g)) are HBM-bound GEMVs.  Instead of relying on registers for
// memory-level parallelism, one producer warp per CTA issues 1-D bulk copies
// (cp.async.bulk, "TMA") of 16 KB row tiles into a STAGES-deep shared-memory
// ring guarded by mbarriers; eight consumer warps compute from shared memory.
// Bytes in flight per SM = STAGES x 16 KB x CTAs/SM, independent of registers.
#pragma once

#include "lsb_kernels.cuh"

namespace lsb {

template <typename TS, int HP>
struct StreamCfg {
    static constexpr int ROWB = HP * (int)sizeof(TS);
    static constexpr int TR = (8192 / ROWB) < 8 ? 8 : (8192 / ROWB);  // rows per tile (8 KB)
    static constexpr int TILEB = TR * ROWB;
    static constexpr int V4 = 16 / (int)sizeof(TS);  // elements per 16-byte chunk
    static constexpr int NPL = HP / 32;              // elements per lane per row
    static constexpr int NCH = NPL / V4;             // 16-byte chunks per lane per row
    // per-row side data staged with each tile: forward {b, s, shift - X, m, U slot, qbar - X}
    // (6 doubles), VJP tv (1 double)
    static constexpr int EPB = TR * 48;
    static constexpr int STAGEB = TILEB + EPB;
    static_assert(NCH >= 1, "row must span >= 32 x 16 bytes");
    static_assert(TILEB % 16 == 0 && STAGEB % 16 == 0, "stage alignment");
};

// Stage count of the streaming kernels' rings.  Tiles are consumed warp-per-tile
// (tile i by consumer warp i % 8), so the stage count MUST be a multiple of 8:
// then the previous user of a stage is the same warp, and a warp can never wait
// on a phase two behind (mbarrier parity aliasing).
constexpr int kStreamStages = 8;
constexpr int kStreamThreads = 288;  // 8 consumer warps + 1 producer warp

template <typename TS, int HP>
__host__ __device__ constexpr size_t stream_smem_bytes() {
    return (size_t)kStreamStages * StreamCfg<TS, HP>::STAGEB + 2 * kStreamStages * sizeof(uint64_t) + 128;
}

// 16-byte chunk idx of a row for this lane, widened to fp64.
template <typename TS>
__device__ __forceinline__ void lds_chunk(const TS* rowp, int idx, double* out);
template <>
__device__ __forceinline__ void lds_chunk<float>(const float* rowp, int idx, double* o) {
    const float4 v = *reinterpret_cast<const float4*>(rowp + idx * 4);
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
    o[3] = v.w;
}
template <>
__device__ __forceinline__ void lds_chunk<double>(const double* rowp, int idx, double* o) {
    const double2 v = *reinterpret_cast<const double2*>(rowp + idx * 2);
    o[0] = v.x;
    o[1] = v.y;
}

// Producer: stream tiles [t0, t1) of W_out plus per-row side data into the ring.
//   fwd: packed per-row record {b, s, shift - X, m, U slot, qbar - X}; vjp: tv.
template <typename TS, int HP, bool FWD>
__device__ __forceinline__ void stream_producer(const EvalParams<TS>& p, int t0, int t1, unsigned char* ring,
                                                uint64_t* full, uint64_t* empty) {
    using C = StreamCfg<TS, HP>;
    const uint64_t pol = l2_policy(p.w_resident);
    const uint64_t keep = l2_policy(1);
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
        const int s = i % kStreamStages, k = i / kStreamStages;
        if (k > 0) mbar_wait(&empty[s], (k - 1) & 1);
        const int r0 = t * C::TR;
        const int rows = min(C::TR, p.n - r0);
        unsigned char* st = ring + (size_t)s * C::STAGEB;
        const unsigned wbytes = (unsigned)rows * C::ROWB;
        if (FWD) {
            mbar_expect_tx(&full[s], wbytes + rows * 48);
            tma_load_1d(st, p.Wout + (size_t)r0 * HP, wbytes, &full[s], pol);
            tma_load_1d(st + C::TILEB, p.eprow + (size_t)r0 * 6, rows * 48, &full[s], keep);
        } else {
            const unsigned ub = ((unsigned)rows * 8 + 15) & ~15u;
            mbar_expect_tx(&full[s], wbytes + ub);
            tma_load_1d(st, p.Wout + (size_t)r0 * HP, wbytes, &full[s], pol);
            tma_load_1d(st + C::TILEB, p.tv + r0, ub, &full[s], keep);
        }
    }
}

// One warp computes every row of a forward tile: TR independent dot products,
// interleaved butterfly reductions, lane j runs the epilogue of row j.
template <typename TS, int HP>
__device__ __forceinline__ double fwd_tile(const EvalParams<TS>& p, const unsigned char* st, int t,
                                           const double (&y)[StreamCfg<TS, HP>::NCH][StreamCfg<TS, HP>::V4],
                                           int has_inertia, double inv_dt2, bool ident) {
    using C = StreamCfg<TS, HP>;
    const int lane = threadIdx.x & 31;
    const int rows = min(C::TR, p.n - t * C::TR);
    const TS* tile = reinterpret_cast<const TS*>(st);
    const double* ep = reinterpret_cast<const double*>(st + C::TILEB);
    double acc[C::TR];
#pragma unroll
    for (int j = 0; j < C::TR; ++j) {
        acc[j] = 0.0;
        if (j < rows) {
            const TS* rowp = tile + (size_t)j * HP;
#pragma unroll
            for (int c = 0; c < C::NCH; ++c) {
                double w[C::V4];
                lds_chunk<TS>(rowp, c * 32 + lane, w);
#pragma unroll
                for (int q = 0; q < C::V4; ++q) acc[j] = fma(w[q], y[c][q], acc[j]);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int j = 0; j < C::TR; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    double mine = 0.0;
#pragma unroll
    for (int j = 0; j < C::TR; ++j)
        if (lane == j) mine = acc[j];
    double e = 0.0;
    if (lane < rows) {
        const int row = t * C::TR + lane;
        const double* e6 = ep + lane * 6;
        const double a = mine + e6[0];
        double phi = a;
        if (!ident) {
            phi = act_eval(p.out_act, a, 0);
            p.dsout[row] = e6[1] * act_eval(p.out_act, a, 1);
        }
        const double uval = e6[1] * phi + e6[2];
        p.U[(int)e6[4]] = uval;
        if (has_inertia) {
            const double diff = uval - e6[5];
            p.rin[row] = inv_dt2 * (e6[3] * diff);
            e = e6[3] * diff * diff;
        }
    }
    return e;
}

// One warp accumulates a VJP tile into its per-lane column accumulators.
template <typename TS, int HP>
__device__ __forceinline__ void vjp_tile(const EvalParams<TS>& p, const unsigned char* st, int t,
                                         double (&acc)[StreamCfg<TS, HP>::NCH][StreamCfg<TS, HP>::V4]) {
    using C = StreamCfg<TS, HP>;
    const int lane = threadIdx.x & 31;
    const int rows = min(C::TR, p.n - t * C::TR);
    const TS* tile = reinterpret_cast<const TS*>(st);
    const double* tv = reinterpret_cast<const double*>(st + C::TILEB);
#pragma unroll
    for (int j = 0; j < C::TR; ++j) {
        if (j < rows) {
            const double tval = tv[j];
            const TS* rowp = tile + (size_t)j * HP;
#pragma unroll
            for (int c = 0; c < C::NCH; ++c) {
                double w[C::V4];
                lds_chunk<TS>(rowp, c * 32 + lane, w);
#pragma unroll
                for (int q = 0; q < C::V4; ++q) acc[c][q] = fma(w[q], tval, acc[c][q]);
            }
        }
    }
}

// ---------------------------------------------------------------- K2 (TMA): output layer forward
template <typename TS, int HP>
__global__ void __launch_bounds__(kStreamThreads) out_fwd_tma_kernel(const EvalParams<TS> p) {
    using C = StreamCfg<TS, HP>;
    extern __shared__ __align__(128) unsigned char ssm[];
    unsigned char* ring = ssm;
    uint64_t* full = reinterpret_cast<uint64_t*>(ssm + (size_t)kStreamStages * C::STAGEB);
    uint64_t* empty = full + kStreamStages;
    __shared__ double red[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < kStreamStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int ntiles = (p.n + C::TR - 1) / C::TR;
    const int t0 = (int)(((long long)ntiles * blockIdx.x) / gridDim.x);
    const int t1 = (int)(((long long)ntiles * (blockIdx.x + 1)) / gridDim.x);
    double eacc = 0.0;
    const double inv_dt2 = p.st->inv_dt2;
    if (warp == 8) {
        if (lane == 0) stream_producer<TS, HP, true>(p, t0, t1, ring, full, empty);
    } else {
        double y[C::NCH][C::V4];
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
#pragma unroll
            for (int q = 0; q < C::V4; ++q) y[c][q] = p.y_last[(c * 32 + lane) * C::V4 + q];
        const int has_inertia = p.st->has_inertia;
        const bool ident = p.out_act == kIdentity;
        // warp-per-tile: tile i is consumed entirely by warp i % 8
        for (int t = t0 + warp, i = warp; t < t1; t += 8, i += 8) {
            const int s = i % kStreamStages, k = i / kStreamStages;
            mbar_wait(&full[s], k & 1);
            const unsigned char* st = ring + (size_t)s * C::STAGEB;
            eacc += fwd_tile<TS, HP>(p, st, t, y, has_inertia, inv_dt2, ident);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
    const double tot = block_sum(eacc, red);
    if (tid == 0) p.e_part_out[blockIdx.x] = 0.5 * inv_dt2 * tot;
}

// ---------------------------------------------------------------- K3b: vertex gather (+ inertia)
// tv_i = s_i phi'(a_i) (sum of the per-tet forces on DOF i in ascending tet id
// + inertia residual) -- the full-space gradient times the output scaling.
// One free vertex, 4 cooperating lanes: lane q sums segment entries k = b + q,
// b + q + 4, ... of the vertex's CSR force vectors (ascending tet id), the four
// partials are combined in fixed lane order; + inertia, times s -> tv (3 rows).
// Must be called by all lanes of the warp (lanes 4v..4v+3 share vertex v).
template <typename TS>
__device__ __forceinline__ void gather_vertex4(const EvalParams<TS>& p, int f, int has_inertia, bool ident) {
    const int lane = threadIdx.x & 31, q = lane & 3;
    double gx = 0.0, gy = 0.0, gz = 0.0;
    if (f < p.n_free) {
        const int b = __ldg(p.csr_ptr + f), e = __ldg(p.csr_ptr + f + 1);
        const double2* F = reinterpret_cast<const double2*>(p.forces);
#pragma unroll 4
        for (int k = b + q; k < e; k += 4) {
            const double2 a = __ldcg(F + 2 * (size_t)k);
            const double2 c = __ldcg(F + 2 * (size_t)k + 1);
            gx += a.x;
            gy += a.y;
            gz += c.x;
        }
    }
    // fixed-order combine: (q0 + q1) + (q2 + q3)
    gx += __shfl_xor_sync(0xffffffffu, gx, 1);
    gy += __shfl_xor_sync(0xffffffffu, gy, 1);
    gz += __shfl_xor_sync(0xffffffffu, gz, 1);
    gx += __shfl_xor_sync(0xffffffffu, gx, 2);
    gy += __shfl_xor_sync(0xffffffffu, gy, 2);
    gz += __shfl_xor_sync(0xffffffffu, gz, 2);
    if (f < p.n_free && q < 3) {
        const int row = 3 * f + q;
        double g = q == 0 ? gx : (q == 1 ? gy : gz);
        if (has_inertia) g += __ldcg(p.rin + row);
        p.tv[row] = g * (ident ? p.eprow[6 * (size_t)row + 1] : __ldcg(p.dsout + row));
    }
}

template <typename TS>
__global__ void __launch_bounds__(256) gather_kernel(const EvalParams<TS> p) {
    const DevState* st = p.st;
    if (!st->need_grad) return;
    const bool ident = p.out_act == kIdentity;
    const int has_inertia = st->has_inertia;
    const int nthr = gridDim.x * blockDim.x;
    // warp-uniform trip count: gather_vertex4 shuffles across the whole warp
    for (int wb = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; wb < 4 * p.n_free; wb += nthr)
        gather_vertex4(p, (wb + (threadIdx.x & 31)) >> 2, has_inertia, ident);
}

// ---------------------------------------------------------------- K4 (TMA): VJP partials
template <typename TS, int HP>
__global__ void __launch_bounds__(kStreamThreads) vjp_tma_kernel(const EvalParams<TS> p) {
    using C = StreamCfg<TS, HP>;
    extern __shared__ __align__(128) unsigned char ssm[];
    unsigned char* ring = ssm;
    uint64_t* full = reinterpret_cast<uint64_t*>(ssm + (size_t)kStreamStages * C::STAGEB);
    uint64_t* empty = full + kStreamStages;
    double* wred = reinterpret_cast<double*>(empty + kStreamStages);  // 8 x HP
    __shared__ int am_grp_last;
    DevState* st = p.st;
    if (!st->need_grad) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < kStreamStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int ntiles = (p.n + C::TR - 1) / C::TR;
    const int t0 = (int)(((long long)ntiles * blockIdx.x) / gridDim.x);
    const int t1 = (int)(((long long)ntiles * (blockIdx.x + 1)) / gridDim.x);
    double acc[C::NCH][C::V4];
#pragma unroll
    for (int c = 0; c < C::NCH; ++c)
#pragma unroll
        for (int q = 0; q < C::V4; ++q) acc[c][q] = 0.0;
    if (warp == 8) {
        if (lane == 0) stream_producer<TS, HP, false>(p, t0, t1, ring, full, empty);
    } else {
        for (int t = t0 + warp, i = warp; t < t1; t += 8, i += 8) {
            const int s = i % kStreamStages, k = i / kStreamStages;
            mbar_wait(&full[s], k & 1);
            vjp_tile<TS, HP>(p, ring + (size_t)s * C::STAGEB, t, acc);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
#pragma unroll
            for (int q = 0; q < C::V4; ++q) wred[warp * HP + (c * 32 + lane) * C::V4 + q] = acc[c][q];
    }
    __syncthreads();
    for (int j = tid; j < HP; j += blockDim.x) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += wred[w * HP + j];
        p.ybar_part[(size_t)blockIdx.x * HP + j] = s;
    }
    // group-last block sums its group's partials in block order
    __threadfence();
    __syncthreads();
    const int grp = blockIdx.x / p.group;
    const int g0 = grp * p.group, g1 = min(g0 + p.group, (int)gridDim.x);
    if (tid == 0) {
        const unsigned prev = atomicAdd(p.grp_cnt + grp, 1u);
        am_grp_last = (prev == (unsigned)(g1 - g0 - 1));
    }
    __syncthreads();
    if (!am_grp_last) return;
    __threadfence();
    for (int j = tid; j < HP; j += blockDim.x) {
        double s = 0.0;
        for (int b = g0; b < g1; ++b) s += __ldcg(p.ybar_part + (size_t)b * HP + j);
        p.ybar_grp[(size_t)grp * HP + j] = s;
    }
    if (tid == 0) p.grp_cnt[grp] = 0;
}

}  // namespace lsb
