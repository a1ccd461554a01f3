// TMA-pipelined streaming of the decoder output layer W_out (n x hp, row-major).
//
// Both passes over W_out per evaluation (forward u = W y and the VJP
// ybar = W^T (s g)) are HBM-bound GEMVs.  Rows are cut into ~8 KB tiles; each
// warp owns SPW shared-memory stages and issues its OWN 1-D bulk copies
// (cp.async.bulk, "TMA") for the tiles it will consume next (tile t0 + w + NW*i
// goes to warp w, slot i % SPW), waiting only on its own full mbarriers.  No
// producer warp and no empty barriers: measured on B200 (tools/probe/stream_bw),
// a single producer thread caps the stream at ~4.0 TB/s with 8 KB copies, while
// per-warp issue reaches 5.8 TB/s cold / 6.5 TB/s L2-warm.
#pragma once

#include <type_traits>

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

constexpr int kStreamThreads = 256;  // stream kernels: 8 warps, every warp consumes and issues
constexpr int kStreamSpw = 1;        // stages per warp in the stream kernels (several CTAs per SM)

template <typename TS, int HP>
__host__ __device__ constexpr size_t stream_smem_bytes() {
    return (size_t)(kStreamThreads / 32) * kStreamSpw * StreamCfg<TS, HP>::STAGEB + 512;
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

// ---- per-warp bulk-copy issue (lane 0 only) ---------------------------------------------------
// forward tile t: W rows + packed per-row records {b, s, shift - X, m, U slot, qbar - X}
template <typename TS, int HP>
__device__ __forceinline__ void issue_fwd(const EvalParams<TS>& p, int t, unsigned char* stg, uint64_t* bar,
                                          uint64_t pol, uint64_t keep) {
    using C = StreamCfg<TS, HP>;
    const int r0 = t * C::TR, rows = min(C::TR, p.n - r0);
    mbar_expect_tx(bar, (unsigned)rows * C::ROWB + rows * 48);
    tma_load_1d(stg, p.Wout + (size_t)r0 * HP, rows * C::ROWB, bar, pol);
    tma_load_1d(stg + C::TILEB, p.eprow + (size_t)r0 * 6, rows * 48, bar, keep);
}
template <typename TS, int HP>
__device__ __forceinline__ unsigned tv_bytes(const EvalParams<TS>& p, int t) {
    using C = StreamCfg<TS, HP>;
    const int rows = min(C::TR, p.n - t * C::TR);
    return ((unsigned)rows * 8 + 15) & ~15u;  // tv is padded to a 16-byte multiple
}
// VJP tile t, W part (may be issued before tv is ready: expect_tx covers both parts)
template <typename TS, int HP>
__device__ __forceinline__ void issue_vjp_w(const EvalParams<TS>& p, int t, unsigned char* stg, uint64_t* bar,
                                            uint64_t pol) {
    using C = StreamCfg<TS, HP>;
    const int r0 = t * C::TR, rows = min(C::TR, p.n - r0);
    mbar_expect_tx(bar, (unsigned)rows * C::ROWB + tv_bytes<TS, HP>(p, t));
    tma_load_1d(stg, p.Wout + (size_t)r0 * HP, rows * C::ROWB, bar, pol);
}
// VJP tile t, W rows only (tv comes from shared memory)
template <typename TS, int HP>
__device__ __forceinline__ void issue_w_only(const EvalParams<TS>& p, int t, unsigned char* stg, uint64_t* bar,
                                             uint64_t pol) {
    using C = StreamCfg<TS, HP>;
    const int r0 = t * C::TR, rows = min(C::TR, p.n - r0);
    mbar_expect_tx(bar, (unsigned)rows * C::ROWB);
    tma_load_1d(stg, p.Wout + (size_t)r0 * HP, rows * C::ROWB, bar, pol);
}
template <typename TS, int HP>
__device__ __forceinline__ void issue_vjp_tv(const EvalParams<TS>& p, int t, unsigned char* stg, uint64_t* bar,
                                             uint64_t keep) {
    using C = StreamCfg<TS, HP>;
    tma_load_1d(stg + C::TILEB, p.tv + (size_t)t * C::TR, tv_bytes<TS, HP>(p, t), bar, keep);
}

// Per-warp self-issued ring.  Warp w owns stages w + nw*j (j < spw); `ph` holds
// one parity bit per slot and persists across phases (warp-uniform).
struct WarpRing {
    unsigned char* ring;
    uint64_t* full;
    int nw, spw, stageb;
    uint32_t ph;
    __device__ int stage(int j) const { return (int)(threadIdx.x >> 5) + nw * j; }
    __device__ unsigned char* buf(int j) const { return ring + (size_t)stage(j) * stageb; }
    __device__ uint64_t* bar(int j) const { return full + stage(j); }
    __device__ void wait(int j) {
        mbar_wait(bar(j), (ph >> j) & 1u);
        ph ^= 1u << j;
    }
    // number of this warp's tiles in [t0, t1)
    __device__ int count(int t0, int t1) const {
        const int f = t0 + (int)(threadIdx.x >> 5);
        return f < t1 ? (t1 - f + nw - 1) / nw : 0;
    }
};

// Prefetch (lane 0): this warp's first min(spw, count) tiles of [t0, t1).
template <typename Issue>
__device__ __forceinline__ void ring_prefetch(const WarpRing& r, int t0, int t1, Issue issue) {
    if ((threadIdx.x & 31) != 0) return;
    const int n = min(r.spw, r.count(t0, t1));
    for (int j = 0; j < n; ++j) issue(t0 + (int)(threadIdx.x >> 5) + r.nw * j, r.buf(j), r.bar(j));
}

// Consume this warp's tiles of [t0, t1) in order (the first min(spw, count) already
// issued); a consumed slot is refilled with the tile spw ahead.
template <typename Issue, typename Body>
__device__ __forceinline__ void ring_run(WarpRing& r, int t0, int t1, Issue issue, Body body) {
    const int lane = threadIdx.x & 31;
    int i = 0;
    for (int t = t0 + (int)(threadIdx.x >> 5); t < t1; t += r.nw, ++i) {
        const int j = i % r.spw;
        r.wait(j);
        body(t, r.buf(j));
        __syncwarp();
        const int tn = t + r.nw * r.spw;
        if (lane == 0 && tn < t1) issue(tn, r.buf(j), r.bar(j));
    }
}

// Wait out prefetched-but-unconsumed tiles (before the CTA exits).
__device__ __forceinline__ void ring_drain(WarpRing& r, int t0, int t1) {
    const int n = min(r.spw, r.count(t0, t1));
    for (int j = 0; j < n; ++j) r.wait(j);
}

// Init the full barriers of an nst-stage ring (thread 0) + fence; caller syncs.
__device__ __forceinline__ void ring_init(uint64_t* full, int nst) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
        mbar_fence_init();
    }
}

// Multi-row reduction + epilogue of a forward tile from the per-lane row partials acc[TR]:
// recursive-halving multi-row reduction, lane (32 / TR) j runs the epilogue of row j.
template <typename TS, int HP>
__device__ __forceinline__ double fwd_epilogue(const EvalParams<TS>& p, const unsigned char* st, int t,
                                               double (&acc)[StreamCfg<TS, HP>::TR], int has_inertia, double inv_dt2,
                                               bool ident) {
    using C = StreamCfg<TS, HP>;
    const int lane = threadIdx.x & 31;
    const int rows = min(C::TR, p.n - t * C::TR);
    const double* ep = reinterpret_cast<const double*>(st + C::TILEB);
    // recursive-halving multi-row reduction: at offset o the lanes with bit o set keep
    // the upper half of their rows and receive the partner's copy of it, so TR rows
    // cost TR - 1 + log2(32 / TR) shuffles (not 5 TR).  Lane l ends up with the full
    // sum of row l / (32 / TR).
    static_assert(C::TR == 8 || C::TR == 16, "tile rows");
    constexpr int LPR = 32 / C::TR;
#pragma unroll
    for (int o = 16, n = C::TR; n > 1; o >>= 1) {
        n >>= 1;
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < n; ++k) {
            const double give = up ? acc[k] : acc[k + n];
            const double keep = up ? acc[k + n] : acc[k];
            acc[k] = keep + __shfl_xor_sync(0xffffffffu, give, o);
        }
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
    const double mine = acc[0];
    const int jr = lane / LPR;
    double e = 0.0;
    if (lane % LPR == 0 && jr < rows) {
        const int row = t * C::TR + jr;
        const double* e6 = ep + jr * 6;
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

// One warp computes every row of a forward tile: TR independent dot products,
// one multi-row reduction, lane (32 / TR) j runs the epilogue of row j.
template <typename TS, int HP>
__device__ __forceinline__ double fwd_tile(const EvalParams<TS>& p, const unsigned char* st, int t,
                                           const double (&y)[StreamCfg<TS, HP>::NCH][StreamCfg<TS, HP>::V4],
                                           int has_inertia, double inv_dt2, bool ident) {
    using C = StreamCfg<TS, HP>;
    const int lane = threadIdx.x & 31;
    const int rows = min(C::TR, p.n - t * C::TR);
    const TS* tile = reinterpret_cast<const TS*>(st);
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
    return fwd_epilogue<TS, HP>(p, st, t, acc, has_inertia, inv_dt2, ident);
}

// fp32-storage mode, reduced-cost tile math: the fp64 operand is split into fp32 hi + lo parts
// (y = hi + lo to ~2^-48), each lane sums its NCH x 4 products w hi + w lo of a row in fp32
// (fp32 weights times the split operand: the per-lane partial is exact to ~1e-7 relative, the
// level of the fp32 rounding of W itself) and the partials are promoted to fp64 for the
// cross-lane reduction and the epilogue.  Two FFMA per weight instead of an F2F conversion and
// an fp64 FMA -- the streaming warps' issue cost, not their bytes, bounds the fused sweep.
template <int HP>
__device__ __forceinline__ double fwd_tile_mixed(const EvalParams<float>& p, const unsigned char* st, int t,
                                                 const float (&yh)[StreamCfg<float, HP>::NCH][4],
                                                 const float (&yl)[StreamCfg<float, HP>::NCH][4], int has_inertia,
                                                 double inv_dt2, bool ident) {
    using C = StreamCfg<float, HP>;
    const int lane = threadIdx.x & 31;
    const int rows = min(C::TR, p.n - t * C::TR);
    const float* tile = reinterpret_cast<const float*>(st);
    double acc[C::TR];
#pragma unroll
    for (int j = 0; j < C::TR; ++j) {
        float sh = 0.f, sl = 0.f;
        if (j < rows) {
            const float* rowp = tile + (size_t)j * HP;
#pragma unroll
            for (int c = 0; c < C::NCH; ++c) {
                const float4 w = *reinterpret_cast<const float4*>(rowp + (c * 32 + lane) * 4);
                sh = fmaf(w.x, yh[c][0], sh);
                sl = fmaf(w.x, yl[c][0], sl);
                sh = fmaf(w.y, yh[c][1], sh);
                sl = fmaf(w.y, yl[c][1], sl);
                sh = fmaf(w.z, yh[c][2], sh);
                sl = fmaf(w.z, yl[c][2], sl);
                sh = fmaf(w.w, yh[c][3], sh);
                sl = fmaf(w.w, yl[c][3], sl);
            }
        }
        acc[j] = (double)sh + (double)sl;
    }
    return fwd_epilogue<float, HP>(p, st, t, acc, has_inertia, inv_dt2, ident);
}

// VJP counterpart: per tile, each lane's NCH x 4 column sums over the tile's TR rows in fp32
// (tv split into hi + lo), promoted to fp64 into the item accumulators.
template <int HP>
__device__ __forceinline__ void vjp_tile_mixed(const EvalParams<float>& p, const unsigned char* st, const double* tv,
                                               int t, double (&acc)[StreamCfg<float, HP>::NCH][4]) {
    using C = StreamCfg<float, HP>;
    const int lane = threadIdx.x & 31;
    const int rows = min(C::TR, p.n - t * C::TR);
    const float* tile = reinterpret_cast<const float*>(st);
    float sh[C::NCH][4], sl[C::NCH][4];
#pragma unroll
    for (int c = 0; c < C::NCH; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) sh[c][q] = sl[c][q] = 0.f;
#pragma unroll
    for (int j = 0; j < C::TR; ++j) {
        if (j < rows) {
            const double tval = tv[j];
            const float th = (float)tval, tl = (float)(tval - (double)th);
            const float* rowp = tile + (size_t)j * HP;
#pragma unroll
            for (int c = 0; c < C::NCH; ++c) {
                const float4 w = *reinterpret_cast<const float4*>(rowp + (c * 32 + lane) * 4);
                sh[c][0] = fmaf(w.x, th, sh[c][0]);
                sl[c][0] = fmaf(w.x, tl, sl[c][0]);
                sh[c][1] = fmaf(w.y, th, sh[c][1]);
                sl[c][1] = fmaf(w.y, tl, sl[c][1]);
                sh[c][2] = fmaf(w.z, th, sh[c][2]);
                sl[c][2] = fmaf(w.z, tl, sl[c][2]);
                sh[c][3] = fmaf(w.w, th, sh[c][3]);
                sl[c][3] = fmaf(w.w, tl, sl[c][3]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < C::NCH; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[c][q] += (double)sh[c][q] + (double)sl[c][q];
}

// One warp accumulates a VJP tile into its per-lane column accumulators.
template <typename TS, int HP>
__device__ __forceinline__ void vjp_tile(const EvalParams<TS>& p, const unsigned char* st, const double* tv, int t,
                                         double (&acc)[StreamCfg<TS, HP>::NCH][StreamCfg<TS, HP>::V4]) {
    using C = StreamCfg<TS, HP>;
    const int lane = threadIdx.x & 31;
    const int rows = min(C::TR, p.n - t * C::TR);
    const TS* tile = reinterpret_cast<const TS*>(st);
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
    __shared__ double red[32];
    const int lane = threadIdx.x & 31;
    constexpr int NW = kStreamThreads / 32;
    WarpRing r{ssm + 512, reinterpret_cast<uint64_t*>(ssm), NW, kStreamSpw, C::STAGEB, 0u};
    ring_init(r.full, NW * kStreamSpw);
    __syncthreads();
    const int ntiles = (p.n + C::TR - 1) / C::TR;
    const int t0 = (int)(((long long)ntiles * blockIdx.x) / gridDim.x);
    const int t1 = (int)(((long long)ntiles * (blockIdx.x + 1)) / gridDim.x);
    const uint64_t pol = l2_policy(p.w_resident), keep = l2_policy(1);
    // the range's last w_keep_tiles W tiles stay in L2 (evict_last) across the element pass: the VJP
    // re-reads them there (with evict_first, which demotes them) instead of from HBM
    const int tkeep = t1 - p.w_keep_tiles;
    auto issue = [&](int t, unsigned char* b, uint64_t* bar) {
        issue_fwd<TS, HP>(p, t, b, bar, t >= tkeep ? keep : pol, keep);
    };
    ring_prefetch(r, t0, t1, issue);  // W tiles and row records do not depend on the previous kernel
    if (p.l2_pf_tiles > 0) {  // while the control kernel runs (programmatic launch): next tiles into L2
        const int a = min(t1, t0 + NW * kStreamSpw), b = min(t1, a + p.l2_pf_tiles);
        if (b > a) prefetch_l2_range(p.Wout + (size_t)a * C::TR * HP, (size_t)(b - a) * C::TILEB, 8192);
    }
    griddep_wait();
    griddep_launch();  // after the wait: dependents never start ahead of this kernel's own inputs
    const double inv_dt2 = p.st->inv_dt2;
    const int has_inertia = p.st->has_inertia;
    const bool ident = p.out_act == kIdentity;
    double y[C::NCH][C::V4];
#pragma unroll
    for (int c = 0; c < C::NCH; ++c)
#pragma unroll
        for (int q = 0; q < C::V4; ++q) y[c][q] = p.y_last[(c * 32 + lane) * C::V4 + q];
    double eacc = 0.0;
    ring_run(r, t0, t1, issue, [&](int t, const unsigned char* b) {
        eacc += fwd_tile<TS, HP>(p, b, t, y, has_inertia, inv_dt2, ident);  // HBM-bound: fp64 math is free
    });
    const double tot = block_sum(eacc, red);
    if (threadIdx.x == 0) p.e_part_out[blockIdx.x] = 0.5 * inv_dt2 * tot;
}


// tv for the rows [R0, R1) of one CTA into shared memory, one thread per free
// vertex: its CSR segment (ascending tet id) is summed in order from one batch of
// up to 24 independent 256-bit loads (one request per 32-byte force entry).
// Vertices straddling the range edge are computed by both neighbours, identically.
// ---------------------------------------------------------------- K3b: vertex gather (+ inertia)
// tv_i = s_i phi'(a_i) (sum of the per-tet forces on DOF i in ascending tet id + inertia
// residual) -- the full-space gradient times the output scaling.
__device__ __forceinline__ double4 ld_cg_d4(const double* p) {
    double4 v;
    asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p));
    return v;
}
// One free vertex f: its CSR segment (ascending tet id) summed in order from one batch
// of up to 24 independent 256-bit loads; rows 3f..3f+2 inside [R0, R1) are written to
// dst[row - R0] as tv = s (g + inertia residual).
// The row scale s comes from the compact sout array (streaming kernels: eprow is no longer in
// L2) or from the row records' column 1 (the persistent kernel, where they are L2-hot).
template <typename TS>
__device__ __forceinline__ void gather_vertex1(const EvalParams<TS>& p, int f, int R0, int R1, double* dst,
                                               int has_inertia, bool ident, bool scale_compact = true) {
    const int b = __ldg(p.csr_ptr + f), e = __ldg(p.csr_ptr + f + 1);
    double rin[3] = {0.0, 0.0, 0.0}, sc[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int row = 3 * f + c;
        if (has_inertia) rin[c] = __ldcg(p.rin + row);
        sc[c] = ident ? (scale_compact ? __ldg(p.sout + row) : __ldg(p.eprow + 6 * (size_t)row + 1))
                      : __ldcg(p.dsout + row);
    }
    double gx = 0.0, gy = 0.0, gz = 0.0;
    if constexpr (std::is_same<TS, float>::value) {  // fp32-storage mode: 16-byte float entries
        const float4* F4 = reinterpret_cast<const float4*>(p.forces);
        for (int k0 = b; k0 < e; k0 += 24) {
            float4 v[24];
#pragma unroll
            for (int u = 0; u < 24; ++u) v[u] = k0 + u < e ? __ldcg(F4 + k0 + u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 24; ++u) {
                gx += (double)v[u].x;
                gy += (double)v[u].y;
                gz += (double)v[u].z;
            }
        }
    } else {
        for (int k0 = b; k0 < e; k0 += 24) {
            double4 v[24];
#pragma unroll
            for (int u = 0; u < 24; ++u)
                v[u] = k0 + u < e ? ld_cg_d4(p.forces + 4 * (size_t)(k0 + u)) : make_double4(0.0, 0.0, 0.0, 0.0);
#pragma unroll
            for (int u = 0; u < 24; ++u) {
                gx += v[u].x;
                gy += v[u].y;
                gz += v[u].z;
            }
        }
    }
    const double g[3] = {gx, gy, gz};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int row = 3 * f + c;
        if (row >= R0 && row < R1) dst[row - R0] = (g[c] + rin[c]) * sc[c];
    }
}

// tv for the rows [R0, R1) of one CTA (all threads call it); vertices straddling the
// range edge are computed by both neighbours, identically.
template <typename TS>
__device__ __forceinline__ void gather_rows_smem(const EvalParams<TS>& p, int R0, int R1, double* tv_s,
                                                 int has_inertia, bool ident, bool scale_compact = true) {
    const int f0 = R0 / 3, nf = R1 > R0 ? (R1 - 1) / 3 - f0 + 1 : 0;
    for (int k = threadIdx.x; k < nf; k += blockDim.x)
        gather_vertex1(p, f0 + k, R0, R1, tv_s, has_inertia, ident, scale_compact);
}

template <typename TS>
__global__ void __launch_bounds__(256) gather_kernel(const EvalParams<TS> p) {
    const DevState* st = p.st;
    if (!st->need_grad) return;
    const bool ident = p.out_act == kIdentity;
    const int has_inertia = st->has_inertia;
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < p.n_free; f += gridDim.x * blockDim.x)
        gather_vertex1(p, f, 0, p.n, p.tv, has_inertia, ident);
}

// ---------------------------------------------------------------- K4 (TMA): VJP partials
template <typename TS, int HP>
__global__ void __launch_bounds__(kStreamThreads) vjp_tma_kernel(const EvalParams<TS> p) {
    using C = StreamCfg<TS, HP>;
    extern __shared__ __align__(128) unsigned char ssm[];
    constexpr int NW = kStreamThreads / 32;
    __shared__ int am_grp_last;
    DevState* st = p.st;
    if (!st->need_grad) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    WarpRing r{ssm + 512, reinterpret_cast<uint64_t*>(ssm), NW, kStreamSpw, C::STAGEB, 0u};
    double* wred = reinterpret_cast<double*>(ssm + 512 + (size_t)NW * kStreamSpw * C::STAGEB);  // NW x HP
    ring_init(r.full, NW * kStreamSpw);
    __syncthreads();
    const int ntiles = (p.n + C::TR - 1) / C::TR;
    const int t0 = (int)(((long long)ntiles * blockIdx.x) / gridDim.x);
    const int t1 = (int)(((long long)ntiles * (blockIdx.x + 1)) / gridDim.x);
    const uint64_t pol = l2_policy(p.w_resident), keep = l2_policy(1);
    auto issue = [&](int t, unsigned char* b, uint64_t* bar) {
        issue_vjp_w<TS, HP>(p, t, b, bar, pol);
        issue_vjp_tv<TS, HP>(p, t, b, bar, keep);
    };
    ring_prefetch(r, t0, t1, issue);
    double acc[C::NCH][C::V4];
#pragma unroll
    for (int c = 0; c < C::NCH; ++c)
#pragma unroll
        for (int q = 0; q < C::V4; ++q) acc[c][q] = 0.0;
    ring_run(r, t0, t1, issue, [&](int t, const unsigned char* b) {
        vjp_tile<TS, HP>(p, b, reinterpret_cast<const double*>(b + C::TILEB), t, acc);
    });
#pragma unroll
    for (int c = 0; c < C::NCH; ++c)
#pragma unroll
        for (int q = 0; q < C::V4; ++q) wred[warp * HP + (c * 32 + lane) * C::V4 + q] = acc[c][q];
    __syncthreads();
    for (int j = tid; j < HP; j += blockDim.x) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += wred[w * HP + j];
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

// tv of the TR rows of tile t, gathered by one warp: the tile's (<= TR/3 + 2) free vertices get
// LG lanes each, which sum strided slices of the vertex's CSR segment; an xor butterfly within
// the lane group (bit-identical on every lane of the group) completes each vertex's force, and
// lane j < TR forms row t TR + j.  Issued right before the tile's W rows are waited for, so its
// L2 latency hides behind the W stream; vertices straddling two tiles are gathered by both.
template <typename TS, int TR>
__device__ __forceinline__ void warp_gather_tile(const EvalParams<TS>& p, int t, double* tvw, int has_inertia,
                                                 bool ident) {
    constexpr int LG = TR == 8 ? 8 : 4;  // lanes per vertex (TR 8: <= 4 vertices; TR 16: <= 7)
    const int lane = threadIdx.x & 31;
    const int R0 = t * TR, R1 = min(R0 + TR, p.n);
    const int f0 = R0 / 3, nvtx = (R1 - 1) / 3 - f0 + 1;
    const int vi = lane / LG, sub = lane % LG;
    double g[3] = {0.0, 0.0, 0.0};
    if (vi < nvtx) {
        const int f = f0 + vi;
        const int b = __ldg(p.csr_ptr + f), e = __ldg(p.csr_ptr + f + 1);
        if constexpr (std::is_same<TS, float>::value) {
            const float4* F4 = reinterpret_cast<const float4*>(p.forces);
            for (int k = b + sub; k < e; k += LG) {
                const float4 v = __ldcg(F4 + k);
                g[0] += (double)v.x;
                g[1] += (double)v.y;
                g[2] += (double)v.z;
            }
        } else {
            for (int k = b + sub; k < e; k += LG) {
                const double4 v = ld_cg_d4(p.forces + 4 * (size_t)k);
                g[0] += v.x;
                g[1] += v.y;
                g[2] += v.z;
            }
        }
    }
#pragma unroll
    for (int o = 1; o < LG; o <<= 1)
#pragma unroll
        for (int c = 0; c < 3; ++c) g[c] += __shfl_xor_sync(0xffffffffu, g[c], o);
    const int row = R0 + (lane < TR ? lane : 0);
    const int src = (row / 3 - f0) * LG, comp = row % 3;
    const double gx = __shfl_sync(0xffffffffu, g[0], src);
    const double gy = __shfl_sync(0xffffffffu, g[1], src);
    const double gz = __shfl_sync(0xffffffffu, g[2], src);
    if (lane < TR && row < R1) {
        const double gc = comp == 0 ? gx : (comp == 1 ? gy : gz);
        const double rin = has_inertia ? __ldcg(p.rin + row) : 0.0;
        const double sc = ident ? __ldg(p.sout + row) : __ldcg(p.dsout + row);
        tvw[lane] = (gc + rin) * sc;
    }
    __syncwarp();
}

// vjp_gather_tma_kernel with the gather done per warp and per tile (warp_gather_tile) instead of
// a CTA-wide prologue: no tv scratch, and the gather latency overlaps the stream.
template <typename TS, int HP>
__global__ void __launch_bounds__(kStreamThreads) vjp_wgather_tma_kernel(const EvalParams<TS> p) {
    using C = StreamCfg<TS, HP>;
    extern __shared__ __align__(128) unsigned char ssm[];
    constexpr int NW = kStreamThreads / 32;
    __shared__ int am_grp_last;
    __shared__ double tvw_all[NW][C::TR];
    DevState* st = p.st;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    WarpRing r{ssm + 512, reinterpret_cast<uint64_t*>(ssm), NW, kStreamSpw, C::TILEB, 0u};
    double* wred = reinterpret_cast<double*>(ssm + 512);  // NW x HP, in the drained ring
    static_assert(NW * HP * 8 <= NW * kStreamSpw * C::TILEB, "column sums fit in the ring");
    double* tvw = tvw_all[warp];
    ring_init(r.full, NW * kStreamSpw);
    __syncthreads();
    const int ntiles = (p.n + C::TR - 1) / C::TR;
    const int t0 = (int)(((long long)ntiles * blockIdx.x) / gridDim.x);
    const int t1 = (int)(((long long)ntiles * (blockIdx.x + 1)) / gridDim.x);
    const uint64_t pol = l2_policy(p.w_resident);
    auto issue = [&](int t, unsigned char* b, uint64_t* bar) { issue_w_only<TS, HP>(p, t, b, bar, pol); };
    ring_prefetch(r, t0, t1, issue);  // W tiles do not depend on the element pass
    griddep_wait();
    griddep_launch();
    if (!st->need_grad) {  // value only: let the prefetched tiles land before the CTA exits
        ring_drain(r, t0, t1);
        return;
    }
    const int has_inertia = st->has_inertia;
    const bool ident = p.out_act == kIdentity;
    double acc[C::NCH][C::V4];
#pragma unroll
    for (int c = 0; c < C::NCH; ++c)
#pragma unroll
        for (int q = 0; q < C::V4; ++q) acc[c][q] = 0.0;
    int i = 0;
    for (int t = t0 + warp; t < t1; t += NW, ++i) {
        warp_gather_tile<TS, C::TR>(p, t, tvw, has_inertia, ident);
        const int j = i % kStreamSpw;
        r.wait(j);
        vjp_tile<TS, HP>(p, r.buf(j), tvw, t, acc);
        __syncwarp();
        const int tn = t + NW * kStreamSpw;
        if (lane == 0 && tn < t1) issue(tn, r.buf(j), r.bar(j));
    }
    __syncthreads();  // every warp is done with its stages: wred may overwrite the ring
#pragma unroll
    for (int c = 0; c < C::NCH; ++c)
#pragma unroll
        for (int q = 0; q < C::V4; ++q) wred[warp * HP + (c * 32 + lane) * C::V4 + q] = acc[c][q];
    __syncthreads();
    for (int jj = tid; jj < HP; jj += blockDim.x) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) sum += wred[w * HP + jj];
        p.ybar_part[(size_t)blockIdx.x * HP + jj] = sum;
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
    for (int jj = tid; jj < HP; jj += blockDim.x) {
        double sum = 0.0;
        for (int b = g0; b < g1; ++b) sum += __ldcg(p.ybar_part + (size_t)b * HP + jj);
        p.ybar_grp[(size_t)grp * HP + jj] = sum;
    }
    if (tid == 0) p.grp_cnt[grp] = 0;
}

// ---------------------------------------------------------------- K3b + K4 fused: gather + VJP
// vjp_tma_kernel with the vertex gather folded in: each CTA gathers tv for its own rows
// into shared memory (gather_rows_smem, as the persistent kernel does) while its first W
// tiles are already in flight, then streams W only.  Saves the gather kernel's launch and
// its tv round trip through global memory.
template <typename TS, int HP>
__global__ void __launch_bounds__(kStreamThreads) vjp_gather_tma_kernel(const EvalParams<TS> p) {
    using C = StreamCfg<TS, HP>;
    extern __shared__ __align__(128) unsigned char ssm[];
    constexpr int NW = kStreamThreads / 32;
    __shared__ int am_grp_last;
    DevState* st = p.st;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // stages hold W rows only (tv is in shared memory); the per-warp column sums reuse the ring
    // once it is drained, so three CTAs fit per SM
    WarpRing r{ssm + 512, reinterpret_cast<uint64_t*>(ssm), NW, kStreamSpw, C::TILEB, 0u};
    double* wred = reinterpret_cast<double*>(ssm + 512);                                           // NW x HP
    double* tv_s = reinterpret_cast<double*>(ssm + 512 + (size_t)NW * kStreamSpw * C::TILEB);     // own rows
    static_assert(NW * HP * 8 <= NW * kStreamSpw * C::TILEB, "column sums fit in the ring");
    ring_init(r.full, NW * kStreamSpw);
    __syncthreads();
    const int ntiles = (p.n + C::TR - 1) / C::TR;
    const int t0 = (int)(((long long)ntiles * blockIdx.x) / gridDim.x);
    const int t1 = (int)(((long long)ntiles * (blockIdx.x + 1)) / gridDim.x);
    const uint64_t pol = l2_policy(p.w_resident);
    auto issue = [&](int t, unsigned char* b, uint64_t* bar) { issue_w_only<TS, HP>(p, t, b, bar, pol); };
    ring_prefetch(r, t0, t1, issue);  // W tiles do not depend on the element pass
    griddep_wait();
    griddep_launch();
    if (!st->need_grad) {  // value only: let the prefetched tiles land before the CTA exits
        ring_drain(r, t0, t1);
        return;
    }
    const int R0 = t0 * C::TR, R1 = min(t1 * C::TR, p.n);
    gather_rows_smem(p, R0, R1, tv_s, st->has_inertia, p.out_act == kIdentity);
    __syncthreads();
    double acc[C::NCH][C::V4];
#pragma unroll
    for (int c = 0; c < C::NCH; ++c)
#pragma unroll
        for (int q = 0; q < C::V4; ++q) acc[c][q] = 0.0;
    ring_run(r, t0, t1, issue, [&](int t, const unsigned char* b) {
        vjp_tile<TS, HP>(p, b, tv_s + (t * C::TR - R0), t, acc);  // fp64 math: the mixed form measured no faster here
    });
    __syncthreads();  // every warp is done with its stages: wred may overwrite the ring
#pragma unroll
    for (int c = 0; c < C::NCH; ++c)
#pragma unroll
        for (int q = 0; q < C::V4; ++q) wred[warp * HP + (c * 32 + lane) * C::V4 + q] = acc[c][q];
    __syncthreads();
    for (int j = tid; j < HP; j += blockDim.x) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += wred[w * HP + j];
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
