// Persistent "solve" kernel: one cooperative launch (grid of thread-block
// clusters) runs a whole objective evaluation, L-BFGS solve or implicit-Euler
// step, with grid barriers between phases instead of kernel boundaries.
//
//   cluster 0 (the control cluster) keeps the hidden-layer weight slices and the
//   solver state in shared memory for the lifetime of the launch;
//   every CTA owns a TMA ring (producer warp 8) used by the two W_out streams;
//   the Armijo / need-gradient decision is evaluated redundantly by every CTA
//   from the same partials (identical fixed-order sums), so it costs no barrier.
//
// Per evaluation:  out_fwd | grid | elem | grid | [gather | grid | vjp | grid] | ctrl | grid
#pragma once

#include "lsb_stream.cuh"

namespace lsb {

#ifndef LSB_SOLVE_THREADS
#define LSB_SOLVE_THREADS 288
#endif
constexpr int kSolveThreads = LSB_SOLVE_THREADS;  // 9 warps: all stream (self-issued rings) and all compute
constexpr int kSolveMaxStages = 36;
constexpr int kSolveMaxGrid = 160;  // control-cluster partial sums: 5 x 32 lanes
#ifndef LSB_SOLVE_ELEM_F32
#define LSB_SOLVE_ELEM_F32 1
#endif
constexpr int kSolveBarBytes = 512;  // full barriers (kSolveMaxStages x 8 B, padded)

// Launch-wide scalars the non-control CTAs need (written by the control CTA).
struct SolveShared {
    int mode, phase, want_grad, done;
    double f, armijo_slope;  // f + 1e-4 alpha gtd threshold pieces
    int status;
    unsigned grid_bar;       // grid barrier word (generation = top bit; never reset)
    unsigned staged_seq;     // = SolveParams::seq once the control cluster's staging landed
};

// Grid-wide barrier of the persistent kernel (all CTAs co-resident: the grid is
// sized from cudaOccupancyMaxActiveClusters).  CTA 0 adds 2^31 - (G - 1), every
// other CTA adds 1, so the top bit flips exactly when all G have arrived; waiters
// spin until their generation bit changes.  gpu-scope fences on both sides order
// every thread's prior writes (via bar.sync) before every later read.
__device__ __forceinline__ void grid_barrier(unsigned* word, int cta, int G, bool fences = true) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned inc = cta == 0 ? (0x80000000u - (unsigned)(G - 1)) : 1u;
        if (fences) __threadfence();
        unsigned old, cur;
        asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(word), "r"(inc) : "memory");
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(word) : "memory");
        } while (((old ^ cur) & 0x80000000u) == 0);
        if (fences) __threadfence();
    }
    __syncthreads();
}

// Split-phase form: arrive (returns the pre-add word, thread 0) ... wait.
__device__ __forceinline__ unsigned grid_arrive(unsigned* word, int cta, int G, bool fences = true) {
    __syncthreads();
    unsigned old = 0;
    if (threadIdx.x == 0) {
        const unsigned inc = cta == 0 ? (0x80000000u - (unsigned)(G - 1)) : 1u;
        if (fences) __threadfence();
        asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(word), "r"(inc) : "memory");
    }
    return old;
}
__device__ __forceinline__ void grid_wait(unsigned* word, unsigned old, bool fences = true) {
    if (threadIdx.x == 0) {
        unsigned cur;
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(word) : "memory");
        } while (((old ^ cur) & 0x80000000u) == 0);
        if (fences) __threadfence();
    }
    __syncthreads();
}

// First W_out tile of CTA k when the CS control CTAs take weight wc and the others 1.
__host__ __device__ __forceinline__ int solve_tile_start(int ntiles, int k, int G, int CS, float wc) {
    const double W = k <= CS ? k * (double)wc : CS * (double)wc + (k - CS);
    const double Wt = CS * (double)wc + (G - CS);
    return k >= G ? ntiles : (int)((double)ntiles * W / Wt);
}

struct SolveParams {
    int task;         // 0 = eval (ctrl start + one evaluation), 1 = minimize, 2 = step
    int quasi;        // step: quasi-static
    int want_grad;    // eval: gradient wanted
    int spw;          // ring stages per warp, non-control CTAs
    int spw_ctrl;     // ring stages per warp, control CTAs (their control area follows the ring)
    int tv_off;       // byte offset of the tv/partials scratch (non-control CTAs)
    int tv_off_ctrl;  // ditto, control CTAs (after their control area)
    int tv_cap;       // its capacity in doubles (>= rows per CTA and >= hp)
    int tv_global;    // 1: tv lives in global memory and streams with the VJP tiles (large n)
    int wsl_words;    // control-area weight slices, in 8-byte words (stored as TS)
    unsigned seq;     // launch sequence number (host-incremented)
    // developer A/B switches (LSB_SOLVE_EXP; 0 = the production path).  Bits 1 / 4 skip the tile
    // math / the tv gather (timing only, results invalid); 2: VJP prefetch after the gather;
    // 8: no cold-start L2 prefetch; 32: cycle stamps; 64: generic control cluster; 128: no
    // deferral of the non-control CTAs' first ring prefetch; 2048: fast path with cluster
    // barriers instead of st.async; 4096: L2 prefetch without waiting for the control staging;
    // 8192: 1 MB prefetch pieces; 16384: fence.sc around the grid barrier's atomic / poll
    int exp;
    float ctrl_tile_w;  // control CTAs' share of the W_out tiles relative to the others
    float pf_frac;      // fraction of W_out prefetched into L2 at a cold start
    // dynamics
    const double* u_state;
    const double* v_state;
    const double* a_ext;
    double* z_state;
    double* u_state_w;
    double* v_state_w;
    const char* vpinned;
    const double* pin_disp;
    SolveShared* sh;
    long long* launch_acc;
    unsigned long long* trace;  // optional phase timestamps (CTA 0), nullptr = off
    // direct evaluation (task 0 through lsb_eval): z by value, result {E, status, grad[r]}
    // written by CTA 0 into host-mapped memory (nullptr = off)
    double* out_map;
    int z_in;
    double z[kMaxLatent];
};


// ---- control-cluster helpers (weights resident in smem) -------------------------------------------
// The hidden MLP is row-partitioned over the CS CTAs of cluster 0 (part_lo).  Both
// directions are push-based: a CTA stores what other CTAs need straight into their
// shared memory (DSMEM), then one cluster barrier per layer publishes it, so every
// operand read is local.
constexpr int kCtrlRecv = 1024;  // CS x (rows per CTA) receive slots (<= 16 x 64)
struct CtrlSmem {
    double* wsl;      // staged W row slices
    double* xin0;     // layer inputs (kMaxHidden each), double-buffered across layers
    double* xin1;
    double* rbuf0;    // backward receive buffers [src CTA][own row] (kCtrlRecv each)
    double* rbuf1;
    // selects instead of runtime-indexed member arrays: keeps the struct in registers
    __device__ __forceinline__ double* xin(int k) const { return k ? xin1 : xin0; }
    __device__ __forceinline__ double* rbuf(int k) const { return k ? rbuf1 : rbuf0; }
    double* tmp;      // ybar reduction scratch (kSolveThreads)
    double* bsl;      // kMaxLayers * 64
    double* asl;      // kMaxLayers * 64
    DevState* sst;
    uint64_t* wbar;  // kMaxLayers + 1 staging barriers (static smem)
    int* woff;       // kMaxLayers weight-slice offsets (static smem)
};
constexpr size_t ctrl_fixed_words() {
    return 2 * kMaxHidden + 2 * kCtrlRecv + kSolveThreads + 2 * kMaxLayers * 64 + sizeof(DevState) / sizeof(double) + 8;
}

// owner CTA of row j under part_lo(R, CS, .) (32-bit arithmetic; R <= kMaxHidden)
template <int CS>
__device__ __forceinline__ int part_owner(int j, int R) {
    int q = (j * CS) / R;
    if (q < CS - 1 && (R * (q + 1)) / CS <= j) ++q;
    if ((R * q) / CS > j) --q;
    return q;
}

// Stage this CTA's weight/bias row slices (+ the solver state on CTA 0): 16-byte
// aligned pieces as 1-D bulk copies completing on one mbarrier per layer (wbar[l])
// and one for the state (wbar[kMaxLayers]), so layer 0 can start while the rest
// is in flight; misaligned pieces fall back to cp.async (waited here).  The copies are
// issued in parallel by lane 0 of different warps (warp 0: the state, warp 1 + l: layer
// l), since one thread's issue loop costs ~1 us per layer.  Users wait with
// ctrl_wait_layer / ctrl_wait_state (parity 0: free once complete).
__device__ __forceinline__ bool bulk_ok(const void* dst, const void* src, size_t bytes) {
    return ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | bytes) & 15u) == 0;
}
template <typename TS, int CS>
__device__ __forceinline__ void ctrl_stage(const EvalParams<TS>& p, CtrlSmem& cs, int c, bool with_state, uint64_t* wbar) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    if (tid == 0) {
        for (int l = 0; l <= kMaxLayers; ++l) mbar_init(&wbar[l], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const uint64_t keep = l2_policy(1);
    bool async_used = false;
    if (warp == 0 && with_state && c == 0) {
        griddep_wait();  // the solver state is written by the previous kernel
        double* sd = reinterpret_cast<double*>(cs.sst);
        const double* ss = reinterpret_cast<const double*>(p.st);
        const bool s_bulk = bulk_ok(sd, ss, sizeof(DevState));
        if (!s_bulk) {
            for (int k = lane; k < (int)(sizeof(DevState) / sizeof(double)); k += 32) cp_async8(sd + k, ss + k);
            async_used = true;
        }
        if (lane == 0) {
            if (s_bulk) tma_load_1d(sd, ss, (unsigned)sizeof(DevState), &wbar[kMaxLayers], keep);
            mbar_expect_tx(&wbar[kMaxLayers], s_bulk ? (unsigned)sizeof(DevState) : 0u);
        }
    }
    TS* wsl = reinterpret_cast<TS*>(cs.wsl);
    for (int l = warp - 1; l >= 0 && l < p.nhid; l += nw - 1) {
        int off = 0;
        for (int k = 0; k < l; ++k) {
            const int Rk = p.hrows[k];
            off += ((part_lo(Rk, CS, c + 1) - part_lo(Rk, CS, c)) * p.hcols[k] + 3) & ~3;
        }
        const int R = p.hrows[l], C = p.hcols[l];
        const int i0 = part_lo(R, CS, c), i1 = part_lo(R, CS, c + 1);
        if (lane == 0) cs.woff[l] = off;
        TS* wd = wsl + off;
        const TS* ws = p.Wh_s + p.hoff[l] + (size_t)i0 * C;
        const size_t wb = (size_t)(i1 - i0) * C * sizeof(TS);
        double* bd = cs.bsl + l * 64;
        const double* bs = p.bh + p.boff[l] + i0;
        const size_t bb = (size_t)(i1 - i0) * 8;
        const bool w_bulk = bulk_ok(wd, ws, wb), b_bulk = bulk_ok(bd, bs, bb);
        if (!w_bulk) {
            for (int k = lane; k < (i1 - i0) * C; k += 32) wd[k] = ws[k];
            async_used = true;  // plain copies: published by the barrier below
        }
        if (!b_bulk) {
            for (int k = lane; k < i1 - i0; k += 32) cp_async8(bd + k, bs + k);
            async_used = true;
        }
        if (lane == 0) {
            unsigned tx = 0;
            if (w_bulk && wb) {
                tma_load_1d(wd, ws, (unsigned)wb, &wbar[l], keep);
                tx += (unsigned)wb;
            }
            if (b_bulk && bb) {
                tma_load_1d(bd, bs, (unsigned)bb, &wbar[l], keep);
                tx += (unsigned)bb;
            }
            mbar_expect_tx(&wbar[l], tx);  // arrive + expect: completes when the bytes land
        }
    }
    if (__syncthreads_or(async_used)) {
        cp_async_wait_all();
        __syncthreads();
    }
    __syncthreads();  // woff
}
__device__ __forceinline__ void ctrl_wait_layer(uint64_t* wbar, int l) { mbar_wait(&wbar[l], 0); }
__device__ __forceinline__ void ctrl_wait_state(uint64_t* wbar) { mbar_wait(&wbar[kMaxLayers], 0); }

// Backward through the hidden layers.  ybar of the last hidden layer is the
// fixed-order sum of the per-CTA partials (G x hp); each CTA reduces its own
// rows.  Layer l: partial p_c[j] = sum_{own i} W[i][j] gy[i] is pushed to the owner
// of j (layer l-1 rows; CTA 0 for l = 0), which sums the CS partials in CTA order.
// Result -> sst->gz (CTA 0).  Ends with __syncthreads.
template <typename TS, int CS, typename Stamp>
__device__ __forceinline__ void ctrl_backward(const EvalParams<TS>& p, CtrlSmem& cs, cg::cluster_group& cluster, int c, int G,
                              const double* ypart, Stamp& stamp) {
    const int tid = threadIdx.x, nt = blockDim.x;
    if (p.nhid == 0) {
        if (c == 0)
            for (int j = tid; j < p.r; j += nt) {
                double s = 0.0;
                for (int b = 0; b < G; ++b) s += __ldcg(ypart + (size_t)b * p.hp + j);
                cs.sst->gz[j] = s;
            }
        __syncthreads();
        return;
    }
    double gy[2];  // this thread's own-row gradients (rows tid, tid + nt), layer being processed
    {
        const int Rl = p.hrows[p.nhid - 1];
        const int j0 = part_lo(Rl, CS, c), ncol = part_lo(Rl, CS, c + 1) - j0;
        const int per = max(1, nt / max(ncol, 1));  // threads per column
        const int col = tid % max(ncol, 1), q = tid / max(ncol, 1);
        if (q < per && col < ncol) {
            double s = 0.0;
            for (int b0 = q; b0 < G; b0 += 8 * per) {
                double v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int b = b0 + k * per;
                    v[k] = b < G ? __ldcg(ypart + (size_t)b * p.hp + j0 + col) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) s += v[k];
            }
            cs.tmp[q * ncol + col] = s;
        }
        __syncthreads();
        for (int k = 0; k < 2; ++k) {
            const int i = tid + k * nt;
            double s = 0.0;
            if (i < ncol)
                for (int qq = 0; qq < per; ++qq) s += cs.tmp[qq * ncol + i];
            gy[k] = s;
        }
        __syncthreads();  // tmp is reused below
    }
    stamp(-400);
    for (int l = p.nhid - 1; l >= 0; --l) {
        const int R = p.hrows[l], C = p.hcols[l];
        const int i0 = part_lo(R, CS, c), nrow = part_lo(R, CS, c + 1) - i0;
        stamp(-(410 + l * 10 + 0));
        double* gys = cs.tmp;  // own-row gradient times act' (nrow <= 64)
        for (int k = 0; k < 2; ++k) {
            const int i = tid + k * nt;
            if (i < nrow) gys[i] = gy[k] * act_eval(p.hact[l], cs.asl[l * 64 + i], 1);
        }
        __syncthreads();
        stamp(-(410 + l * 10 + 1));
        const TS* Ws = reinterpret_cast<const TS*>(cs.wsl) + cs.woff[l];
        ctrl_wait_layer(cs.wbar, l);
        double* rb = cs.rbuf(l & 1);
        const int Rp = l > 0 ? p.hrows[l - 1] : C;
        for (int j = tid; j < C; j += nt) {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int i = 0;
            for (; i + 4 <= nrow; i += 4) {
                s0 = fma((double)Ws[i * C + j], gys[i], s0);
                s1 = fma((double)Ws[(i + 1) * C + j], gys[i + 1], s1);
                s2 = fma((double)Ws[(i + 2) * C + j], gys[i + 2], s2);
                s3 = fma((double)Ws[(i + 3) * C + j], gys[i + 3], s3);
            }
            for (; i < nrow; ++i) s0 = fma((double)Ws[i * C + j], gys[i], s0);
            const double s = (s0 + s1) + (s2 + s3);
            const int o = l > 0 ? part_owner<CS>(j, Rp) : 0;
            const int jl = l > 0 ? j - part_lo(Rp, CS, o) : j;
            dsmem_st_f64(dsmem_addr(rb + c * 64 + jl, o), s);
        }
        stamp(-(410 + l * 10 + 2));
        cluster.sync();
        stamp(-(410 + l * 10 + 3));
        // own rows of layer l-1 (or z for l = 0 on CTA 0): fixed CTA-order sum
        const int nown = l > 0 ? part_lo(Rp, CS, c + 1) - part_lo(Rp, CS, c) : (c == 0 ? C : 0);
        for (int k = 0; k < 2; ++k) {
            const int i = tid + k * nt;
            double s = 0.0;
            if (i < nown) {
#pragma unroll
                for (int q = 0; q < CS; ++q) s += rb[q * 64 + i];
            }
            gy[k] = s;
            if (l == 0 && i < nown) cs.sst->gz[i] = s;
        }
    }
    __syncthreads();
}

// Forward through the hidden layers at sst->zt (CTA 0); the owner of each output
// row pushes it into every CTA's next-layer input buffer.  y_last -> p.y_last.
template <typename TS, int CS, typename Stamp>
__device__ __forceinline__ void ctrl_forward(const EvalParams<TS>& p, CtrlSmem& cs, cg::cluster_group& cluster, int c, Stamp& stamp) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nw = blockDim.x >> 5;
    {
        const double* zsrc = cluster.map_shared_rank(cs.sst->zt, 0);
        for (int j = tid; j < p.r; j += blockDim.x) cs.xin(0)[j] = zsrc[j];
    }
    __syncthreads();
    for (int l = 0; l < p.nhid; ++l) {
        const int R = p.hrows[l], C = p.hcols[l];
        const int i0 = part_lo(R, CS, c), nrow = part_lo(R, CS, c + 1) - i0;
        const double* x = cs.xin(l & 1);
        double* xn = cs.xin((l & 1) ^ 1);
        const TS* Ws = reinterpret_cast<const TS*>(cs.wsl) + cs.woff[l];
        stamp(-(300 + l * 10 + 0));
        ctrl_wait_layer(cs.wbar, l);
        stamp(-(300 + l * 10 + 1));
        // rows per warp: the smallest power of two that covers nrow in one pass (<= 8),
        // LPR = 32 / rpw lanes share one row (split-K) and reduce with log2(LPR) shuffles
        int rpw = 1;
        while (rpw < 8 && rpw * nw < nrow) rpw <<= 1;
        const int LPR = 32 / rpw, sub = lane / LPR, sl = lane % LPR;
        for (int i = warp * rpw + sub; i - sub < nrow; i += nw * rpw) {
            const bool live = i < nrow;
            double s0 = 0.0, s1 = 0.0;
            if (live) {
                const TS* wr = Ws + i * C;
                int j = sl;
                for (; j + LPR < C; j += 2 * LPR) {
                    s0 = fma((double)wr[j], x[j], s0);
                    s1 = fma((double)wr[j + LPR], x[j + LPR], s1);
                }
                if (j < C) s0 = fma((double)wr[j], x[j], s0);
            }
            double s = s0 + s1;
            stamp(-(300 + l * 10 + 2));
            for (int o = LPR >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            stamp(-(300 + l * 10 + 3));
            if (live) {
                const double a = s + cs.bsl[l * 64 + i];
                const double y = act_eval(p.hact[l], a, 0);
                stamp(-(300 + l * 10 + 4 + (y == 12345.0)));
                for (int q = sl; q < CS; q += LPR) dsmem_st_f64(dsmem_addr(xn + i0 + i, q), y);
                if (sl == 0) cs.asl[l * 64 + i] = a;
            }
            stamp(-(300 + l * 10 + 6));
        }
        cluster.sync();
        stamp(-(300 + l * 10 + 7));
    }
    if (c == 0) {
        const double* x = cs.xin(p.nhid & 1);
        const int R = p.nhid > 0 ? p.hrows[p.nhid - 1] : p.r;
        for (int j = tid; j < p.hp; j += blockDim.x) p.y_last[j] = j < R ? x[j] : 0.0;
    }
}

// ---- DSMEM data-carried signalling for the fast path ----------------------------------------------
// Layer exchanges without cluster barriers: a producer stores each value into the consumer
// CTA with st.async, which also credits its byte count to an mbarrier in that CTA
// (complete_tx); the consumer waits for the layer's full byte count.  Barriers: fx[l] =
// input of forward layer l (l = 1..nhid, nhid = the last layer's output), bx[l] = partials
// of backward layer l; each completes once per pass, parities in fph / bph.  Every barrier
// is armed (arrive.expect_tx) before the cluster barrier that precedes its pass, so no byte
// can land in an unarmed phase.
struct CtrlSig {
    uint64_t fx[kMaxLayers + 1];
    uint64_t bx[kMaxLayers];
    unsigned fph, bph;
};
__device__ __forceinline__ CtrlSig& ctrl_sig() {
    __shared__ __align__(8) CtrlSig sig;
    return sig;
}
__device__ __forceinline__ void ctrl_sig_init() {
    CtrlSig& g = ctrl_sig();
    if (threadIdx.x == 0) {
        for (int l = 0; l <= kMaxLayers; ++l) mbar_init(&g.fx[l], 1);
        for (int l = 0; l < kMaxLayers; ++l) mbar_init(&g.bx[l], 1);
        g.fph = 0;
        g.bph = 0;
        mbar_fence_init();
    }
}
__device__ __forceinline__ void st_async_f64(uint32_t remote_addr, double v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(remote_addr),
                 "l"(__double_as_longlong(v)), "r"(remote_bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---- uniform-width fast path of the control cluster -------------------------------------------------
// When every hidden layer is HP wide (HP = the padded output-layer input width, a template
// parameter) and HP splits evenly over the CS CTAs, the row partition is static: CTA c owns
// rows [c RPC, (c+1) RPC) of every layer, so loop bounds, lane roles and owners are
// compile-time constants.  Same data flow as ctrl_forward / ctrl_backward (push over DSMEM,
// one cluster barrier per layer); shorter dependent chains per layer: fully unrolled dot
// products with 4 accumulators, unrolled shuffle trees, no integer division.
template <int HP, int CS>
struct CtrlFast {
    static constexpr int RPC = HP / CS;                  // rows per CTA
    static constexpr int RPW = RPC >= 8 ? RPC / 8 : 1;   // rows per warp (warps 0..7, or 0..RPC-1)
    static constexpr int LPR = 32 / RPW;                 // lanes per row
    static constexpr int NCL = HP / LPR;                 // products per lane (layers >= 1)
    static constexpr int NG = (2 * HP <= kSolveThreads) ? (HP <= 64 ? 4 : 2) : 1;  // backward row groups
    static constexpr bool kValid = HP % CS == 0 && RPC <= 64 && (RPC >= 8 ? RPC % 8 == 0 : true) &&
                                   LPR >= CS && NCL >= 1 && HP % LPR == 0 && RPC % NG == 0 &&
                                   HP * NG <= kSolveThreads && HP <= 256;
};

template <typename TS, int HP, int CS>
__device__ __forceinline__ bool ctrl_fast_ok(const EvalParams<TS>& p) {
    if constexpr (!CtrlFast<HP, CS>::kValid) {
        return false;
    } else {
        if (p.nhid < 1 || p.r > 64 || p.r < 1) return false;
        for (int l = 0; l < p.nhid; ++l)
            if (p.hrows[l] != HP || p.hcols[l] != (l == 0 ? p.r : HP)) return false;
        return true;
    }
}

template <typename TS, int HP, int CS>
__device__ __forceinline__ void ctrl_forward_fast(const EvalParams<TS>& p, CtrlSmem& cs, cg::cluster_group& cluster, int c) {
    using F = CtrlFast<HP, CS>;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {
        const double* zsrc = cluster.map_shared_rank(cs.sst->zt, 0);
        for (int j = tid; j < p.r; j += blockDim.x) cs.xin(0)[j] = zsrc[j];
    }
    __syncthreads();
    const int sub = lane / F::LPR, sl = lane % F::LPR;  // compile-time divisors
    const int il = warp * F::RPW + sub;                 // local row (live iff < RPC)
    const bool live = warp < 8 && il < F::RPC;
    const int i0 = c * F::RPC;
    // remote addresses of this lane's push target (CTA sl) for both input buffers
    const uint32_t dst0 = sl < CS ? dsmem_addr(cs.xin(0) + i0 + il, sl) : 0u;
    const uint32_t dst1 = sl < CS ? dsmem_addr(cs.xin(1) + i0 + il, sl) : 0u;
    for (int l = 0; l < p.nhid; ++l) {
        const double* x = cs.xin(l & 1);
        const TS* Ws = reinterpret_cast<const TS*>(cs.wsl) + cs.woff[l];
        ctrl_wait_layer(cs.wbar, l);
        if (live) {
            double a[4] = {0.0, 0.0, 0.0, 0.0};
            if (l == 0) {
                const TS* wr = Ws + il * p.r;
#pragma unroll
                for (int k = 0; k < (64 + F::LPR - 1) / F::LPR; ++k) {
                    const int j = sl + k * F::LPR;
                    if (j < p.r) a[k & 3] = fma((double)wr[j], x[j], a[k & 3]);
                }
            } else {
                const TS* wr = Ws + il * HP + sl;
                const double* xr = x + sl;
#pragma unroll
                for (int k = 0; k < F::NCL; ++k) a[k & 3] = fma((double)wr[k * F::LPR], xr[k * F::LPR], a[k & 3]);
            }
            double s = (a[0] + a[1]) + (a[2] + a[3]);
#pragma unroll
            for (int o = F::LPR >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            const double pre = s + cs.bsl[l * 64 + il];
            if (sl < CS) dsmem_st_f64((l & 1) ? dst0 : dst1, act_eval(p.hact[l], pre, 0));
            // the fast backward reads act'(pre) (computed here, off its critical path)
            if (sl == 0) cs.asl[l * 64 + il] = act_eval(p.hact[l], pre, 1);
        }
        cluster.sync();
    }
    if (c == 0) {
        const double* x = cs.xin(p.nhid & 1);
        for (int j = tid; j < p.hp; j += blockDim.x) p.y_last[j] = j < HP ? x[j] : 0.0;
    }
}

// Backward counterpart (see ctrl_backward): ybar of the last hidden layer is the fixed-order
// sum of the G cluster partials; per layer, partial_c[j] = sum_{own i} W[i][j] gys[i] goes to
// the owner of j, which sums the CS partials in CTA order.  Result -> sst->gz (CTA 0).
template <typename TS, int HP, int CS>
__device__ __forceinline__ void ctrl_backward_fast(const EvalParams<TS>& p, CtrlSmem& cs, cg::cluster_group& cluster, int c, int G,
                                                   const double* ypart) {
    using F = CtrlFast<HP, CS>;
    const int tid = threadIdx.x;
    const int i0 = c * F::RPC;
    double gy = 0.0;  // own-row gradient (threads tid < RPC)
    {
        // ybar: RPC columns x G partials; spread over the block, then a fixed-order fold
        constexpr int PER = kSolveThreads / F::RPC;  // threads per column
        const int col = tid % F::RPC, q = tid / F::RPC;
        double v = 0.0;
        if (q < PER)
            for (int b = q; b < G; b += PER) v += __ldcg(ypart + (size_t)b * p.hp + i0 + col);
        if (q < PER) cs.tmp[q * F::RPC + col] = v;
        __syncthreads();
        if (tid < F::RPC) {
            double s = 0.0;
#pragma unroll 8
            for (int qq = 0; qq < PER; ++qq) s += cs.tmp[qq * F::RPC + tid];
            gy = s;
        }
        __syncthreads();
    }
    const int g = tid % F::NG, j = tid / F::NG;  // thread -> (column, row group)
    constexpr int RG = F::RPC / F::NG;           // rows per group
    for (int l = p.nhid - 1; l >= 0; --l) {
        double* gys = cs.tmp;
        if (tid < F::RPC) gys[tid] = gy * cs.asl[l * 64 + tid];  // act'(pre), stored by ctrl_forward_fast
        const TS* Ws = reinterpret_cast<const TS*>(cs.wsl) + cs.woff[l];
        ctrl_wait_layer(cs.wbar, l);
        __syncthreads();
        double* rb = cs.rbuf(l & 1);
        const int C = l == 0 ? p.r : HP;
        double s = 0.0;
        if (j < C) {
            double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int k = 0; k < RG; ++k) {
                const int i = g * RG + k;
                a[k & 3] = fma((double)Ws[i * C + j], gys[i], a[k & 3]);
            }
            s = (a[0] + a[1]) + (a[2] + a[3]);
        }
        // partner lanes (same column) are adjacent and share the branch outcome
#pragma unroll
        for (int o = 1; o < F::NG; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (j < C && g == 0) {
            const int o = l > 0 ? j / F::RPC : 0;
            const int jl = l > 0 ? j - o * F::RPC : j;
            dsmem_st_f64(dsmem_addr(rb + c * 64 + jl, o), s);
        }
        cluster.sync();
        const int nown = l > 0 ? F::RPC : (c == 0 ? p.r : 0);
        if (tid < nown) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < CS; ++q) s += rb[q * 64 + tid];
            gy = s;
            if (l == 0) cs.sst->gz[tid] = s;
        }
    }
    __syncthreads();
}

// Arm the fast forward's / backward's exchange barriers (thread 0; call before the cluster
// barrier that precedes the pass).
template <int HP, int CS>
__device__ __forceinline__ void ctrl_arm_forward(int nhid) {
    CtrlSig& g = ctrl_sig();
    if (threadIdx.x == 0)
        for (int l = 1; l <= nhid; ++l) mbar_expect_tx(&g.fx[l], HP * 8u);
}
template <int HP, int CS>
__device__ __forceinline__ void ctrl_arm_backward(int nhid, int r, int c) {
    using F = CtrlFast<HP, CS>;
    CtrlSig& g = ctrl_sig();
    if (threadIdx.x == 0)
        for (int l = 0; l < nhid; ++l)
            mbar_expect_tx(&g.bx[l], l > 0 ? (unsigned)(CS * F::RPC * 8) : (c == 0 ? (unsigned)(CS * r * 8) : 0u));
}

// ctrl_forward_fast with the exchange carried by st.async (no cluster barrier per layer).
template <typename TS, int HP, int CS>
__device__ __forceinline__ void ctrl_forward_async(const EvalParams<TS>& p, CtrlSmem& cs, cg::cluster_group& cluster, int c) {
    using F = CtrlFast<HP, CS>;
    CtrlSig& g = ctrl_sig();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {
        const double* zsrc = cluster.map_shared_rank(cs.sst->zt, 0);
        for (int j = tid; j < p.r; j += blockDim.x) cs.xin(0)[j] = zsrc[j];
    }
    const unsigned ph = g.fph;
    __syncthreads();
    const int sub = lane / F::LPR, sl = lane % F::LPR;
    const int il = warp * F::RPW + sub;
    const bool live = warp < 8 && il < F::RPC;
    const int i0 = c * F::RPC;
    const uint32_t dst0 = sl < CS ? dsmem_addr(cs.xin(0) + i0 + il, sl) : 0u;
    const uint32_t dst1 = sl < CS ? dsmem_addr(cs.xin(1) + i0 + il, sl) : 0u;
    for (int l = 0; l < p.nhid; ++l) {
        const double* x = cs.xin(l & 1);
        const TS* Ws = reinterpret_cast<const TS*>(cs.wsl) + cs.woff[l];
        ctrl_wait_layer(cs.wbar, l);
        if (l > 0) mbar_wait_cluster(&g.fx[l], ph);
        if (live) {
            double a[4] = {0.0, 0.0, 0.0, 0.0};
            if (l == 0) {
                const TS* wr = Ws + il * p.r;
#pragma unroll
                for (int k = 0; k < (64 + F::LPR - 1) / F::LPR; ++k) {
                    const int j = sl + k * F::LPR;
                    if (j < p.r) a[k & 3] = fma((double)wr[j], x[j], a[k & 3]);
                }
            } else {
                const TS* wr = Ws + il * HP + sl;
                const double* xr = x + sl;
#pragma unroll
                for (int k = 0; k < F::NCL; ++k) a[k & 3] = fma((double)wr[k * F::LPR], xr[k * F::LPR], a[k & 3]);
            }
            double s = (a[0] + a[1]) + (a[2] + a[3]);
#pragma unroll
            for (int o = F::LPR >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            const double pre = s + cs.bsl[l * 64 + il];
            if (sl < CS)
                st_async_f64((l & 1) ? dst0 : dst1, act_eval(p.hact[l], pre, 0), dsmem_addr(&g.fx[l + 1], sl));
            if (sl == 0) cs.asl[l * 64 + il] = act_eval(p.hact[l], pre, 1);
        }
    }
    mbar_wait_cluster(&g.fx[p.nhid], ph);
    if (c == 0) {
        const double* x = cs.xin(p.nhid & 1);
        for (int j = tid; j < p.hp; j += blockDim.x) p.y_last[j] = j < HP ? x[j] : 0.0;
    }
    __syncthreads();
    if (tid == 0) g.fph = ph ^ 1u;
}

// ctrl_backward_fast with the exchange carried by st.async.
template <typename TS, int HP, int CS, typename Stamp>
__device__ __forceinline__ void ctrl_backward_async(const EvalParams<TS>& p, CtrlSmem& cs, cg::cluster_group& cluster, int c, int G,
                                                    const double* ypart, Stamp& stamp) {
    using F = CtrlFast<HP, CS>;
    CtrlSig& g = ctrl_sig();
    const int tid = threadIdx.x;
    const int i0 = c * F::RPC;
    const unsigned ph = g.bph;
    stamp(-600);
    double gy = 0.0;
    {
        constexpr int PER = kSolveThreads / F::RPC;
        const int col = tid % F::RPC, q = tid / F::RPC;
        double v = 0.0;
        if (q < PER)
            for (int b = q; b < G; b += PER) v += __ldcg(ypart + (size_t)b * p.hp + i0 + col);
        if (q < PER) cs.tmp[q * F::RPC + col] = v;
        __syncthreads();
        if (tid < F::RPC) {
            double s = 0.0;
#pragma unroll 8
            for (int qq = 0; qq < PER; ++qq) s += cs.tmp[qq * F::RPC + tid];
            gy = s;
        }
        __syncthreads();
    }
    stamp(-601);
    const int g4 = tid % F::NG, j = tid / F::NG;
    constexpr int RG = F::RPC / F::NG;
    for (int l = p.nhid - 1; l >= 0; --l) {
        double* gys = cs.tmp + (l & 1) * 64;  // alternate: the next layer's writes race no reader
        if (tid < F::RPC) gys[tid] = gy * cs.asl[l * 64 + tid];
        const TS* Ws = reinterpret_cast<const TS*>(cs.wsl) + cs.woff[l];
        ctrl_wait_layer(cs.wbar, l);
        __syncthreads();
        stamp(-(610 + 10 * l));
        double* rb = cs.rbuf(l & 1);
        const int C = l == 0 ? p.r : HP;
        double s = 0.0;
        if (j < C) {
            double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int k = 0; k < RG; ++k) {
                const int i = g4 * RG + k;
                a[k & 3] = fma((double)Ws[i * C + j], gys[i], a[k & 3]);
            }
            s = (a[0] + a[1]) + (a[2] + a[3]);
        }
#pragma unroll
        for (int o = 1; o < F::NG; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (j < C && g4 == 0) {
            const int o = l > 0 ? j / F::RPC : 0;
            const int jl = l > 0 ? j - o * F::RPC : j;
            st_async_f64(dsmem_addr(rb + c * 64 + jl, o), s, dsmem_addr(&g.bx[l], o));
        }
        stamp(-(611 + 10 * l));
        mbar_wait_cluster(&g.bx[l], ph);
        stamp(-(612 + 10 * l));
        const int nown = l > 0 ? F::RPC : (c == 0 ? p.r : 0);
        if (tid < nown) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < CS; ++q) t += rb[q * 64 + tid];
            gy = t;
            if (l == 0) cs.sst->gz[tid] = t;
        }
    }
    __syncthreads();
    if (tid == 0) g.bph = ph ^ 1u;
    ctrl_arm_backward<HP, CS>(p.nhid, p.r, c);  // the next pass's phase (every byte of this one landed)
}

// ---- the persistent kernel ---------------------------------------------------------------------------
template <typename TS, int HP, int CS>
__global__ void __launch_bounds__(kSolveThreads, 1) solve_kernel(const EvalParams<TS> p, const SolveParams sp) {
    using C = StreamCfg<TS, HP>;
    extern __shared__ __align__(128) unsigned char smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const int G = gridDim.x, cta = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool is_ctrl = cta < CS;  // cluster 0 (clusters are contiguous block ranges)
    const int crank = (int)cluster.block_rank();
    // ---- shared memory carve-up: [barriers | ring (9 x spw stages) | control area (cluster 0)]
    // Control CTAs run a shorter ring (the control area follows it); the others use
    // the whole allocation.
    constexpr int NW = kSolveThreads / 32;
    WarpRing ring{smem + kSolveBarBytes, reinterpret_cast<uint64_t*>(smem), NW, is_ctrl ? sp.spw_ctrl : sp.spw,
                  C::STAGEB, 0u};
    double* cbase = reinterpret_cast<double*>(smem + kSolveBarBytes + (size_t)NW * sp.spw_ctrl * C::STAGEB);
    CtrlSmem cs;
    cs.wsl = cbase;
    cs.xin0 = cbase + sp.wsl_words;
    cs.xin1 = cs.xin0 + kMaxHidden;
    cs.rbuf0 = cs.xin1 + kMaxHidden;
    cs.rbuf1 = cs.rbuf0 + kCtrlRecv;
    cs.tmp = cs.rbuf1 + kCtrlRecv;
    cs.bsl = cs.tmp + kSolveThreads;
    cs.asl = cs.bsl + kMaxLayers * 64;
    cs.sst = reinterpret_cast<DevState*>(cs.asl + kMaxLayers * 64);
    __shared__ double red[32];
    __shared__ double s_energy[2];
    __shared__ int s_flag;
    ring_init(ring.full, NW * ring.spw);
    __syncthreads();
    const int ntiles = (p.n + C::TR - 1) / C::TR;
    // W_out tiles per CTA: the control CTAs run a shallower ring (their control area follows
    // it) and start streaming after the hidden forward, so they take a reduced share
    // (sp.ctrl_tile_w of a full one) of the forward / VJP tiles
    const int t0 = solve_tile_start(ntiles, cta, G, CS, sp.ctrl_tile_w);
    const int t1 = solve_tile_start(ntiles, cta + 1, G, CS, sp.ctrl_tile_w);
    const uint64_t pol_w = l2_policy(p.w_resident), pol_keep = l2_policy(1);
    auto issue_f = [&](int t, unsigned char* b, uint64_t* bar) { issue_fwd<TS, HP>(p, t, b, bar, pol_w, pol_keep); };
    double* tv_s = reinterpret_cast<double*>(smem + (is_ctrl ? sp.tv_off_ctrl : sp.tv_off));
    auto issue_vw = [&](int t, unsigned char* b, uint64_t* bar) { issue_vjp_w<TS, HP>(p, t, b, bar, pol_w); };
    auto issue_vjp = [&](int t, unsigned char* b, uint64_t* bar) {
        if (sp.tv_global) {
            issue_vjp_w<TS, HP>(p, t, b, bar, pol_w);
            issue_vjp_tv<TS, HP>(p, t, b, bar, pol_keep);
        } else {
            issue_fwd<TS, HP>(p, t, b, bar, pol_w, pol_keep);
        }
    };
    DevState* st = p.st;
    SolveShared* sh = sp.sh;
    const bool fast_ctrl = !(sp.exp & 64) && ctrl_fast_ok<TS, HP, CS>(p);
    const bool async_ctrl = fast_ctrl && !(sp.exp & 2048);  // st.async layer exchange
    // The barrier word's atom.add.release.gpu (after bar.sync) and the poll's ld.acquire.gpu
    // (before bar.sync) order every CTA's prior writes before every later read; the extra
    // fence.sc on both sides cost ~2 us per evaluation under load (exp bit 16384 restores it).
    const bool gfence = (sp.exp & 16384) != 0;
    auto gbar = [&]() { grid_barrier(&sp.sh->grid_bar, cta, G, gfence); };
    int tr = 0;
    auto stamp = [&](int tag) {
        // tag < 0: fine-grained cycle stamp (clock64), recorded only with LSB_SOLVE_EXP & 32
        if (sp.trace && cta == 0 && tid == 0 && tr < 255 && (tag >= 0 || (sp.exp & 32))) {
            sp.trace[1 + 2 * tr] = (unsigned long long)(tag >= 0 ? tag : -tag);
            sp.trace[2 + 2 * tr] = tag >= 0 ? globaltimer() : (unsigned long long)clock64();
            sp.trace[0] = (unsigned long long)(++tr);
        }
    };
    stamp(0);
    if (sp.trace && tid == 0 && cta < 256) sp.trace[512 + cta] = globaltimer();

    // ---- control cluster: stage weights (+ state) once.  Issued before any other bulk
    // traffic: an SM's TMA engine serves requests in order.
    __shared__ __align__(8) uint64_t s_wbar[kMaxLayers + 1];
    __shared__ int s_woff[kMaxLayers];
    cs.wbar = s_wbar;
    cs.woff = s_woff;
    if (is_ctrl) ctrl_stage<TS, CS>(p, cs, crank, true, s_wbar);
    stamp(6);
    // the first forward tiles do not depend on z: prefetch now (a step rewrites the
    // qbar column of the row records first, so it prefetches after that)
    // (non-control CTAs issue theirs once the control staging has landed: their bulk reads
    // would otherwise queue ahead of it in HBM)
    const bool defer_pf = p.w_resident && !is_ctrl && !(sp.exp & 8) && !(sp.exp & 128);
    // (the control CTAs issue theirs after the hidden forward: their staging and forward are
    // the critical path of the launch)
    if (sp.task != 2 && !defer_pf && !is_ctrl) ring_prefetch(ring, t0, t1, issue_f);
    if (is_ctrl && crank == 0) {
        stamp(4);
        ctrl_wait_state(s_wbar);  // the state is written below
        if (sp.z_in) {  // z passed with the launch (no separate upload)
            for (int i = tid; i < p.r; i += blockDim.x) cs.sst->zt[i] = sp.z[i];
            __syncthreads();
        }
        stamp(5);
        if (p.nhid > 0) ctrl_wait_layer(s_wbar, 0);
        if (tid == 0) asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(&sp.sh->staged_seq), "r"(sp.seq) : "memory");
    }
    stamp(1);

    // ---- step prologue: qbar - X and warm start (all CTAs), reference reduced_step :249-256
    if (sp.task == 2) {
        const double dt = is_ctrl && crank == 0 ? cs.sst->dt : __ldcg(&st->dt);
        for (int i = cta * blockDim.x + tid; i < p.n; i += G * blockDim.x) {
            const int f = i / 3, c = i - 3 * f;
            const size_t vi = (size_t)p.vfree[f] * 3 + c;
            const double ut = sp.quasi ? 0.0 : sp.u_state[vi] + dt * sp.v_state[vi] + (dt * dt) * sp.a_ext[i];
            p.eprow[6 * (size_t)i + 5] = ut;
        }
        if (is_ctrl && crank == 0) {
            for (int i = tid; i < p.r; i += blockDim.x) cs.sst->zt[i] = sp.z_state[i];
            if (tid == 0) {
                cs.sst->has_inertia = sp.quasi ? 0 : 1;
                cs.sst->inv_dt2 = 1.0 / (dt * dt);
                cs.sst->quasi_static = sp.quasi;
            }
        }
    }
    // ---- start: reset solver state, hidden forward at zt
    if (is_ctrl) {
        if (crank == 0 && tid == 0) {
            DevState* s = cs.sst;
            s->mode = sp.task == 0 ? kModeEval : kModeLbfgs;
            s->want_grad = sp.task == 0 ? sp.want_grad : 1;
            s->status = kStOk;
            s->phase = kPhaseInit;
            s->done = 0;
            s->code = 4;
            s->iter = 0;
            s->ls = 0;
            s->hist_n = 0;
            s->hist_head = 0;
            s->value_evals = 0;
            s->grad_evals = 0;
            s->need_grad = 0;
            s->accept = 0;
            s->gnorm = 0.0;
            s->loop_iters = 0;
            s->t_start = globaltimer();
            sh->mode = s->mode;
            sh->phase = s->phase;
            sh->want_grad = s->want_grad;
            sh->done = 0;
            sh->status = kStOk;
            sh->f = 0.0;
            sh->armijo_slope = 0.0;
            st->has_inertia = s->has_inertia;
            st->inv_dt2 = s->inv_dt2;
        }
        if (async_ctrl) {
            ctrl_sig_init();
            __syncthreads();
            ctrl_arm_forward<HP, CS>(p.nhid);
            ctrl_arm_backward<HP, CS>(p.nhid, p.r, crank);
        }
        cluster.sync();
        if (async_ctrl) ctrl_forward_async<TS, HP, CS>(p, cs, cluster, crank);
        else if (fast_ctrl) ctrl_forward_fast<TS, HP, CS>(p, cs, cluster, crank);
        else ctrl_forward<TS, CS>(p, cs, cluster, crank, stamp);
    }
    stamp(2);
    if (is_ctrl && sp.task != 2) ring_prefetch(ring, t0, t1, issue_f);
    fence_proxy_async();  // generic-proxy row-record writes -> later bulk copies
    {
        const unsigned gold = grid_arrive(&sp.sh->grid_bar, cta, G, gfence);
        if (sp.trace && tid == 0 && cta < 256) sp.trace[512 + 256 + cta] = globaltimer();
        // cold start (e.g. after an L2 flush): while the control cluster runs the hidden forward,
        // pull this CTA's share of W_out, the row records and the element arrays into L2 (only
        // when W_out is L2-resident by policy).  Issued after this CTA's grid-barrier arrival:
        // bulk-copy issue stalls while the SM's TMA queue is full, and must not delay the barrier.
        if (p.w_resident && !is_ctrl && !(sp.exp & 8)) {
            // the non-control CTAs cover every row / tet; they start once the control
            // cluster's (latency-critical) staging has landed, so the bulk traffic overlaps
            // the hidden forward instead of delaying it
            if (lane == 0 && !(sp.exp & 4096)) {
                unsigned s;
                do {
                    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(s) : "l"(&sp.sh->staged_seq) : "memory");
                } while (s != sp.seq);
            }
            __syncwarp();
            if (sp.task != 2 && defer_pf) ring_prefetch(ring, t0, t1, issue_f);
            const int q = cta - CS, Q = G - CS;
            const size_t r0 = (size_t)p.n * q / Q, r1 = (size_t)p.n * (q + 1) / Q;
            const uintptr_t piece = (sp.exp & 8192) ? (uintptr_t)1 << 20 : 32768;
            // the first pf_frac of this CTA's W_out share (the rest streams on demand)
            const size_t wrows = (size_t)((double)(r1 - r0) * sp.pf_frac);
            prefetch_l2_range(p.Wout + r0 * HP, wrows * C::ROWB, piece);
            prefetch_l2_range(p.eprow + r0 * 6, (r1 - r0) * 48, piece);
            const size_t e0 = (size_t)p.E * q / Q, e1 = (size_t)p.E * (q + 1) / Q;
            prefetch_l2_range(p.tets + e0, (e1 - e0) * sizeof(int4), piece);
            prefetch_l2_range(p.fpos + e0, (e1 - e0) * sizeof(int4), piece);
            prefetch_l2_range(p.rec + e0 * 12, (e1 - e0) * 12 * sizeof(TS), piece);
        }
        grid_wait(&sp.sh->grid_bar, gold, gfence);
    }
    stamp(3);
    if (sp.task == 2) ring_prefetch(ring, t0, t1, issue_f);

    bool ring_pending = true;  // a prefetch of the ring is outstanding (drained before exit)
    bool first_pass = true;    // trace: per-CTA phase-end times of the first evaluation
    double inv_dt2 = __ldcg(&st->inv_dt2);
    int has_inertia = __ldcg(&st->has_inertia);
    for (;;) {
        // whether this point's gradient may be needed (known from the solver phase alone; see
        // the speculative VJP below)
        int spec;
        {
            const int phase = __ldcg(&sh->phase), mode = __ldcg(&sh->mode);
            spec = phase == kPhaseFinalDecode ? 0 : (mode == kModeEval ? __ldcg(&sh->want_grad) : 1);
        }
        // ================= out_fwd (self-issued TMA rings; first tiles already in flight)
        {
            double eacc = 0.0;
            {
                double y[C::NCH][C::V4];
#pragma unroll
                for (int c = 0; c < C::NCH; ++c)
#pragma unroll
                    for (int q = 0; q < C::V4; ++q) y[c][q] = __ldcg(p.y_last + (c * 32 + lane) * C::V4 + q);
                const bool ident = p.out_act == kIdentity;
                ring_run(ring, t0, t1, issue_f, [&](int t, const unsigned char* b) {
                    if (!(sp.exp & 1)) eacc += fwd_tile<TS, HP>(p, b, t, y, has_inertia, inv_dt2, ident);
                });
            }
            // the ring streams the same W tiles for every pass: put the next pass's first tiles in
            // flight now (with tv in global memory the VJP's tiles carry tv instead of the row
            // records: their W part goes now, the tv part after the gather)
            if (sp.tv_global && spec) ring_prefetch(ring, t0, t1, issue_vw);
            else if (!(sp.exp & 2)) ring_prefetch(ring, t0, t1, issue_f);
            const double tot = block_sum(eacc, red);
            if (tid == 0) p.e_part_out[cta] = 0.5 * inv_dt2 * tot;
        }
        stamp(10);
        if (sp.trace && tid == 0 && cta < 256 && first_pass) sp.trace[512 + 256 * 2 + cta] = globaltimer();
        gbar();
        stamp(11);
        // ================= element pass
        {
            double eacc = 0.0;
            const int stride = G * blockDim.x;
            // two tets in flight per thread: both index loads, then all 8 vertex gathers
            for (int e0 = cta * blockDim.x + tid; e0 < p.E; e0 += 2 * stride) {
                const int e1 = e0 + stride;
                const bool has1 = e1 < p.E;
                const int4 ta = __ldg(p.tets + e0);
                const int4 tb = has1 ? __ldg(p.tets + e1) : ta;
                double u[2][4][3];
                load_u(p.U, ta.x, u[0][0]);
                load_u(p.U, ta.y, u[0][1]);
                load_u(p.U, ta.z, u[0][2]);
                load_u(p.U, ta.w, u[0][3]);
                load_u(p.U, tb.x, u[1][0]);
                load_u(p.U, tb.y, u[1][1]);
                load_u(p.U, tb.z, u[1][2]);
                load_u(p.U, tb.w, u[1][3]);
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    if (k == 1 && !has1) break;
                    const int e = k ? e1 : e0;
#if LSB_SOLVE_ELEM_F32
                    // fp32-storage mode: fp32 element arithmetic, as on the multi-kernel path
                    eacc += elem_tet<TS>(p.rec, (size_t)e, u[k], __ldg(p.fpos + e), p.forces,
                                         std::is_same<TS, float>::value ? 1 : 0);
#else
                    double rc[12];
                    load_rec<TS>(p.rec, (size_t)e, rc);
                    double f[12];
                    eacc += tet_energy_forces(u[k][0], u[k][1], u[k][2], u[k][3], rc, f);
                    store_forces_csr_t<TS>(p.forces, __ldg(p.fpos + e), f);
#endif
                }
            }
            const double tot = block_sum(eacc, red);
            if (tid == 0) p.e_part_elem[cta] = tot;
        }
        stamp(20);
        if (sp.trace && tid == 0 && cta < 256 && first_pass) sp.trace[512 + 256 * 3 + cta] = globaltimer();
        gbar();
        stamp(21);
        // ================= gradient, speculatively: whether the line search accepts this
        // point (Armijo) needs E, but the VJP is wanted in all other cases and nearly always
        // here, so every CTA runs it when it may be needed and the control cluster alone
        // sums the energy partials and decides (a rejected point's gradient is discarded).
        if (spec) {
            // ================= vjp: tv for this CTA's rows (CSR gather, 2 lanes per vertex)
            // while its first W tiles are in flight, then the self-issued TMA rings
            {
                const int R0 = t0 * C::TR, R1 = min(t1 * C::TR, p.n);
                // control CTAs: the energy partials' loads are issued now and summed after the
                // VJP, off the critical path (G <= 160)
                double pe[5], pi[5];
                if (is_ctrl && warp == 0) {
#pragma unroll
                    for (int k = 0; k < 5; ++k) {
                        const int b = lane + 32 * k;
                        pe[k] = b < G ? __ldcg(p.e_part_elem + b) : 0.0;
                        pi[k] = b < G ? __ldcg(p.e_part_out + b) : 0.0;
                    }
                }
                if (!(sp.exp & 4))
                    gather_rows_smem(p, R0, R1, sp.tv_global ? p.tv + R0 : tv_s, has_inertia, p.out_act == kIdentity,
                                     false);
                if (sp.tv_global) fence_proxy_async();  // generic tv writes -> this CTA's bulk copies
                __syncthreads();
                stamp(30);
                if (sp.exp & 2) ring_prefetch(ring, t0, t1, issue_f);
                if (sp.tv_global && lane == 0) {  // the tv parts of the tiles already in flight
                    const int n = min(ring.spw, ring.count(t0, t1));
                    for (int j = 0; j < n; ++j)
                        issue_vjp_tv<TS, HP>(p, t0 + warp + NW * j, ring.buf(j), ring.bar(j), pol_keep);
                }
                double acc[C::NCH][C::V4];
#pragma unroll
                for (int c = 0; c < C::NCH; ++c)
#pragma unroll
                    for (int q = 0; q < C::V4; ++q) acc[c][q] = 0.0;
                ring_run(ring, t0, t1, issue_vjp, [&](int t, const unsigned char* b) {
                    const double* tvp = sp.tv_global ? reinterpret_cast<const double*>(b + C::TILEB)
                                                     : tv_s + (t * C::TR - R0);
                    if (!(sp.exp & 1)) vjp_tile<TS, HP>(p, b, tvp, t, acc);
                });
                // per-warp partials -> this CTA's ybar partial (fixed warp order) through the
                // idle ring; then the ring is refilled and the cluster pre-reduces over DSMEM
                // (rank order) so the control cluster sums G / CS cluster partials
                __syncthreads();
                double* wred = reinterpret_cast<double*>(ring.ring);  // NW x HP doubles <= ring bytes
#pragma unroll
                for (int c = 0; c < C::NCH; ++c)
#pragma unroll
                    for (int q = 0; q < C::V4; ++q) wred[warp * HP + (c * 32 + lane) * C::V4 + q] = acc[c][q];
                __syncthreads();
                double* cpart = tv_s;  // tv is consumed
                for (int j = tid; j < HP; j += blockDim.x) {
                    double s = 0.0;
#pragma unroll
                    for (int w = 0; w < NW; ++w) s += wred[w * HP + j];
                    cpart[j] = s;
                }
                if (is_ctrl && warp == 0) {
                    double s_el = 0.0, s_in = 0.0;
#pragma unroll
                    for (int k = 0; k < 5; ++k) {
                        s_el += pe[k];
                        s_in += pi[k];
                    }
                    s_el = warp_sum(s_el);
                    s_in = warp_sum(s_in);
                    if (lane == 0) {
                        s_energy[0] = s_el;
                        s_energy[1] = s_in;
                    }
                }
                __syncthreads();
                if (sp.task != 0) ring_prefetch(ring, t0, t1, issue_f);  // the next pass's first tiles
                else ring_pending = false;
                cluster.sync();
                {
                    const int j0 = part_lo(HP, CS, crank), j1 = part_lo(HP, CS, crank + 1);
                    for (int j = j0 + tid; j < j1; j += blockDim.x) {
                        double v[CS];
#pragma unroll
                        for (int r = 0; r < CS; ++r) v[r] = dsmem_ld_f64(dsmem_addr(cpart + j, r));
                        double s = 0.0;
#pragma unroll
                        for (int r = 0; r < CS; ++r) s += v[r];
                        p.ybar_part[(size_t)(cta / CS) * HP + j] = s;
                    }
                }
            }
            stamp(40);
            if (sp.trace && tid == 0 && cta < 256 && first_pass) sp.trace[512 + 256 * 4 + cta] = globaltimer();
            gbar();
            stamp(41);
        }
        // ================= control cluster: gradient, L-BFGS, next hidden forward
        if (is_ctrl) {
            DevState* s = cs.sst;
            // energy (warp 0, fixed lane order; already summed during the VJP when it ran)
            // and the real decision (every control CTA)
            if (!spec && warp == 0) {
                double s_el = 0.0, s_in = 0.0;
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    const int b = lane + 32 * k;
                    s_el += b < G ? __ldcg(p.e_part_elem + b) : 0.0;
                    s_in += b < G ? __ldcg(p.e_part_out + b) : 0.0;
                }
                s_el = warp_sum(s_el);
                s_in = warp_sum(s_in);
                if (lane == 0) {
                    s_energy[0] = s_el;
                    s_energy[1] = s_in;
                }
            }
            __syncthreads();
            const double E = s_energy[0] + (has_inertia ? s_energy[1] : 0.0);
            int need;
            {
                const int phase = __ldcg(&sh->phase), mode = __ldcg(&sh->mode);
                if (phase == kPhaseFinalDecode || !isfinite(E)) need = 0;
                else if (mode == kModeEval) need = __ldcg(&sh->want_grad);
                else if (phase == kPhaseInit) need = 1;
                else need = E <= __ldcg(&sh->f) + __ldcg(&sh->armijo_slope);
            }
            if (crank == 0 && tid == 0) {
                s->f_eval = E;
                s->need_grad = need;
                const bool skip = s->phase == kPhaseFinalDecode;
                if (!skip) s->value_evals++;
                if (!skip && !isfinite(E)) s->status = kStNonFinite;
                if (s->mode == kModeLbfgs && s->phase == kPhaseLineSearch && !skip) s->accept = need;
                if (need) s->grad_evals++;
            }
            // pre-activations of the point just evaluated are in asl (own rows)
            stamp(-390);
            // (async: the backward's barriers were armed at the start / by the previous pass, so
            // no cluster barrier is needed before the first st.async)
            if (async_ctrl) __syncthreads();
            else cluster.sync();
            stamp(-391);
            if (need) {
                if (async_ctrl) ctrl_backward_async<TS, HP, CS>(p, cs, cluster, crank, G / CS, p.ybar_part, stamp);
                else if (fast_ctrl) ctrl_backward_fast<TS, HP, CS>(p, cs, cluster, crank, G / CS, p.ybar_part);
                else ctrl_backward<TS, CS>(p, cs, cluster, crank, G / CS, p.ybar_part, stamp);
            }
            if (crank == 0) {
                if (warp == 0) {
                    int m = 0;
                    if (s->mode == kModeLbfgs) m = lbfgs_control(s, p.r);
                    else if (lane == 0) s->done = 1;
                    if (lane == 0) {
                        s->loop_iters++;
                        if (!m) {
                            s->phase = kPhaseDone;
                            s->t_end = globaltimer();
                        }
                        s_flag = m;
                        sh->done = m ? 0 : 1;
                        sh->phase = s->phase;
                        sh->f = s->f;
                        sh->armijo_slope = 1e-4 * s->alpha * s->gtd;
                        sh->status = s->status;
                    }
                }
                __syncthreads();
            }
            stamp(-392);
            // a single evaluation (task 0) has no next forward
            int more = 0;
            if (sp.task != 0) {
                if (async_ctrl) ctrl_arm_forward<HP, CS>(p.nhid);
                cluster.sync();
                stamp(-393);
                more = *cluster.map_shared_rank(&s_flag, 0);
            }
            if (more) {
                if (async_ctrl) ctrl_forward_async<TS, HP, CS>(p, cs, cluster, crank);
                else if (fast_ctrl) ctrl_forward_fast<TS, HP, CS>(p, cs, cluster, crank);
                else ctrl_forward<TS, CS>(p, cs, cluster, crank, stamp);
            }
        }
        stamp(50);
        // a single evaluation ends here: its control cluster decides alone, and no CTA needs
        // the state of another before exiting
        if (sp.task == 0) break;
        first_pass = false;
        gbar();
        stamp(51);
        if (__ldcg(&sh->done)) break;
    }
    if (ring_pending) ring_drain(ring, t0, t1);
    stamp(60);
    // ---- epilogue: publish state; step finalize (reference reduced_step :266-276)
    if (is_ctrl && crank == 0) {
        __syncthreads();
        const int nvec = sizeof(DevState) / 16;  // 16-byte sized and aligned
        int4* dst = reinterpret_cast<int4*>(st);
        const int4* src = reinterpret_cast<const int4*>(cs.sst);
        for (int k = tid; k < nvec; k += blockDim.x) dst[k] = src[k];
        if (sp.out_map) {  // the evaluation's result straight into host memory
            for (int i = tid; i < p.r; i += blockDim.x) sp.out_map[2 + i] = cs.sst->gz[i];
            if (tid == 0) {
                sp.out_map[0] = cs.sst->f_eval;
                sp.out_map[1] = (double)cs.sst->status;
            }
        }
    }
    if (sp.task == 2) {
        gbar();
        const double dt = __ldcg(&st->dt);
        for (int v = cta * blockDim.x + tid; v < p.V; v += G * blockDim.x)
            for (int c = 0; c < 3; ++c) {
                const size_t k = (size_t)v * 3 + c;
                const double un = sp.vpinned[v] ? sp.pin_disp[k] : __ldcg(p.U + (size_t)v * 4 + c);
                sp.v_state_w[k] = sp.quasi ? 0.0 : (un - sp.u_state[k]) / dt;
                sp.u_state_w[k] = un;
            }
        if (cta == 0) {
            const int idx = st->step_idx;
            for (int i = tid; i < p.r; i += blockDim.x) {
                sp.z_state[i] = st->x[i];
                if (st->z_traj) st->z_traj[(size_t)idx * p.r + i] = st->x[i];
            }
            if (tid == 0) {
                struct Rep {
                    int code, iterations;
                    double gnorm, ms;
                    int ve, ge;
                };
                Rep* reps = static_cast<Rep*>(st->reports);
                Rep rr;
                rr.code = st->status != kStOk ? -st->status : st->code;
                rr.iterations = st->iter;
                rr.gnorm = st->gnorm;
                rr.ms = (double)(st->t_end - st->t_start) * 1e-6;
                rr.ve = st->value_evals;
                rr.ge = st->grad_evals;
                if (reps) reps[idx] = rr;
                st->step_idx = idx + 1;
                st->t += dt;
            }
        }
    }
    if (cta == 0 && tid == 0 && sp.launch_acc) sp.launch_acc[0] += 0;  // single launch
    stamp(61);
    cluster.sync();  // keep DSMEM alive until every remote read is done
    stamp(62);
}

// ---- multi-kernel path: the control cluster as its own launch, fast path ----------------------------
// Same role as ctrl_kernel (lsb_kernels.cuh) -- kCtrlStart: reset the solver state and run the
// hidden forward at zt; kCtrlAfterEval: hidden backward (if the gradient is needed), L-BFGS
// step, and the next hidden forward if the solve continues -- for decoders whose hidden layers
// are all HP wide, using the uniform-width fast path (ctrl_forward_async / ctrl_backward_async).
// act'(a) of the last forward is kept in p.a_hid between launches (ctrl_kernel keeps a there;
// a context uses one of the two kernels).
template <typename TS, int HP, int CS>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(kSolveThreads, 1)
    ctrl_fast_kernel(const EvalParams<TS> p, int cmode, int start_mode, int start_want_grad) {
    using F = CtrlFast<HP, CS>;
    extern __shared__ __align__(128) unsigned char smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const int c = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int wsl_elems = 0;
    for (int l = 0; l < p.nhid; ++l) wsl_elems += (F::RPC * p.hcols[l] + 3) & ~3;
    const int wsl_words = (int)((wsl_elems * sizeof(TS) + 7) / 8);
    double* cbase = reinterpret_cast<double*>(smem);
    CtrlSmem cs;
    cs.wsl = cbase;
    cs.xin0 = cbase + wsl_words;
    cs.xin1 = cs.xin0 + kMaxHidden;
    cs.rbuf0 = cs.xin1 + kMaxHidden;
    cs.rbuf1 = cs.rbuf0 + kCtrlRecv;
    cs.tmp = cs.rbuf1 + kCtrlRecv;
    cs.bsl = cs.tmp + kSolveThreads;
    cs.asl = cs.bsl + kMaxLayers * 64;
    cs.sst = reinterpret_cast<DevState*>(cs.asl + kMaxLayers * 64);
    __shared__ __align__(8) uint64_t s_wbar[kMaxLayers + 1];
    __shared__ int s_woff[kMaxLayers];
    __shared__ int more_s;
    cs.wbar = s_wbar;
    cs.woff = s_woff;
    ctrl_sig_init();
    ctrl_stage<TS, CS>(p, cs, c, true, s_wbar);  // weights staged while the previous kernel drains
    griddep_wait();
    griddep_launch();
    if (c == 0) ctrl_wait_state(s_wbar);
    DevState* sst = cs.sst;
    const int need = cmode == kCtrlAfterEval ? __ldcg(&p.st->need_grad) : 0;
    int more = 1;
    if (cmode == kCtrlAfterEval) {
        if (need) {
            for (int k = tid; k < p.nhid * F::RPC; k += blockDim.x) {
                const int l = k / F::RPC, i = k - l * F::RPC;
                cs.asl[l * 64 + i] = __ldcg(p.a_hid + l * kMaxHidden + c * F::RPC + i);
            }
            ctrl_arm_backward<HP, CS>(p.nhid, p.r, c);
            cluster.sync();
            auto nostamp = [](int) {};
            ctrl_backward_async<TS, HP, CS>(p, cs, cluster, c, p.n_groups, p.ybar_grp, nostamp);
        }
        __syncthreads();
        if (c == 0) {
            if (warp == 0) {
                int m = 0;
                if (sst->mode == kModeLbfgs) m = lbfgs_control(sst, p.r);
                else if (lane == 0) sst->done = 1;
                if (lane == 0) {
                    sst->loop_iters++;
                    if (!m) {
                        sst->phase = kPhaseDone;
                        sst->t_end = globaltimer();
                    }
                    more_s = m;
                }
            }
            __syncthreads();
            more = more_s;
        }
    } else if (c == 0 && tid == 0) {  // kCtrlStart: fresh evaluation / solve at st->zt
        sst->mode = start_mode;
        sst->want_grad = start_want_grad;
        sst->status = kStOk;
        sst->phase = kPhaseInit;
        sst->done = 0;
        sst->code = 4;
        sst->iter = 0;
        sst->ls = 0;
        sst->hist_n = 0;
        sst->hist_head = 0;
        sst->value_evals = 0;
        sst->grad_evals = 0;
        sst->need_grad = 0;
        sst->accept = 0;
        sst->gnorm = 0.0;
        sst->loop_iters = 0;
        sst->t_start = globaltimer();
    }
    if (c == 0 && tid == 0) more_s = more;
    ctrl_arm_forward<HP, CS>(p.nhid);
    cluster.sync();
    more = *cluster.map_shared_rank(&more_s, 0);
    if (more) {
        ctrl_forward_async<TS, HP, CS>(p, cs, cluster, c);
        for (int k = tid; k < p.nhid * F::RPC; k += blockDim.x) {
            const int l = k / F::RPC, i = k - l * F::RPC;
            p.a_hid[l * kMaxHidden + c * F::RPC + i] = cs.asl[l * 64 + i];
        }
    }
    if (c == 0) {
        __syncthreads();
        const int nvec = sizeof(DevState) / 16;  // 16-byte sized and aligned
        int4* dst = reinterpret_cast<int4*>(p.st);
        const int4* src = reinterpret_cast<const int4*>(sst);
        for (int k = tid; k < nvec; k += blockDim.x) dst[k] = src[k];
        if (tid == 0 && p.in_graph) cudaGraphSetConditional(p.cond, more ? 1u : 0u);
    }
    cluster.sync();  // keep shared memory alive until all remote reads are done
}

// smem bytes of ctrl_fast_kernel for a decoder with hidden input widths hcols[0..nhid)
template <typename TS>
inline size_t ctrl_fast_smem(int nhid, const int* hcols, int rpc) {
    size_t e = 0;
    for (int l = 0; l < nhid; ++l) e += ((size_t)rpc * hcols[l] + 3) & ~(size_t)3;
    return ((e * sizeof(TS) + 7) / 8 + ctrl_fixed_words()) * sizeof(double);
}

}  // namespace lsb
