// Dataflow "sweep" pass of the multi-kernel path (large n, e.g. config 3): the output-layer
// forward stream, the element pass, the vertex gather and the VJP stream of one evaluation as
// ONE persistent, warp-specialised kernel (one CTA per SM).
//
// Why: as separate kernels (out_fwd -> elem -> vjp_gather) the element pass (~36 us on config 3,
// latency-bound on vertex gathers) and the kernel boundaries sit between the two HBM-bound W_out
// streams.  A tet only needs the displacements of its own 4 vertices and a VJP row only needs the
// forces of the tets around its vertex; with the bar's x-slab-major numbering both are local.
//
// Work items (host-built plan, lsb_context.cu setup_sweep):
//   F f  forward rows of kSwItemTiles W_out tiles: u -> U, inertia residual, energy partial
//   E b  kSwTets tets (needs F items <= depF[b]): energy partial, forces -> CSR slots
//   G g  gather of kSwGatherRows rows (needs E items <= depG[g]): tv = s (g + inertia) -> global
//   V v  VJP rows of kSwItemTiles tiles (needs G items <= depV[v]): ybar_item = W^T tv
//
// Roles inside every CTA:
//   * kSwStreamWarps streaming warps, each with its own kSwStages-deep ring of bulk copies (W tile
//     + per-row records, or W tile + tv rows), claim F items and then V items from the stream
//     queue (ticket t < nf: F t, else V t - nf) and never stop streaming for element work: the
//     issue cursor runs across item boundaries (one item claimed ahead);
//   * the element group (kSwElemWarps warps, named barrier 1) claims E and G items from the element
//     queue (host order: every G item after the E items it gathers from, with a lag of about one
//     grid of tickets).
// Deadlock-free: every F item is claimed before any V item, E items wait only on F items, G only
// on E, V only on G; a claimed item is held by a running warp.  Co-residency is not required.
//
// Readiness: per-item done flags carry the launch sequence number (no reset); a monotone watermark
// per item kind (number of leading done items) is advanced by waiters with warp-wide flag scans.
//
// Determinism: every partial is per item (energies of F and E items, ybar of V items) and every
// total sums them in item order (V groups of kSwGroup by the group's last finisher, then the
// control kernel over groups): results do not depend on which warp ran which item.
//
// The gradient is speculative inside an L-BFGS solve (V items run before the Armijo decision of
// their evaluation is known, as in the persistent kernel); value-only evaluations (lsb_eval
// without gradient, the final decode of a step) run no G and V items.
#pragma once

#include "lsb_stream.cuh"

// Developer timing experiments (tools/build_explib.sh only; results invalid): bit 1 skips the
// element math of E items, bit 2 the gather of G items, bit 4 the tile math of F / V items.
#ifndef LSB_SWEEP_EXP
#define LSB_SWEEP_EXP 0
#endif

namespace lsb {

constexpr int kSwStreamWarps = 8;
constexpr int kSwElemWarps = 8;
constexpr int kSwThreads = 32 * (kSwStreamWarps + kSwElemWarps);
constexpr int kSwElemThreads = 32 * kSwElemWarps;
constexpr int kSwStages = 3;                        // ring stages per streaming warp
constexpr int kSwItemTiles = 16;                    // W_out tiles per F / V item
constexpr int kSwTets = 2 * kSwElemThreads;         // tets per E item (two per element thread)
constexpr int kSwGatherRows = 3 * kSwElemThreads;   // rows per G item (one free vertex per thread)
constexpr int kSwGroup = 32;                        // V items per ybar group partial
enum SweepKind : int { kSwE = 1, kSwG = 2 };

struct SweepCounters {  // tickets / e_fin / watermarks zeroed and seq advanced by the last CTA of a launch
    unsigned sticket, eticket, exit_cnt, e_fin;
    unsigned seq, pad0, pad1, pad2;  // seq: launch sequence number (starts at 1), tags the done flags
    int f_wm, e_wm, g_wm, pad3;
};

struct SweepParams {
    const int* eorder;  // element queue: ticket -> (kind << 28) | index
    int etotal, nf, ne, ng, nv, ngroups;
    const int* depF;    // ne: largest F item an E item reads (-1: none)
    const int* depG;    // ng: largest E item a G item gathers from (-1: none)
    const int* depV;    // nv: largest G item a V item reads tv from
    unsigned* f_done;   // nf: launch sequence number when done
    unsigned* e_done;   // ne
    unsigned* g_done;   // ng
    double* e_f;        // nf: inertia energy partial of each F item (times 1/(2h^2))
    double* e_e;        // ne: elastic energy of each E item
    double* ybar_item;  // nv x hp
    double* ybar_grp;   // ngroups x hp
    unsigned* grp_cnt;  // ngroups (self-resetting)
    SweepCounters* ctr;
    unsigned long long* trace;  // developer trace (LSB_TRACE=1): {unit << 32 | kind idx, t0, t_ready, t1}
    int trace_cap;              // trace records (nf + nv + etotal)
};

template <typename TS, int HP>
__host__ __device__ constexpr size_t sweep_smem_bytes() {
    return 128 + (size_t)kSwStreamWarps * kSwStages * StreamCfg<TS, HP>::STAGEB;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acquire_s32(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void atom_max_release(int* p, int v) {
    asm volatile("red.release.gpu.global.max.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Displacements of vertex v through L2 (rows written by other CTAs during the launch).
__device__ __forceinline__ void load_u_cg(const double* U, int v, double* o) {
    const double2 a = __ldcg(reinterpret_cast<const double2*>(U + (size_t)v * 4));
    o[0] = a.x;
    o[1] = a.y;
    o[2] = __ldcg(U + (size_t)v * 4 + 2);
}

// Warp-wide: advance the watermark `wm` over done[] flags equal to seq (up to count); returns the
// watermark this warp observed / established.
__device__ __forceinline__ int sweep_advance(int* wm, const unsigned* done, int count, unsigned seq) {
    const int lane = threadIdx.x & 31;
    int w = __shfl_sync(0xffffffffu, lane == 0 ? ld_acquire_s32(wm) : 0, 0);
    const int w0 = w;
    while (w < count) {
        const int k = w + lane;
        const bool ok = k < count && ld_acquire_u32(done + k) == seq;
        const unsigned b = __ballot_sync(0xffffffffu, ok);
        if (b == 0xffffffffu) {
            w += 32;
            continue;
        }
        w += __ffs(~b) - 1;
        break;
    }
    if (w > w0 && lane == 0) atom_max_release(wm, w);
    return w;
}

// Warp-wide: wait until watermark > need (need < 0: nothing to wait for).
__device__ __forceinline__ void sweep_wait(int* wm, const unsigned* done, int count, unsigned seq, int need) {
    if (need < 0) return;
    if (__shfl_sync(0xffffffffu, (threadIdx.x & 31) == 0 ? ld_acquire_s32(wm) : 0, 0) > need) return;
    while (sweep_advance(wm, done, count, seq) <= need) __nanosleep(64);
}

__device__ __forceinline__ void elem_bar() { named_bar_sync(1, kSwElemThreads); }

// Sum over the element group (fixed tree: deterministic).
__device__ __forceinline__ double elem_group_sum(double v, double* scratch) {
    const int lane = threadIdx.x & 31, ew = (threadIdx.x >> 5) - kSwStreamWarps;
    v = warp_sum(v);
    elem_bar();
    if (lane == 0) scratch[ew] = v;
    elem_bar();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kSwElemWarps; ++w) t += scratch[w];
    elem_bar();
    return t;
}

template <typename TS, int HP>
__global__ void __launch_bounds__(kSwThreads, 1) sweep_kernel(const EvalParams<TS> p, const SweepParams sp) {
    using C = StreamCfg<TS, HP>;
    extern __shared__ __align__(128) unsigned char ssm[];
    __shared__ double red[32];
    __shared__ int s_eitem, s_last;
    __shared__ unsigned s_seq;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint64_t* full = reinterpret_cast<uint64_t*>(ssm);  // kSwStreamWarps x kSwStages
    griddep_wait();  // launched with a programmatic edge from the control kernel: y and the state first
    if (tid == 0) {
        for (int s = 0; s < kSwStreamWarps * kSwStages; ++s) mbar_init(&full[s], 1);
        mbar_fence_init();
        s_seq = __ldcg(&sp.ctr->seq);
    }
    __syncthreads();
    SweepCounters* ctr = sp.ctr;
    const unsigned seq = s_seq;
    DevState* st = p.st;
    const int spec = st->phase != kPhaseFinalDecode && (st->mode != kModeEval || st->want_grad);
    const double inv_dt2 = st->inv_dt2;
    const int has_inertia = st->has_inertia;
    const bool ident = p.out_act == kIdentity;
    const int ntiles = (p.n + C::TR - 1) / C::TR;
    const int stotal = sp.nf + (spec ? sp.nv : 0);

    if (warp < kSwStreamWarps) {
        // ======================= streaming warp: F items, then V items =======================
        unsigned char* ring = ssm + 128 + (size_t)warp * kSwStages * C::STAGEB;
        uint64_t* bars = full + warp * kSwStages;
        const uint64_t pol = l2_policy(p.w_resident), keep = l2_policy(1);
        constexpr bool kMixed = std::is_same<TS, float>::value;  // fp32 storage: reduced-cost tile math
        double y[C::NCH][C::V4];
        float yh[C::NCH][4], yl[C::NCH][4];
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
#pragma unroll
            for (int q = 0; q < C::V4; ++q) {
                y[c][q] = p.y_last[(c * 32 + lane) * C::V4 + q];
                if constexpr (kMixed) {
                    yh[c][q] = (float)y[c][q];
                    yl[c][q] = (float)(y[c][q] - (double)yh[c][q]);
                }
            }
        auto claim = [&]() {
            int t = 0;
            if (lane == 0) t = (int)atomicAdd(&ctr->sticket, 1u);
            return __shfl_sync(0xffffffffu, t, 0);
        };
        auto tiles_of = [&](int it, int& t0, int& t1) {
            const int idx = it < sp.nf ? it : it - sp.nf;
            t0 = idx * kSwItemTiles;
            t1 = min(ntiles, t0 + kSwItemTiles);
        };
        int A = claim();  // item being consumed
        int B = claim();  // next item
        int ia = A, it_ = 0, itn = 0;  // issue cursor: item, next tile, tile end
        if (ia < stotal) tiles_of(ia, it_, itn);
        unsigned is = 0, cs = 0;  // issued / consumed tile counts (stage = count % kSwStages)
        uint32_t ph = 0;          // parity bit per stage
        // issue tiles while a stage is free; the cursor moves from A to B (never further)
        auto fill = [&]() {
            while (is - cs < (unsigned)kSwStages && ia < stotal) {
                if (it_ >= itn) {  // cursor item exhausted: move to the next claimed item, if known
                    const int nx = ia == A ? B : (ia == B ? stotal : A);
                    if (nx >= stotal) break;
                    ia = nx;
                    tiles_of(ia, it_, itn);
                    continue;
                }
                const int s = (int)(is % kSwStages);
                unsigned char* stg = ring + (size_t)s * C::STAGEB;
                if (ia < sp.nf) {
                    if (lane == 0) issue_fwd<TS, HP>(p, it_, stg, bars + s, pol, keep);
                } else {
                    const int v = ia - sp.nf;
                    if (it_ == v * kSwItemTiles) {
                        // first tile of a V item: the tv of its rows must be final.  Block only for
                        // the item being consumed (it holds no unfinished earlier work); for the
                        // look-ahead item just probe, and retry on the next call.
                        const int need = __ldg(sp.depV + v);
                        if (ia == A) sweep_wait(&ctr->g_wm, sp.g_done, sp.ng, seq, need);
                        else if (sweep_advance(&ctr->g_wm, sp.g_done, sp.ng, seq) <= need) break;
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    if (lane == 0) {
                        issue_vjp_w<TS, HP>(p, it_, stg, bars + s, pol);
                        issue_vjp_tv<TS, HP>(p, it_, stg, bars + s, keep);
                    }
                }
                ++it_;
                ++is;
            }
        };
        while (A < stotal) {
            int t0, t1;
            tiles_of(A, t0, t1);
            const bool isF = A < sp.nf;
            const int idx = isF ? A : A - sp.nf;
            const int nextC = claim();  // consumed when A is done
            unsigned long long tr0 = 0;
            if (sp.trace && lane == 0) tr0 = globaltimer();
            double eacc = 0.0;
            double acc[C::NCH][C::V4];
#pragma unroll
            for (int c = 0; c < C::NCH; ++c)
#pragma unroll
                for (int q = 0; q < C::V4; ++q) acc[c][q] = 0.0;
            for (int t = t0; t < t1; ++t) {
                fill();
                const int s = (int)(cs % kSwStages);
                mbar_wait(bars + s, (ph >> s) & 1u);
                ph ^= 1u << s;
                const unsigned char* stg = ring + (size_t)s * C::STAGEB;
                if constexpr ((LSB_SWEEP_EXP & 4) != 0) {
                    eacc += stg[lane];
                } else if constexpr (kMixed) {
                    if (isF) eacc += fwd_tile_mixed<HP>(p, stg, t, yh, yl, has_inertia, inv_dt2, ident);
                    else vjp_tile_mixed<HP>(p, stg, reinterpret_cast<const double*>(stg + C::TILEB), t, acc);
                } else {
                    if (isF) eacc += fwd_tile<TS, HP>(p, stg, t, y, has_inertia, inv_dt2, ident);
                    else vjp_tile<TS, HP>(p, stg, reinterpret_cast<const double*>(stg + C::TILEB), t, acc);
                }
                __syncwarp();
                ++cs;
            }
            if (isF) {
                const double tot = warp_sum(eacc);
                __threadfence();
                __syncwarp();
                if (lane == 0) {
                    sp.e_f[idx] = 0.5 * inv_dt2 * tot;
                    st_release_u32(sp.f_done + idx, seq);
                }
            } else {
#pragma unroll
                for (int c = 0; c < C::NCH; ++c)
#pragma unroll
                    for (int q = 0; q < C::V4; ++q)
                        sp.ybar_item[(size_t)idx * HP + (c * 32 + lane) * C::V4 + q] = acc[c][q];
                __threadfence();
                __syncwarp();
                const int g = idx / kSwGroup;
                const int g0 = g * kSwGroup, g1 = min(g0 + kSwGroup, sp.nv);
                int last = 0;
                if (lane == 0) last = atomicAdd(sp.grp_cnt + g, 1u) == (unsigned)(g1 - g0 - 1);
                if (__shfl_sync(0xffffffffu, last, 0)) {  // the group's last finisher: item-order sum
                    __threadfence();
#pragma unroll
                    for (int c = 0; c < C::NCH; ++c)
#pragma unroll
                        for (int q = 0; q < C::V4; ++q) {
                            const int j = (c * 32 + lane) * C::V4 + q;
                            double sum = 0.0;
                            for (int b = g0; b < g1; ++b) sum += __ldcg(sp.ybar_item + (size_t)b * HP + j);
                            sp.ybar_grp[(size_t)g * HP + j] = sum;
                        }
                    if (lane == 0) sp.grp_cnt[g] = 0;
                }
            }
            if (sp.trace && lane == 0 && A < sp.trace_cap) {
                sp.trace[4 * (size_t)A] =
                    ((unsigned long long)(blockIdx.x * 16 + warp) << 32) | (isF ? 0u : 3u << 28) | (unsigned)idx;
                sp.trace[4 * (size_t)A + 1] = tr0;
                sp.trace[4 * (size_t)A + 2] = tr0;
                sp.trace[4 * (size_t)A + 3] = globaltimer();
            }
            A = B;
            B = nextC;
        }
    } else {
        // ======================= element group: E items and G items =======================
        constexpr int kElemF32 = std::is_same<TS, float>::value ? 1 : 0;  // fp32 element arithmetic (fp32 storage)
        const int et = tid - kSwStreamWarps * 32;  // 0 .. kSwElemThreads-1
        auto eclaim = [&]() {
            if (et == 0) s_eitem = (int)atomicAdd(&ctr->eticket, 1u);
            elem_bar();
            const int v = s_eitem;
            elem_bar();
            return v;
        };
        int cur = eclaim();
        while (cur < sp.etotal) {
            const int code = __ldg(sp.eorder + cur);
            const int kind = code >> 28, idx = code & 0x0fffffff;
            unsigned long long tr0 = 0, tr1 = 0;
            if (sp.trace && et == 0) tr0 = globaltimer();
            if (kind == kSwE) {
                if (warp == kSwStreamWarps) sweep_wait(&ctr->f_wm, sp.f_done, sp.nf, seq, __ldg(sp.depF + idx));
                if (sp.trace && et == 0) tr1 = globaltimer();
                elem_bar();
                double eacc = 0.0;
                if constexpr ((LSB_SWEEP_EXP & 1) == 0) {
                    const int e0 = idx * kSwTets + et, e1 = e0 + kSwElemThreads;
                    const bool h0 = e0 < p.E, h1 = e1 < p.E;
                    const int4 q0 = h0 ? __ldg(p.tets + e0) : make_int4(0, 0, 0, 0);
                    const int4 q1 = h1 ? __ldg(p.tets + e1) : q0;
                    double u[2][4][3];
                    load_u_cg(p.U, q0.x, u[0][0]);
                    load_u_cg(p.U, q0.y, u[0][1]);
                    load_u_cg(p.U, q0.z, u[0][2]);
                    load_u_cg(p.U, q0.w, u[0][3]);
                    load_u_cg(p.U, q1.x, u[1][0]);
                    load_u_cg(p.U, q1.y, u[1][1]);
                    load_u_cg(p.U, q1.z, u[1][2]);
                    load_u_cg(p.U, q1.w, u[1][3]);
                    if (h0) eacc += elem_tet<TS>(p.rec, (size_t)e0, u[0], __ldg(p.fpos + e0), p.forces, kElemF32);
                    if (h1) eacc += elem_tet<TS>(p.rec, (size_t)e1, u[1], __ldg(p.fpos + e1), p.forces, kElemF32);
                }
                __threadfence();
                const double tot = elem_group_sum(eacc, red);
                if (et == 0) {
                    sp.e_e[idx] = tot;
                    st_release_u32(sp.e_done + idx, seq);
                    s_last = atomicAdd(&ctr->e_fin, 1u) == (unsigned)(sp.ne - 1);
                }
                elem_bar();
                if (s_last) {
                    // last element item: total energy in item order once every F item is done,
                    // Armijo decision (as elem_kernel's last block)
                    if (warp == kSwStreamWarps) sweep_wait(&ctr->f_wm, sp.f_done, sp.nf, seq, sp.nf - 1);
                    elem_bar();
                    double s = 0.0;
                    for (int b = et; b < sp.nf; b += kSwElemThreads) s += __ldcg(sp.e_f + b);
                    const double e_in = elem_group_sum(s, red);
                    s = 0.0;
                    for (int b = et; b < sp.ne; b += kSwElemThreads) s += __ldcg(sp.e_e + b);
                    const double e_el = elem_group_sum(s, red);
                    if (et == 0) {
                        const bool skip = st->phase == kPhaseFinalDecode;
                        const double Et = e_el + (st->has_inertia ? e_in : 0.0);
                        st->f_eval = Et;
                        if (!skip) st->value_evals++;
                        int need = 0;
                        if (skip) {
                            need = 0;
                        } else if (!isfinite(Et)) {  // reduced_solver.cpp:198-199 (throws)
                            st->status = kStNonFinite;
                        } else if (st->mode == kModeEval) {
                            need = st->want_grad;
                        } else if (st->phase == kPhaseInit) {
                            need = 1;
                        } else {  // Armijo test (reduced_solver.cpp:49)
                            const int acc = Et <= st->f + 1e-4 * st->alpha * st->gtd;
                            st->accept = acc;
                            need = acc;
                        }
                        st->need_grad = need;
                        if (need) st->grad_evals++;
                    }
                }
            } else if (spec) {
                // G item: tv = s (g + inertia residual) for rows [idx GR, ...) into global tv
                if (warp == kSwStreamWarps) sweep_wait(&ctr->e_wm, sp.e_done, sp.ne, seq, __ldg(sp.depG + idx));
                if (sp.trace && et == 0) tr1 = globaltimer();
                elem_bar();
                const int R0 = idx * kSwGatherRows, R1 = min(p.n, R0 + kSwGatherRows);
                const int f0 = R0 / 3, f1 = (R1 - 1) / 3;
                const int f = f0 + et;
                if ((LSB_SWEEP_EXP & 2) == 0 && f <= f1) gather_vertex1(p, f, R0, R1, p.tv + R0, has_inertia, ident);
                __threadfence();
                asm volatile("fence.proxy.async.global;" ::: "memory");
                elem_bar();
                if (et == 0) st_release_u32(sp.g_done + idx, seq);
            }
            if (sp.trace && et == 0) {
                const int rec = sp.nf + sp.nv + cur;
                if (rec < sp.trace_cap) {
                    sp.trace[4 * (size_t)rec] = ((unsigned long long)(blockIdx.x * 16 + kSwStreamWarps) << 32) |
                                                ((unsigned)kind << 28) | (unsigned)idx;
                    sp.trace[4 * (size_t)rec + 1] = tr0;
                    sp.trace[4 * (size_t)rec + 2] = tr1 ? tr1 : tr0;
                    sp.trace[4 * (size_t)rec + 3] = globaltimer();
                }
            }
            cur = eclaim();
        }
    }
    // exit: the last CTA out resets the counters for the next launch
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(&ctr->exit_cnt, 1u) == gridDim.x - 1) {
            ctr->sticket = 0;
            ctr->eticket = 0;
            ctr->e_fin = 0;
            ctr->f_wm = 0;
            ctr->e_wm = 0;
            ctr->g_wm = 0;
            ctr->seq = seq + 1u == 0u ? 1u : seq + 1u;
            __threadfence();
            ctr->exit_cnt = 0;
        }
    }
}

}  // namespace lsb
