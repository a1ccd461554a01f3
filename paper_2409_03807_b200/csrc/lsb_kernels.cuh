// Single-instance E(z) + grad E(z) kernels and the device-resident L-BFGS
// control (SURVEY §2.2 kernels K1..K6).
//
// Precision by role: `TS` is the STORAGE type of the two bandwidth-bound
// arrays (decoder output layer W_out and the per-tet element records): double
// in fp64 mode, float in fp32 mode.  All arithmetic is fp64 in both modes (the
// kernels are HBM-bound and B200 FP64 runs at half the FP32 rate), so the
// objective stays a smooth function of z and the Armijo test keeps resolving
// energy decreases ~1e-9 relative to E (config 3 needs it).
//
// One objective evaluation at the latent point zt is four kernels:
//   out_fwd   (K2)  stream W_out (n x hp, row-major, 32-byte vector loads) against
//                   the last hidden activation y: u = s*phi(W y + b) + (shift - X),
//                   scattered into the vertex displacement array U (fp64);
//                   inertia residual r = m (u - ut) / dt^2; energy partials.
//   elem      (K3)  per tet: gather 4 vertex displacements, A = dU Dm^-1,
//                   cancellation-free stable neo-Hookean psi and P, 12 local forces
//                   vol P Dm^-T into a per-tet buffer; energy partials.  The last
//                   block sums all partials in block order and makes the Armijo
//                   accept decision (so the gradient pass runs only when needed).
//   vjp       (K3b+K4) when the gradient is needed: per free vertex CSR gather
//                   of the per-tet forces in ascending tet id (the scatter order
//                   of the reference assemble) + inertia, times s; second stream
//                   of W_out accumulating ybar = W_out^T (s g) in registers;
//                   deterministic two-level block reduction to group partials.
//   ctrl      (K5+K6, one thread-block cluster): hidden-layer weights staged in
//                   the cluster's shared memory (row slices per CTA, exchanged
//                   through DSMEM per layer); back-propagation of ybar to dE/dz;
//                   the L-BFGS / Armijo state machine on a shared-memory copy of
//                   the solver state; hidden forward of the next trial point;
//                   CUDA-graph WHILE condition.
#pragma once

#include <cooperative_groups.h>

#include "lsb_common.cuh"

namespace lsb {

namespace cg = cooperative_groups;

enum Phase : int { kPhaseInit = 0, kPhaseLineSearch = 1, kPhaseFinalDecode = 2, kPhaseDone = 3 };
enum Mode : int { kModeEval = 0, kModeLbfgs = 1 };
enum DevStatus : int { kStOk = 0, kStNonFinite = 2 };
enum CtrlMode : int { kCtrlStart = 0, kCtrlAfterEval = 1 };

struct alignas(16) DevState {  // 16-byte size: staged by one bulk copy, published with 16-byte stores
    // configuration
    int mode, want_grad;
    double eps;
    int max_iters, max_ls, hist_cap;
    // current evaluation
    double f_eval;
    int need_grad, status, accept;
    double zt[kMaxLatent];  // point being evaluated
    double gz[kMaxLatent];  // gradient at zt (when need_grad)
    // L-BFGS (reference reduced_solver.cpp:58-131)
    int phase, done, code, iter, ls, hist_n, hist_head, value_evals, grad_evals;
    double f, gtd, alpha, gnorm;
    double x[kMaxLatent], g[kMaxLatent], d[kMaxLatent];
    double S[kMaxHistory][kMaxLatent], Y[kMaxHistory][kMaxLatent], alph[kMaxHistory], rho[kMaxHistory];
    unsigned long long t_start, t_end;
    int loop_iters;  // WHILE-body executions of the current solve
    // objective parameters (device-resident so captured graphs stay valid)
    double inv_dt2, dt;
    int has_inertia, quasi_static;
    // dynamics bookkeeping
    int step_idx;
    double t;
    void* reports;   // lsb_exit_report[capacity]
    double* z_traj;  // capacity x r
    // last-block counters (self-resetting)
    unsigned int cnt_elem, cnt_top;
};

template <typename TS>
struct EvalParams {
    int n, n_free, V, E, r, nhid, h, hp, out_act;
    int grid_out, grid_elem, grid_vjp, vpb, group, n_groups;
    int w_resident;   // W_out fits in L2: keep it (evict_last) instead of streaming
    int elem_f32;     // fp32-storage mode: element strain / stress / forces in fp32 arithmetic
    int l2_pf_tiles;  // out_fwd: W tiles per CTA bulk-prefetched into L2 before its dependency wait (PDL)
    int l2_pf_elem;   // elem: first W tiles of every VJP CTA range prefetched into L2 (0: off)
    int w_keep_tiles; // out_fwd: the last W tiles of every CTA range stay in L2 (evict_last) for the VJP's re-read
    // output layer (device layout: rows padded to hp columns)
    const TS* Wout;
    const double* bout;
    const double* sout;
    const double* cout;  // shift - X (free DOFs)
    double* dsout;       // s * phi'(a) (non-identity output activation only)
    // inertia
    const double* mass;
    const double* ut;    // qbar - X (free DOFs)
    double* rin;         // m (u - ut) / dt^2
    double* eprow;       // n x 6: {b, s, shift - X, m, U slot, qbar - X} per output row (TMA-staged)
    double* tv;          // n: s phi'(a) g (gathered full-space gradient, VJP input)
    // mesh
    const int* vfree;
    const int4* tets;
    const TS* rec;       // E x 12: Dminv (row-major 9), vol, mu, lambda
    double* U;           // V x 4 displacement (w unused)
    double* forces;      // nnz x 4: per (tet, free slot) force vectors in CSR order (xyz, pad)
    const int* csr_ptr;
    const int* csr_ent;
    const int4* fpos;    // E: CSR position of each tet slot's force (-1 = pinned vertex)
    // hidden layers (fp64)
    const double* Wh;    // row-major, concatenated
    const TS* Wh_s;      // the same in storage precision (solve kernel control cluster)
    const double* bh;
    int hoff[kMaxLayers], boff[kMaxLayers], hrows[kMaxLayers], hcols[kMaxLayers], hact[kMaxLayers];
    double* a_hid;       // nhid x kMaxHidden pre-activations at zt
    double* y_last;      // hp, zero padded
    // partials
    double* e_part_out;
    double* e_part_elem;
    double* ybar_part;   // grid_vjp x hp
    double* ybar_grp;    // n_groups x hp
    unsigned int* grp_cnt;
    DevState* st;
    cudaGraphConditionalHandle cond;
    int in_graph;
    // cluster control layout
    int cs;              // cluster size
    int ctrl_smem_w;     // doubles of staged weights per CTA
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// W_out loads: streamed (evict_first) when larger than L2, else kept resident.
__device__ __forceinline__ F8 ld_w(const F8* p, int resident) {
    if (resident) {
        F8 r;
        asm("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                       "=f"(r.v[6]), "=f"(r.v[7])
                     : "l"(p));
        return r;
    }
    return ld_stream(p);
}
__device__ __forceinline__ D4 ld_w(const D4* p, int resident) {
    if (resident) {
        D4 r;
        asm("ld.global.nc.L2::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
                     : "l"(p));
        return r;
    }
    return ld_stream(p);
}

// ---------------------------------------------------------------- L-BFGS control
// Warp-level state machine on a shared-memory copy of DevState; returns 1 when
// a further evaluation at st->zt is required.  Mirrors reduced_solver.cpp:58-131
// (history index 0 = oldest pair, pop_front when full; rho = y.s cached per pair).
static __device__ int lbfgs_control(DevState* st, int r) {
    const int lane = threadIdx.x & 31;
    if (st->status != kStOk || st->phase == kPhaseFinalDecode) {
        if (lane == 0) st->done = 1;
        __syncwarp();
        return 0;
    }
    bool start_iter = false;
    if (st->phase == kPhaseInit) {
        __syncwarp();
        if (lane == 0) st->f = st->f_eval;
        for (int i = lane; i < r; i += 32) {
            st->x[i] = st->zt[i];
            st->g[i] = st->gz[i];
        }
        start_iter = true;
    } else if (st->accept) {
        double s_i[2], y_i[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int i = lane + 32 * k;
            s_i[k] = i < r ? st->zt[i] - st->x[i] : 0.0;
            y_i[k] = i < r ? st->gz[i] - st->g[i] : 0.0;
        }
        const double sy = warp_sum(s_i[0] * y_i[0] + s_i[1] * y_i[1]);
        const double ss = warp_sum(s_i[0] * s_i[0] + s_i[1] * s_i[1]);
        const double yy = warp_sum(y_i[0] * y_i[0] + y_i[1] * y_i[1]);
        if (sy > 1e-12 * sqrt(ss) * sqrt(yy)) {  // :115-119
            const int slot = st->hist_n < st->hist_cap ? (st->hist_head + st->hist_n) % st->hist_cap : st->hist_head;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int i = lane + 32 * k;
                if (i < r) {
                    st->S[slot][i] = s_i[k];
                    st->Y[slot][i] = y_i[k];
                }
            }
            __syncwarp();
            if (lane == 0) {
                st->rho[slot] = sy;
                if (st->hist_n < st->hist_cap) st->hist_n++;
                else st->hist_head = (st->hist_head + 1) % st->hist_cap;
            }
        }
        __syncwarp();
        for (int i = lane; i < r; i += 32) {
            st->x[i] = st->zt[i];
            st->g[i] = st->gz[i];
        }
        if (lane == 0) {
            st->f = st->f_eval;
            st->iter++;
        }
        start_iter = true;
    } else {  // Armijo rejection: halve (:50-52)
        __syncwarp();
        if (lane == 0) {
            st->alpha *= 0.5;
            st->ls++;
        }
        __syncwarp();
        if (st->ls >= st->max_ls) {  // exit III; re-decode x (U holds the rejected trial)
            for (int i = lane; i < r; i += 32) st->zt[i] = st->x[i];
            __syncwarp();
            if (lane == 0) {
                st->code = 3;
                st->phase = kPhaseFinalDecode;
            }
            __syncwarp();
            return 1;
        }
        const double a = st->alpha;
        for (int i = lane; i < r; i += 32) st->zt[i] = st->x[i] + a * st->d[i];
        __syncwarp();
        return 1;
    }
    __syncwarp();
    if (!start_iter) return 0;
    double gmax = 0.0;
    for (int i = lane; i < r; i += 32) gmax = fmax(gmax, fabs(st->g[i]));
    gmax = warp_max(gmax);
    if (st->iter >= st->max_iters) {  // loop exhausted (:124-130)
        if (lane == 0) {
            st->gnorm = gmax;
            st->code = gmax < st->eps ? 1 : 4;
            st->done = 1;
        }
        __syncwarp();
        return 0;
    }
    if (lane == 0) st->gnorm = gmax;
    if (gmax < st->eps) {  // exit I (:72-79)
        if (lane == 0) {
            st->code = 1;
            st->done = 1;
        }
        __syncwarp();
        return 0;
    }
    // two-loop recursion (:81-96)
    double dv[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) dv[k] = (lane + 32 * k) < r ? -st->g[lane + 32 * k] : 0.0;
    const int H = st->hist_n;
    for (int k = H - 1; k >= 0; --k) {
        const int slot = (st->hist_head + k) % st->hist_cap;
        double sd = 0.0;
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (lane + 32 * q < r) sd += st->S[slot][lane + 32 * q] * dv[q];
        const double al = warp_sum(sd) / st->rho[slot];
        if (lane == 0) st->alph[k] = al;
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (lane + 32 * q < r) dv[q] -= al * st->Y[slot][lane + 32 * q];
    }
    if (H > 0) {
        const int slot = (st->hist_head + H - 1) % st->hist_cap;
        double yy = 0.0;
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (lane + 32 * q < r) yy += st->Y[slot][lane + 32 * q] * st->Y[slot][lane + 32 * q];
        const double gam = st->rho[slot] / warp_sum(yy);
        dv[0] *= gam;
        dv[1] *= gam;
    }
    __syncwarp();
    for (int k = 0; k < H; ++k) {
        const int slot = (st->hist_head + k) % st->hist_cap;
        double yd = 0.0;
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (lane + 32 * q < r) yd += st->Y[slot][lane + 32 * q] * dv[q];
        const double coef = st->alph[k] - warp_sum(yd) / st->rho[slot];
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (lane + 32 * q < r) dv[q] += coef * st->S[slot][lane + 32 * q];
    }
    double gtd = 0.0;
#pragma unroll
    for (int q = 0; q < 2; ++q)
        if (lane + 32 * q < r) gtd += st->g[lane + 32 * q] * dv[q];
    gtd = warp_sum(gtd);
    if (!(gtd < 0.0)) {  // exit II (:98-102)
        if (lane == 0) {
            st->code = 2;
            st->done = 1;
        }
        __syncwarp();
        return 0;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int i = lane + 32 * q;
        if (i < r) {
            st->d[i] = dv[q];
            st->zt[i] = st->x[i] + dv[q];  // alpha = 1
        }
    }
    if (lane == 0) {
        st->gtd = gtd;
        st->alpha = 1.0;
        st->ls = 0;
        st->phase = kPhaseLineSearch;
    }
    __syncwarp();
    return 1;
}

// Bulk L2 prefetch of the first `tiles` W_out tiles of every CTA range of a streaming kernel
// with `grid` CTAs (ranges [ntiles k / grid, ntiles (k+1) / grid)), spread over the lane-0s of
// the calling grid's warps.  Issued from a latency-bound phase (element pass, control kernel)
// so the next streaming kernel starts on L2-resident tiles.
template <typename TS>
__device__ __forceinline__ void prefetch_stream_heads(const EvalParams<TS>& p, int grid, int tiles) {
    if (tiles <= 0 || grid <= 0 || (threadIdx.x & 31) != 0) return;
    const int rowb = p.hp * (int)sizeof(TS);
    const int tr = 8192 / rowb < 8 ? 8 : 8192 / rowb;
    const int ntiles = (p.n + tr - 1) / tr;
    const int nw = blockDim.x >> 5;
    const int gw = (int)(blockIdx.x * nw + (threadIdx.x >> 5)), tw = (int)(gridDim.x * nw);
    const uint64_t pol = l2_policy(1);
    for (int k = gw; k < grid; k += tw) {
        const int t0 = (int)(((long long)ntiles * k) / grid), t1 = (int)(((long long)ntiles * (k + 1)) / grid);
        const int te = min(t1, t0 + tiles);
        if (te <= t0) continue;
        const char* a = reinterpret_cast<const char*>(p.Wout + (size_t)t0 * tr * p.hp);
        const size_t bytes = (size_t)(min(te * tr, p.n) - t0 * tr) * rowb;
        for (size_t o = 0; o < bytes; o += 65536) {
            const unsigned nb = (unsigned)((bytes - o) < 65536 ? (bytes - o) : 65536);
            asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(a + o), "r"(nb),
                         "l"(pol)
                         : "memory");
        }
    }
}

// ---------------------------------------------------------------- K3: element pass
template <typename TS>
__device__ __forceinline__ void load_rec(const TS* rec, size_t e, double* out12);
template <>
__device__ __forceinline__ void load_rec<float>(const float* rec, size_t e, double* o) {
    const float4* p = reinterpret_cast<const float4*>(rec + e * 12);
    const float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
    o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
    o[8] = c.x; o[9] = c.y; o[10] = c.z; o[11] = c.w;
}
template <>
__device__ __forceinline__ void load_rec<double>(const double* rec, size_t e, double* o) {
    // three 256-bit read-only loads of the 96-byte record
    const double* p = rec + e * 12;
#pragma unroll
    for (int k = 0; k < 3; ++k)
        asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
            : "=d"(o[4 * k]), "=d"(o[4 * k + 1]), "=d"(o[4 * k + 2]), "=d"(o[4 * k + 3])
            : "l"(p + 4 * k));
}
__device__ __forceinline__ void load_u(const double* U, int v, double* o) {
    const double2 a = *reinterpret_cast<const double2*>(U + (size_t)v * 4);
    o[0] = a.x;
    o[1] = a.y;
    o[2] = U[(size_t)v * 4 + 2];
}

// Energy and 12 local forces of one tet from vertex displacements.
// A = (Ds - Ds_rest) Dm^-1 (reference element_frame, energy.cpp:163-175);
// forces = vol P Dm^-T (= vol B^T vec(P), energy.cpp:290-291).
template <typename T>
__device__ __forceinline__ T tet_energy_forces_t(const T* u0, const T* u1, const T* u2, const T* u3, const T* rec,
                                                 T* f) {
    T D[9];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        D[a * 3 + 0] = u1[a] - u0[a];
        D[a * 3 + 1] = u2[a] - u0[a];
        D[a * 3 + 2] = u3[a] - u0[a];
    }
    T A[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            A[a * 3 + b] = D[a * 3 + 0] * rec[0 * 3 + b] + D[a * 3 + 1] * rec[1 * 3 + b] + D[a * 3 + 2] * rec[2 * 3 + b];
    T P[9];
    const T vol = rec[9];
    const T psi = snh_psi_P(A, rec[10], rec[11], P);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        T s0 = 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const T hv =
                vol * (P[a * 3 + 0] * rec[c * 3 + 0] + P[a * 3 + 1] * rec[c * 3 + 1] + P[a * 3 + 2] * rec[c * 3 + 2]);
            f[(c + 1) * 3 + a] = hv;
            s0 += hv;
        }
        f[a] = -s0;
    }
    return vol * psi;
}
__device__ __forceinline__ double tet_energy_forces(const double* u0, const double* u1, const double* u2,
                                                    const double* u3, const double* rec, double* f) {
    return tet_energy_forces_t<double>(u0, u1, u2, u3, rec, f);
}

// fp32-storage mode (TS = float): the edge differences of the fp64 displacements are formed in
// fp64 (no cancellation is introduced by rounding u itself), then the strain, the SNH density
// and stress and the 12 forces run in fp32 -- the forces are stored as fp32 CSR entries anyway,
// and the element energy is returned in fp64 for the fp64 block sums.  Relative error ~1e-7 per
// tet, far inside the fp32 mode's 1e-4 bar and uncorrelated between tets.
__device__ __forceinline__ double tet_energy_forces_f32(const double* u0, const double* u1, const double* u2,
                                                        const double* u3, const float* rc, float* f) {
    float D[9];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        D[a * 3 + 0] = (float)(u1[a] - u0[a]);
        D[a * 3 + 1] = (float)(u2[a] - u0[a]);
        D[a * 3 + 2] = (float)(u3[a] - u0[a]);
    }
    float A[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            A[a * 3 + b] = D[a * 3 + 0] * rc[0 * 3 + b] + D[a * 3 + 1] * rc[1 * 3 + b] + D[a * 3 + 2] * rc[2 * 3 + b];
    float P[9];
    const float vol = rc[9];
    const float psi = snh_psi_P(A, rc[10], rc[11], P);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float s0 = 0.f;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float hv =
                vol * (P[a * 3 + 0] * rc[c * 3 + 0] + P[a * 3 + 1] * rc[c * 3 + 1] + P[a * 3 + 2] * rc[c * 3 + 2]);
            f[(c + 1) * 3 + a] = hv;
            s0 += hv;
        }
        f[a] = -s0;
    }
    return (double)vol * (double)psi;
}
__device__ __forceinline__ void load_rec_f(const float* rec, size_t e, float* o) {
    const float4* p = reinterpret_cast<const float4*>(rec + e * 12);
    const float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
    o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
    o[8] = c.x; o[9] = c.y; o[10] = c.z; o[11] = c.w;
}
// The CSR force entries are re-read by the vertex gather right after the element pass, while
// the W_out stream (evict_first) passes through L2: store them with an evict_last hint.
__device__ __forceinline__ void store_forces_csr_f(double* F, int4 pos, const float* f) {
    float* Ff = reinterpret_cast<float*>(F);
    const int ps[4] = {pos.x, pos.y, pos.z, pos.w};
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (ps[k] >= 0)
            asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(Ff + (size_t)ps[k] * 4),
                         "f"(f[3 * k]), "f"(f[3 * k + 1]), "f"(f[3 * k + 2]), "f"(0.f), "l"(pol)
                         : "memory");
}

// One tet of the element pass: energy, forces to the CSR slots (fp32 arithmetic for TS = float
// when f32 is set, else fp64).
template <typename TS>
__device__ __forceinline__ double elem_tet(const TS* rec, size_t e, const double (&u)[4][3], int4 fpos, double* F,
                                           int f32);

// Scatter one tet's 12 local forces to their vertices' CSR slots: 32-byte {fx, fy, fz, 0}
// double entries, or in fp32-storage mode (TS = float) 16-byte float entries -- the force
// array is a bandwidth-bound intermediate like W_out and the element records;
// the gather sums them in fp64.
template <typename TS>
__device__ __forceinline__ void store_forces_csr_t(double* F, int4 pos, const double* f);
template <>
__device__ __forceinline__ void store_forces_csr_t<float>(double* F, int4 pos, const double* f) {
    float* Ff = reinterpret_cast<float*>(F);
    const int ps[4] = {pos.x, pos.y, pos.z, pos.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (ps[k] >= 0)
            __stcg(reinterpret_cast<float4*>(Ff + (size_t)ps[k] * 4),
                   make_float4((float)f[3 * k], (float)f[3 * k + 1], (float)f[3 * k + 2], 0.f));
}
__device__ __forceinline__ void store_forces_csr(double* F, int4 pos, const double* f) {
    const int ps[4] = {pos.x, pos.y, pos.z, pos.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (ps[k] >= 0) {
            // one 256-bit store of the 32-byte entry {fx, fy, fz, 0}
            asm volatile("st.global.cg.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(F + (size_t)ps[k] * 4), "d"(f[3 * k]),
                         "d"(f[3 * k + 1]), "d"(f[3 * k + 2]), "d"(0.0)
                         : "memory");
        }
}
template <>
__device__ __forceinline__ void store_forces_csr_t<double>(double* F, int4 pos, const double* f) {
    store_forces_csr(F, pos, f);
}
template <>
__device__ __forceinline__ double elem_tet<double>(const double* rec, size_t e, const double (&u)[4][3], int4 fpos,
                                                   double* F, int) {
    double rc[12], f[12];
    load_rec<double>(rec, e, rc);
    const double en = tet_energy_forces(u[0], u[1], u[2], u[3], rc, f);
    store_forces_csr(F, fpos, f);
    return en;
}
template <>
__device__ __forceinline__ double elem_tet<float>(const float* rec, size_t e, const double (&u)[4][3], int4 fpos,
                                                  double* F, int f32) {
    if (f32) {
        float rc[12], f[12];
        load_rec_f(rec, e, rc);
        const double en = tet_energy_forces_f32(u[0], u[1], u[2], u[3], rc, f);
        store_forces_csr_f(F, fpos, f);
        return en;
    }
    double rc[12], f[12];
    load_rec<float>(rec, e, rc);
    const double en = tet_energy_forces(u[0], u[1], u[2], u[3], rc, f);
    store_forces_csr_t<float>(F, fpos, f);
    return en;
}

// fp32 element arithmetic (config 3): 63 registers, four blocks per SM, one tet in flight per thread
// (measured 209.5 us per evaluation against 210.8 with three blocks x two tets); the fp64 forms keep
// two tets in flight at the compiler's register count (forcing more blocks per SM spills them).
template <typename TS, int F32 = 0>
__global__ void __launch_bounds__(256, (F32 && sizeof(TS) == 4) ? 4 : 2) elem_kernel(const EvalParams<TS> p) {
    __shared__ double red[32];
    __shared__ int am_last;
    DevState* st = p.st;
    prefetch_stream_heads(p, p.grid_vjp, p.l2_pf_elem);  // the VJP's first tiles, while tets are latency-bound
    griddep_wait();
    griddep_launch();
    double eacc = 0.0;
    constexpr int NT = (F32 && sizeof(TS) == 4) ? 1 : 2;  // tets in flight per thread
    const int stride = gridDim.x * blockDim.x;
    for (int e0 = blockIdx.x * blockDim.x + threadIdx.x; e0 < p.E; e0 += NT * stride) {
        // NT tets in flight per thread: indices first, then all gathers
        int4 t[NT];
#pragma unroll
        for (int q = 0; q < NT; ++q) t[q] = e0 + q * stride < p.E ? __ldg(p.tets + e0 + q * stride) : make_int4(0, 0, 0, 0);
        double u[NT][4][3];
#pragma unroll
        for (int q = 0; q < NT; ++q) {
            load_u(p.U, t[q].x, u[q][0]);
            load_u(p.U, t[q].y, u[q][1]);
            load_u(p.U, t[q].z, u[q][2]);
            load_u(p.U, t[q].w, u[q][3]);
        }
#pragma unroll
        for (int q = 0; q < NT; ++q) {
            const int e = e0 + q * stride;
            if (e >= p.E) break;
            eacc += elem_tet<TS>(p.rec, (size_t)e, u[q], __ldg(p.fpos + e), p.forces, F32);
        }
    }
    const double tot = block_sum(eacc, red);
    if (threadIdx.x == 0) {
        p.e_part_elem[blockIdx.x] = tot;
        __threadfence();
        const unsigned prev = atomicAdd(&st->cnt_elem, 1u);
        am_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    // Deterministic total: inertia partials then element partials, block order.
    double s = 0.0;
    for (int b = threadIdx.x; b < p.grid_out; b += blockDim.x) s += p.e_part_out[b];
    const double e_in = block_sum(s, red);
    s = 0.0;
    for (int b = threadIdx.x; b < p.grid_elem; b += blockDim.x) s += p.e_part_elem[b];
    const double e_el = block_sum(s, red);
    if (threadIdx.x == 0) {
        st->cnt_elem = 0;
        const bool skip = st->phase == kPhaseFinalDecode;
        const double E = e_el + (st->has_inertia ? e_in : 0.0);
        st->f_eval = E;
        if (!skip) st->value_evals++;
        int need = 0;
        if (skip) {
            need = 0;
        } else if (!isfinite(E)) {  // reduced_solver.cpp:198-199 (throws)
            st->status = kStNonFinite;
        } else if (st->mode == kModeEval) {
            need = st->want_grad;
        } else if (st->phase == kPhaseInit) {
            need = 1;
        } else {  // Armijo test (reduced_solver.cpp:49)
            const int acc = E <= st->f + 1e-4 * st->alpha * st->gtd;
            st->accept = acc;
            need = acc;
        }
        st->need_grad = need;
        if (need) st->grad_evals++;
    }
}

// cp.async staging of count elements of TS (doubles: stage_doubles; floats: 16-byte granules
// when both ends are 16-byte aligned, else 4-byte granules)
template <typename TS>
__device__ __forceinline__ void stage_ts(TS* dst, const TS* src, int count);
template <>
__device__ __forceinline__ void stage_ts<double>(double* dst, const double* src, int count) {
    stage_doubles(dst, src, count);
}
template <>
__device__ __forceinline__ void stage_ts<float>(float* dst, const float* src, int count) {
    const uintptr_t sa = reinterpret_cast<uintptr_t>(src), da = reinterpret_cast<uintptr_t>(dst);
    if (((sa | da) & 15u) == 0) {
        const int body = count / 4;
        for (int k = threadIdx.x; k < body; k += blockDim.x) cp_async16(dst + 4 * k, src + 4 * k);
        for (int k = 4 * body + threadIdx.x; k < count; k += blockDim.x) cp_async4(dst + k, src + k);
    } else {
        for (int k = threadIdx.x; k < count; k += blockDim.x) cp_async4(dst + k, src + k);
    }
}

// ---------------------------------------------------------------- K5/K6: cluster control
// Row partition of a layer with R rows over CS CTAs.
__device__ __forceinline__ int part_lo(int R, int cs, int c) { return (int)(((long long)R * c) / cs); }

// Shared-memory layout of one CTA (doubles): [staged W row slices of every
// hidden layer][ybuf kMaxHidden][slice0 64][slice1 64][part0 kMaxHidden]
// [part1 kMaxHidden][bias slices kMaxLayers*64][a slices kMaxLayers*64][DevState copy].
template <typename TS, int CS>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(256) ctrl_kernel(const EvalParams<TS> p, int cmode,
                                                                              int start_mode, int start_want_grad) {
    extern __shared__ __align__(16) double csm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int c = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nw = blockDim.x >> 5;
    TS* wsl = reinterpret_cast<TS*>(csm);               // staged weight slices (storage precision)
    double* ybuf = csm + p.ctrl_smem_w;                 // kMaxHidden
    // pointer selects rather than runtime-indexed pointer arrays: no local memory (every
    // cluster barrier invalidates L1)
    double* const slice0 = ybuf + kMaxHidden;
    double* const part0 = ybuf + kMaxHidden + 128;
    double* const part1 = ybuf + 2 * kMaxHidden + 128;
    double* bsl = ybuf + 3 * kMaxHidden + 128;          // bias slices (kMaxLayers * 64)
    double* asl = bsl + kMaxLayers * 64;                // pre-activation slices (kMaxLayers * 64)
    DevState* sst = reinterpret_cast<DevState*>(asl + kMaxLayers * 64);
    __shared__ int more_s;
    griddep_wait();
    griddep_launch();
    const int need = cmode == kCtrlAfterEval ? p.st->need_grad : 0;

    // 0. stage own row slices of every hidden layer, biases, pre-activations and
    //    (CTA 0) the solver state into shared memory: all copies in flight at once
    __shared__ int woff[kMaxLayers];
    {
        int off = 0;
        for (int l = 0; l < p.nhid; ++l) {
            const int R = p.hrows[l], C = p.hcols[l];
            const int i0 = part_lo(R, CS, c), i1 = part_lo(R, CS, c + 1);
            if (tid == 0) woff[l] = off;
            stage_ts(wsl + off, p.Wh_s + p.hoff[l] + (size_t)i0 * C, (i1 - i0) * C);
            stage_doubles(bsl + l * 64, p.bh + p.boff[l] + i0, i1 - i0);
            if (need) stage_doubles(asl + l * 64, p.a_hid + l * kMaxHidden + i0, i1 - i0);
            off += ((i1 - i0) * C + 3) & ~3;
        }
    }
    if (c == 0) stage_doubles(reinterpret_cast<double*>(sst), reinterpret_cast<const double*>(p.st),
                              (int)(sizeof(DevState) / sizeof(double)));
    cp_async_wait_all();
    __syncthreads();

    int more = 1;
    if (cmode == kCtrlAfterEval) {
        if (need && p.nhid > 0) {
            // ---- ybar of the last hidden layer, own row slice: sum of group partials
            const int Rl = p.hrows[p.nhid - 1];
            const int j0 = part_lo(Rl, CS, c), j1 = part_lo(Rl, CS, c + 1);
            for (int j = j0 + tid; j < j1; j += blockDim.x) {
                double s = 0.0;
#pragma unroll 8
                for (int b = 0; b < p.n_groups; ++b) s += __ldcg(p.ybar_grp + (size_t)b * p.hp + j);
                slice0[j - j0] = s;
            }
            __syncthreads();
            // ---- backward through hidden layers (transpose of decode_jacobian, net.cpp:159-190)
            for (int l = p.nhid - 1; l >= 0; --l) {
                const int R = p.hrows[l], C = p.hcols[l];
                const int i0 = part_lo(R, CS, c), i1 = part_lo(R, CS, c + 1);
                double* pt = (l & 1) ? part1 : part0;
                for (int i = tid; i < i1 - i0; i += blockDim.x) slice0[i] *= act_eval(p.hact[l], asl[l * 64 + i], 1);
                __syncthreads();
                // partial W^T abar over own rows, all C columns (4 independent chains)
                const TS* Ws = wsl + woff[l];
                const int nr = i1 - i0;
                for (int j = tid; j < C; j += blockDim.x) {
                    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                    int i = 0;
                    for (; i + 4 <= nr; i += 4) {
                        s0 = fma((double)Ws[i * C + j], slice0[i], s0);
                        s1 = fma((double)Ws[(i + 1) * C + j], slice0[i + 1], s1);
                        s2 = fma((double)Ws[(i + 2) * C + j], slice0[i + 2], s2);
                        s3 = fma((double)Ws[(i + 3) * C + j], slice0[i + 3], s3);
                    }
                    for (; i < nr; ++i) s0 = fma((double)Ws[i * C + j], slice0[i], s0);
                    pt[j] = (s0 + s1) + (s2 + s3);
                }
                cluster.sync();
                // own slice of the previous layer's ybar: sum the CS partials in rank order
                if (l > 0) {
                    const int Rp = p.hrows[l - 1];
                    const int k0 = part_lo(Rp, CS, c), k1 = part_lo(Rp, CS, c + 1);
                    for (int j = k0 + tid; j < k1; j += blockDim.x) {
                        double s = 0.0;
                        for (int q = 0; q < CS; ++q) s += cluster.map_shared_rank(pt, q)[j];
                        slice0[j - k0] = s;
                    }
                } else if (c == 0) {
                    for (int j = tid; j < C; j += blockDim.x) {
                        double s = 0.0;
                        for (int q = 0; q < CS; ++q) s += cluster.map_shared_rank(pt, q)[j];
                        sst->gz[j] = s;
                    }
                }
                __syncthreads();
            }
        } else if (need && c == 0) {  // linear decoder: ybar is the gradient
            for (int j = tid; j < p.r; j += blockDim.x) {
                double s = 0.0;
#pragma unroll 8
                for (int b = 0; b < p.n_groups; ++b) s += __ldcg(p.ybar_grp + (size_t)b * p.hp + j);
                sst->gz[j] = s;
            }
        }
        __syncthreads();
        // ---- L-BFGS / eval bookkeeping (CTA 0, warp 0)
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
    } else {  // kCtrlStart: fresh evaluation / solve at st->zt
        if (c == 0 && tid == 0) {
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
        __syncthreads();
    }
    // broadcast `more` and zt from CTA 0 (DSMEM) after the barrier
    if (c == 0 && tid == 0) more_s = more;
    cluster.sync();
    more = *cluster.map_shared_rank(&more_s, 0);
    if (more) {
        // ---- hidden forward at zt (reference mlp_forward, net.cpp:134-142); the owner of each
        // output row pushes it into every CTA's next input buffer (part0/part1), one cluster
        // barrier per layer
        const double* zsrc = cluster.map_shared_rank(sst->zt, 0);
        for (int j = tid; j < p.r; j += blockDim.x) part0[j] = zsrc[j];
        __syncthreads();
        for (int l = 0; l < p.nhid; ++l) {
            const int R = p.hrows[l], C = p.hcols[l];
            const int i0 = part_lo(R, CS, c), i1 = part_lo(R, CS, c + 1);
            const double* x = (l & 1) ? part1 : part0;
            double* xn = (l & 1) ? part0 : part1;
            const TS* Ws = wsl + woff[l];
            for (int i = warp; i < i1 - i0; i += nw) {
                double s = 0.0;
                for (int j = lane; j < C; j += 32) s = fma((double)Ws[i * C + j], x[j], s);
                s = warp_sum(s);
                const double a = s + bsl[l * 64 + i];
                const double y = act_eval(p.hact[l], a, 0);
                if (lane < CS) cluster.map_shared_rank(xn, lane)[i0 + i] = y;
                if (lane == 0) p.a_hid[l * kMaxHidden + i0 + i] = a;
            }
            cluster.sync();
        }
        const double* ylast = (p.nhid & 1) ? part1 : part0;
        if (c == 0) {
            const int h = p.nhid > 0 ? p.hrows[p.nhid - 1] : p.r;
            for (int j = tid; j < p.hp; j += blockDim.x) p.y_last[j] = j < h ? ylast[j] : 0.0;
        }
    }
    // CTA 0 publishes the solver state and sets the WHILE condition
    if (c == 0) {
        __syncthreads();
        const int nwords = sizeof(DevState) / 4;
        int* dst = reinterpret_cast<int*>(p.st);
        const int* src = reinterpret_cast<const int*>(sst);
        for (int k = tid; k < nwords; k += blockDim.x) dst[k] = src[k];
        if (tid == 0 && p.in_graph) cudaGraphSetConditional(p.cond, more ? 1u : 0u);
    }
    cluster.sync();  // keep shared memory alive until all remote reads are done
}

}  // namespace lsb
