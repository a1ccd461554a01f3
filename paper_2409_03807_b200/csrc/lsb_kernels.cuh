// Single-instance E(z) + grad E(z) kernels and the device-resident L-BFGS
// control (SURVEY §2.2 kernels K1..K6).
//
// One objective evaluation at the latent point st->zt is three kernels:
//   out_fwd   (K2)  stream W_out (n x h, row-major, 16-byte vector loads) against
//                   the last hidden activation y: u = s*phi(W y + b) + (shift - X);
//                   scatter u into the vertex displacement array U; inertia
//                   residual r = m (u - ut) / dt^2 and its energy partials.
//   elem      (K3)  per tet: gather 4 vertex displacements, A = dU Dm^-1,
//                   cancellation-free stable neo-Hookean psi and P, 12 local forces
//                   vol P Dm^-T into a per-tet buffer; energy partials.  The last
//                   block sums all energy partials in block order (deterministic)
//                   and makes the Armijo accept decision.
//   vjp_ctrl  (K3b+K4+K5+K6) only when the gradient is needed: per free vertex
//                   CSR gather of the per-tet forces in ascending tet order (the
//                   scatter order of the reference assemble) + inertia, times s;
//                   second stream of W_out accumulating ybar = W_out^T (s g) in
//                   registers; deterministic two-level block reduction; the last
//                   block back-propagates ybar through the hidden layers (fp64),
//                   runs the L-BFGS/Armijo state machine and the hidden forward of
//                   the next trial point, and sets the CUDA-graph WHILE condition.
#pragma once

#include "lsb_common.cuh"

namespace lsb {

enum Phase : int { kPhaseInit = 0, kPhaseLineSearch = 1, kPhaseFinalDecode = 2, kPhaseDone = 3 };
enum Mode : int { kModeEval = 0, kModeLbfgs = 1 };
enum DevStatus : int { kStOk = 0, kStNonFinite = 2 };

struct DevState {
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
    double S[kMaxHistory][kMaxLatent], Y[kMaxHistory][kMaxLatent], alph[kMaxHistory];
    unsigned long long t_start, t_end;
    int loop_iters;      // WHILE-body executions of the current solve
    // objective parameters (device-resident so captured graphs stay valid)
    double inv_dt2, dt;
    int has_inertia, quasi_static;
    // dynamics bookkeeping
    int step_idx;
    double t;
    void* reports;       // lsb_exit_report[capacity]
    double* z_traj;      // capacity x r (nullable)
    // last-block counters (self-resetting)
    unsigned int cnt_elem, cnt_top;
};

template <typename T>
struct EvalParams {
    int n, n_free, V, E, r, nhid, h, hp, out_act;
    int grid_out, grid_elem, grid_vjp, vpb, group, n_groups;
    // output layer (device layout: rows padded to hp columns)
    const T* Wout;
    const T* bout;
    const T* sout;
    const T* cout;  // shift - X (free DOFs)
    T* dsout;       // s * phi'(a) (non-identity output activation only)
    // inertia
    const T* mass;
    const T* ut;    // qbar - X (free DOFs)
    T* rin;         // m (u - ut) / dt^2
    // mesh
    const int* vfree;
    const int4* tets;
    const T* rec;   // E x 12: Dminv (row-major 9), vol, mu, lambda
    T* U;           // V x 4 displacement (w unused)
    T* forces;      // E x 12: local vertex forces (slot-major, xyz)
    const int* csr_ptr;
    const int* csr_ent;
    // hidden layers (fp64)
    const double* Wh;   // row-major, concatenated
    const double* WhT;  // transposed, concatenated
    const double* bh;
    int hoff[kMaxLayers], boff[kMaxLayers], hrows[kMaxLayers], hcols[kMaxLayers], hact[kMaxLayers];
    double* a_hid;      // nhid x kMaxHidden pre-activations at zt
    T* y_last;          // hp, zero padded
    // partials
    double* e_part_out;
    double* e_part_elem;
    double* ybar_part;  // grid_vjp x hp
    double* ybar_grp;   // n_groups x hp
    unsigned int* grp_cnt;
    DevState* st;
    cudaGraphConditionalHandle cond;
    int in_graph;
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------- hidden MLP (fp64, one block)
// Forward of the hidden layers at st->zt (reference mlp_forward, net.cpp:134-142),
// saving pre-activations for the backward pass.  smem: 2 * kMaxHidden doubles.
template <typename T>
__device__ void hidden_forward(const EvalParams<T>& p, double* smem) {
    DevState* st = p.st;
    double* ycur = smem;
    double* ynext = smem + kMaxHidden;
    for (int i = threadIdx.x; i < p.r; i += blockDim.x) ycur[i] = st->zt[i];
    __syncthreads();
    for (int l = 0; l < p.nhid; ++l) {
        const int R = p.hrows[l], C = p.hcols[l];
        const double* WT = p.WhT + p.hoff[l];
        const double* b = p.bh + p.boff[l];
        // TPR threads per row split the column sum; combined in fixed lane order.
        int tpr = 1;
        while (tpr * 2 * R <= (int)blockDim.x && tpr < 32) tpr *= 2;
        const int rows_per_pass = blockDim.x / tpr;
        for (int base = 0; base < R; base += rows_per_pass) {
            const int i = base + threadIdx.x / tpr;
            const int part = threadIdx.x % tpr;
            double acc = 0.0;
            if (i < R)
                for (int j = part; j < C; j += tpr) acc = fma(WT[(size_t)j * R + i], ycur[j], acc);
            for (int o = tpr >> 1; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o, tpr);
            if (i < R && part == 0) {
                const double a = acc + b[i];
                p.a_hid[l * kMaxHidden + i] = a;
                ynext[i] = act_eval(p.hact[l], a, 0);
            }
        }
        __syncthreads();
        double* t = ycur;
        ycur = ynext;
        ynext = t;
    }
    const int h = p.nhid > 0 ? p.hrows[p.nhid - 1] : p.r;
    for (int j = threadIdx.x; j < p.hp; j += blockDim.x) p.y_last[j] = j < h ? (T)ycur[j] : (T)0;
    __syncthreads();
}

// Backward through the hidden layers: ybar (smem, length h) -> gz = dE/dz.
template <typename T>
__device__ void hidden_backward(const EvalParams<T>& p, double* ybar, double* tmp) {
    for (int l = p.nhid - 1; l >= 0; --l) {
        const int R = p.hrows[l], C = p.hcols[l];
        const double* W = p.Wh + p.hoff[l];
        for (int i = threadIdx.x; i < R; i += blockDim.x)
            tmp[i] = ybar[i] * act_eval(p.hact[l], p.a_hid[l * kMaxHidden + i], 1);
        __syncthreads();
        int tpr = 1;
        while (tpr * 2 * C <= (int)blockDim.x && tpr < 32) tpr *= 2;
        const int cols_per_pass = blockDim.x / tpr;
        for (int base = 0; base < C; base += cols_per_pass) {
            const int j = base + threadIdx.x / tpr;
            const int part = threadIdx.x % tpr;
            double acc = 0.0;
            if (j < C)
                for (int i = part; i < R; i += tpr) acc = fma(W[(size_t)i * C + j], tmp[i], acc);
            for (int o = tpr >> 1; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o, tpr);
            __syncthreads();  // all reads of ybar (via tmp) done before overwrite below
            if (j < C && part == 0) ybar[j] = acc;
        }
        __syncthreads();
    }
    for (int j = threadIdx.x; j < p.r; j += blockDim.x) p.st->gz[j] = ybar[j];
    __syncthreads();
}

// ---------------------------------------------------------------- L-BFGS control (warp 0)
// Warp-parallel dot over the latent dimension (r <= 64: two components per lane).
__device__ __forceinline__ double wdot(const double* a, const double* b, int r) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int i = lane; i < r; i += 32) s = fma(a[i], b[i], s);
    return warp_sum(s);
}

// Executed by warp 0 of the control block after an evaluation; returns 1 when a
// further evaluation at st->zt is required.  Mirrors reduced_solver.cpp:58-131.
static __device__ int lbfgs_control(DevState* st, int r) {
    const int lane = threadIdx.x & 31;
    if (st->status != kStOk) {
        st->done = 1;
        return 0;
    }
    if (st->phase == kPhaseFinalDecode) {
        st->done = 1;
        return 0;
    }
    bool start_iter = false;
    if (st->phase == kPhaseInit) {
        if (lane == 0) st->f = st->f_eval;
        for (int i = lane; i < r; i += 32) {
            st->x[i] = st->zt[i];
            st->g[i] = st->gz[i];
        }
        start_iter = true;
    } else {  // line search result at zt = x + alpha d
        if (st->accept) {
            // curvature pair s = trial - x, y = g_new - g (:113-119)
            double s_i[2], y_i[2];
            for (int k = 0, i = lane; k < 2; ++k, i += 32) {
                s_i[k] = i < r ? st->zt[i] - st->x[i] : 0.0;
                y_i[k] = i < r ? st->gz[i] - st->g[i] : 0.0;
            }
            const double sy = warp_sum(s_i[0] * y_i[0] + s_i[1] * y_i[1]);
            const double ss = warp_sum(s_i[0] * s_i[0] + s_i[1] * s_i[1]);
            const double yy = warp_sum(y_i[0] * y_i[0] + y_i[1] * y_i[1]);
            if (sy > 1e-12 * sqrt(ss) * sqrt(yy)) {
                int slot;
                if (st->hist_n < st->hist_cap) {
                    slot = (st->hist_head + st->hist_n) % st->hist_cap;
                } else {  // pop_front then push_back
                    slot = st->hist_head;
                }
                for (int k = 0, i = lane; k < 2; ++k, i += 32)
                    if (i < r) {
                        st->S[slot][i] = s_i[k];
                        st->Y[slot][i] = y_i[k];
                    }
                __syncwarp();
                if (lane == 0) {
                    if (st->hist_n < st->hist_cap) st->hist_n++;
                    else st->hist_head = (st->hist_head + 1) % st->hist_cap;
                }
            }
            for (int i = lane; i < r; i += 32) {
                st->x[i] = st->zt[i];
                st->g[i] = st->gz[i];
            }
            if (lane == 0) {
                st->f = st->f_eval;
                st->iter++;
            }
            start_iter = true;
        } else {
            if (lane == 0) {
                st->alpha *= 0.5;
                st->ls++;
            }
            __syncwarp();
            if (st->ls >= st->max_ls) {  // exit III, then re-decode x (u buffer holds the trial)
                if (lane == 0) {
                    st->code = 3;
                    st->phase = kPhaseFinalDecode;
                }
                for (int i = lane; i < r; i += 32) st->zt[i] = st->x[i];
                __syncwarp();
                return 1;
            }
            const double a = st->alpha;
            for (int i = lane; i < r; i += 32) st->zt[i] = st->x[i] + a * st->d[i];
            __syncwarp();
            return 1;
        }
    }
    __syncwarp();
    if (start_iter) {
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
        // two-loop recursion (:81-96); history index 0 = oldest
        double dv[2];
        for (int k = 0, i = lane; k < 2; ++k, i += 32) dv[k] = i < r ? -st->g[i] : 0.0;
        const int H = st->hist_n;
        for (int k = H - 1; k >= 0; --k) {
            const int slot = (st->hist_head + k) % st->hist_cap;
            const double* s = st->S[slot];
            const double* y = st->Y[slot];
            double sd = 0.0, ys = 0.0;
            for (int q = 0, i = lane; q < 2; ++q, i += 32)
                if (i < r) {
                    sd += s[i] * dv[q];
                    ys += y[i] * s[i];
                }
            sd = warp_sum(sd);
            ys = warp_sum(ys);
            const double al = sd / ys;
            if (lane == 0) st->alph[k] = al;
            for (int q = 0, i = lane; q < 2; ++q, i += 32)
                if (i < r) dv[q] -= al * y[i];
        }
        if (H > 0) {
            const int slot = (st->hist_head + H - 1) % st->hist_cap;
            const double* s = st->S[slot];
            const double* y = st->Y[slot];
            double sy = 0.0, yy = 0.0;
            for (int q = 0, i = lane; q < 2; ++q, i += 32)
                if (i < r) {
                    sy += s[i] * y[i];
                    yy += y[i] * y[i];
                }
            sy = warp_sum(sy);
            yy = warp_sum(yy);
            const double gam = sy / yy;
            dv[0] *= gam;
            dv[1] *= gam;
        }
        __syncwarp();
        for (int k = 0; k < H; ++k) {
            const int slot = (st->hist_head + k) % st->hist_cap;
            const double* s = st->S[slot];
            const double* y = st->Y[slot];
            double yd = 0.0, ys = 0.0;
            for (int q = 0, i = lane; q < 2; ++q, i += 32)
                if (i < r) {
                    yd += y[i] * dv[q];
                    ys += y[i] * s[i];
                }
            yd = warp_sum(yd);
            ys = warp_sum(ys);
            const double beta = yd / ys;
            const double coef = st->alph[k] - beta;
            for (int q = 0, i = lane; q < 2; ++q, i += 32)
                if (i < r) dv[q] += coef * s[i];
        }
        double gtd = 0.0;
        for (int q = 0, i = lane; q < 2; ++q, i += 32)
            if (i < r) gtd += st->g[i] * dv[q];
        gtd = warp_sum(gtd);
        if (!(gtd < 0.0)) {  // exit II (:98-102)
            if (lane == 0) {
                st->code = 2;
                st->done = 1;
            }
            __syncwarp();
            return 0;
        }
        for (int q = 0, i = lane; q < 2; ++q, i += 32)
            if (i < r) {
                st->d[i] = dv[q];
                st->zt[i] = st->x[i] + dv[q];  // alpha = 1
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
    return 0;
}

// ---------------------------------------------------------------- K2: output layer forward
// Lanes-per-row LPR = min(32, hp/VEC); each lane owns NVL 16-byte vectors of y
// and of every row it touches.  UNR row-steps are loaded before use.
template <typename T, int HP>
__global__ void __launch_bounds__(256) out_fwd_kernel(const EvalParams<T> p) {
    using V = typename VecT<T>::type;
    constexpr int VEC = VecT<T>::N;
    constexpr int NVR = HP / VEC;
    constexpr int LPR = NVR < 32 ? NVR : 32;
    constexpr int NVL = NVR / LPR;
    constexpr int RPW = 32 / LPR;
    constexpr int UNR = NVL >= 4 ? 1 : (NVL == 2 ? 2 : 4);
    __shared__ double red[32];
    if (p.st->phase == kPhaseDone) return;
    const int lane = threadIdx.x & 31;
    const int sub = lane / LPR, l = lane % LPR;
    T yv[NVL][VEC];
#pragma unroll
    for (int k = 0; k < NVL; ++k)
#pragma unroll
        for (int q = 0; q < VEC; ++q) yv[k][q] = p.y_last[(l + k * LPR) * VEC + q];
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int tw = (gridDim.x * blockDim.x) >> 5;
    const V* W = reinterpret_cast<const V*>(p.Wout);
    double eacc = 0.0;
    const bool ident = p.out_act == kIdentity;
    const int has_inertia = p.st->has_inertia;
    const double inv_dt2 = p.st->inv_dt2;
    for (int row0 = gw * RPW * UNR; row0 < p.n; row0 += tw * RPW * UNR) {
        V w[UNR][NVL];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int row = row0 + u * RPW + sub;
            if (row < p.n) {
#pragma unroll
                for (int k = 0; k < NVL; ++k) w[u][k] = ld_stream(W + (size_t)row * NVR + l + k * LPR);
            }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int row = row0 + u * RPW + sub;
            T acc = 0;
            if (row < p.n) {
#pragma unroll
                for (int k = 0; k < NVL; ++k) vec_fma(acc, w[u][k], yv[k]);
            }
#pragma unroll
            for (int o = LPR >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (row < p.n && l == 0) {
                const T a = acc + p.bout[row];
                T phi = a;
                if (!ident) {
                    phi = (T)act_eval(p.out_act, (double)a, 0);
                    p.dsout[row] = p.sout[row] * (T)act_eval(p.out_act, (double)a, 1);
                }
                const T uval = p.sout[row] * phi + p.cout[row];
                const int f = row / 3, c = row - 3 * f;
                p.U[(size_t)p.vfree[f] * 4 + c] = uval;
                if (has_inertia) {
                    const T diff = uval - p.ut[row];
                    const T m = p.mass[row];
                    p.rin[row] = (T)(inv_dt2 * (double)(m * diff));
                    eacc += (double)m * (double)diff * (double)diff;
                }
            }
        }
    }
    const double tot = block_sum(eacc, red);
    if (threadIdx.x == 0) p.e_part_out[blockIdx.x] = 0.5 * inv_dt2 * tot;
}

// ---------------------------------------------------------------- K3: element pass
template <typename T>
__device__ __forceinline__ void load_rec(const T* rec, size_t e, T* out12);
template <>
__device__ __forceinline__ void load_rec<float>(const float* rec, size_t e, float* o) {
    const float4* p = reinterpret_cast<const float4*>(rec + e * 12);
    const float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
    o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
    o[8] = c.x; o[9] = c.y; o[10] = c.z; o[11] = c.w;
}
template <>
__device__ __forceinline__ void load_rec<double>(const double* rec, size_t e, double* o) {
    const double2* p = reinterpret_cast<const double2*>(rec + e * 12);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const double2 v = __ldg(p + k);
        o[2 * k] = v.x;
        o[2 * k + 1] = v.y;
    }
}
template <typename T>
__device__ __forceinline__ void load_u(const T* U, int v, T* o);
template <>
__device__ __forceinline__ void load_u<float>(const float* U, int v, float* o) {
    const float4 a = *reinterpret_cast<const float4*>(U + (size_t)v * 4);
    o[0] = a.x; o[1] = a.y; o[2] = a.z;
}
template <>
__device__ __forceinline__ void load_u<double>(const double* U, int v, double* o) {
    const double2 a = *reinterpret_cast<const double2*>(U + (size_t)v * 4);
    o[0] = a.x; o[1] = a.y;
    o[2] = U[(size_t)v * 4 + 2];
}

// Energy and 12 local forces of one tet from vertex displacements.
// A = (Ds - Ds_rest) Dm^-1 (reference element_frame, energy.cpp:163-175);
// forces = vol P Dm^-T (= vol B^T vec(P), energy.cpp:290-291).
template <typename T>
__device__ __forceinline__ T tet_energy_forces(const T* u0, const T* u1, const T* u2, const T* u3,
                                               const T* rec, T* f /*12*/) {
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
            const T h = vol * (P[a * 3 + 0] * rec[c * 3 + 0] + P[a * 3 + 1] * rec[c * 3 + 1] + P[a * 3 + 2] * rec[c * 3 + 2]);
            f[(c + 1) * 3 + a] = h;
            s0 += h;
        }
        f[a] = -s0;
    }
    return vol * psi;
}

template <typename T>
__global__ void __launch_bounds__(256) elem_kernel(const EvalParams<T> p) {
    __shared__ double red[32];
    __shared__ int am_last;
    DevState* st = p.st;
    if (st->phase == kPhaseDone) return;
    const bool skip = st->phase == kPhaseFinalDecode;
    double eacc = 0.0;
    if (!skip) {
        for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < p.E; e += gridDim.x * blockDim.x) {
            const int4 t = __ldg(p.tets + e);
            T rec[12];
            load_rec<T>(p.rec, (size_t)e, rec);
            T u0[3], u1[3], u2[3], u3[3];
            load_u<T>(p.U, t.x, u0);
            load_u<T>(p.U, t.y, u1);
            load_u<T>(p.U, t.z, u2);
            load_u<T>(p.U, t.w, u3);
            T f[12];
            eacc += (double)tet_energy_forces<T>(u0, u1, u2, u3, rec, f);
            T* out = p.forces + (size_t)e * 12;
#pragma unroll
            for (int k = 0; k < 12; ++k) out[k] = f[k];
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
        const double E = e_el + (st->has_inertia ? e_in : 0.0);
        st->f_eval = E;
        if (!skip) st->value_evals++;
        int need = 0;
        if (skip) {
            need = 0;
        } else if (!isfinite(E)) {  // reduced_solver.cpp:198-199 (throws)
            st->status = kStNonFinite;
            need = 0;
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

// ---------------------------------------------------------------- K4: gather + VJP + control
template <typename T, int HP>
__global__ void __launch_bounds__(256) vjp_ctrl_kernel(const EvalParams<T> p) {
    using V = typename VecT<T>::type;
    constexpr int VEC = VecT<T>::N;
    constexpr int NVR = HP / VEC;
    constexpr int LPR = NVR < 32 ? NVR : 32;
    constexpr int NVL = NVR / LPR;
    constexpr int RPW = 32 / LPR;
    constexpr int NWARP = 8;
    extern __shared__ double dsm[];
    // layout: tv[3*vpb] (T), wred[NWARP][HP] (double)
    double* wred = dsm;                                        // NWARP*HP
    T* tv = reinterpret_cast<T*>(dsm + NWARP * HP);            // 3*vpb
    __shared__ double red[32];
    __shared__ int am_last, am_grp_last;
    DevState* st = p.st;
    if (st->phase == kPhaseDone) return;
    const bool need = st->need_grad != 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane / LPR, l = lane % LPR;

    if (need) {
        T acc[NVL][VEC];
#pragma unroll
        for (int k = 0; k < NVL; ++k)
#pragma unroll
            for (int q = 0; q < VEC; ++q) acc[k][q] = 0;
        const V* W = reinterpret_cast<const V*>(p.Wout);
        const int nslab = (p.n_free + p.vpb - 1) / p.vpb;
        const bool ident = p.out_act == kIdentity;
        const int has_inertia = st->has_inertia;
        for (int slab = blockIdx.x; slab < nslab; slab += gridDim.x) {
            const int f0 = slab * p.vpb;
            const int f1 = min(f0 + p.vpb, p.n_free);
            const int R = 3 * (f1 - f0);
            // phase 1: g = sum of incident tet forces (ascending tet id) + inertia, times s
            for (int t = threadIdx.x; t < R; t += blockDim.x) {
                const int f = f0 + t / 3, c = t % 3;
                const int b = __ldg(p.csr_ptr + f), e = __ldg(p.csr_ptr + f + 1);
                T g = 0;
                for (int k = b; k < e; ++k) g += p.forces[(size_t)__ldg(p.csr_ent + k) * 3 + c];
                const int row = 3 * f + c;
                if (has_inertia) g += p.rin[row];
                tv[t] = g * (ident ? p.sout[row] : p.dsout[row]);
            }
            __syncthreads();
            // phase 2: ybar += W_out[rows]^T tv
            for (int rr = warp * RPW + sub; rr < R; rr += NWARP * RPW) {
                const T tval = tv[rr];
                const size_t row = (size_t)3 * f0 + rr;
#pragma unroll
                for (int k = 0; k < NVL; ++k) {
                    const V w = ld_stream(W + row * NVR + l + k * LPR);
                    vec_axpy(acc[k], w, tval);
                }
            }
            __syncthreads();
        }
        // combine sub-rows within the warp (RPW > 1), then warps in fixed order
#pragma unroll
        for (int k = 0; k < NVL; ++k)
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
                T v = acc[k][q];
                for (int o = LPR; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                acc[k][q] = v;
            }
        if (sub == 0) {
#pragma unroll
            for (int k = 0; k < NVL; ++k)
#pragma unroll
                for (int q = 0; q < VEC; ++q) wred[warp * HP + (l + k * LPR) * VEC + q] = (double)acc[k][q];
        }
        __syncthreads();
        for (int j = threadIdx.x; j < HP; j += blockDim.x) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NWARP; ++w) s += wred[w * HP + j];
            p.ybar_part[(size_t)blockIdx.x * HP + j] = s;
        }
        // level 1: group-last block sums its group's partials in block order
        __threadfence();
        __syncthreads();
        const int grp = blockIdx.x / p.group;
        const int g0 = grp * p.group, g1 = min(g0 + p.group, (int)gridDim.x);
        if (threadIdx.x == 0) {
            const unsigned prev = atomicAdd(p.grp_cnt + grp, 1u);
            am_grp_last = (prev == (unsigned)(g1 - g0 - 1));
        }
        __syncthreads();
        if (!am_grp_last) return;
        __threadfence();
        for (int j = threadIdx.x; j < HP; j += blockDim.x) {
            double s = 0.0;
            for (int b = g0; b < g1; ++b) s += p.ybar_part[(size_t)b * HP + j];
            p.ybar_grp[(size_t)grp * HP + j] = s;
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            p.grp_cnt[grp] = 0;
            const unsigned prev = atomicAdd(&st->cnt_top, 1u);
            am_last = (prev == (unsigned)(p.n_groups - 1));
        }
        __syncthreads();
        if (!am_last) return;
        __threadfence();
    } else {
        if (threadIdx.x == 0) {
            const unsigned prev = atomicAdd(&st->cnt_top, 1u);
            am_last = (prev == gridDim.x - 1);
        }
        __syncthreads();
        if (!am_last) return;
        __threadfence();
    }
    // ---------------- last block: gradient, control, next hidden forward
    if (threadIdx.x == 0) {
        st->cnt_top = 0;
        st->loop_iters++;
    }
    double* ybar = dsm;                 // kMaxHidden
    double* tmp = dsm + kMaxHidden;     // kMaxHidden
    if (need) {
        for (int j = threadIdx.x; j < HP; j += blockDim.x) {
            double s = 0.0;
            for (int b = 0; b < p.n_groups; ++b) s += p.ybar_grp[(size_t)b * HP + j];
            ybar[j] = s;
        }
        __syncthreads();
        hidden_backward(p, ybar, tmp);
    }
    __shared__ int more;
    if (warp == 0) {
        int m = 0;
        if (st->mode == kModeLbfgs) {
            m = lbfgs_control(st, p.r);
        } else {
            st->done = 1;
        }
        if (lane == 0) {
            more = m;
            if (!m) {
                st->phase = kPhaseDone;
                st->t_end = globaltimer();
            }
        }
    }
    __syncthreads();
    if (more) hidden_forward(p, dsm);
    if (threadIdx.x == 0 && p.in_graph) cudaGraphSetConditional(p.cond, more ? 1u : 0u);
}

// ---------------------------------------------------------------- setup kernels
// Start an evaluation / minimisation at st->zt (already written): hidden forward.
template <typename T>
__global__ void __launch_bounds__(256) start_kernel(const EvalParams<T> p, int mode, int want_grad) {
    extern __shared__ double dsm[];
    DevState* st = p.st;
    if (threadIdx.x == 0) {
        st->mode = mode;
        st->want_grad = want_grad;
        st->status = kStOk;
        st->phase = kPhaseInit;
        st->done = 0;
        st->code = 4;
        st->iter = 0;
        st->ls = 0;
        st->hist_n = 0;
        st->hist_head = 0;
        st->value_evals = 0;
        st->grad_evals = 0;
        st->need_grad = 0;
        st->accept = 0;
        st->gnorm = 0.0;
        st->loop_iters = 0;
        st->t_start = globaltimer();
    }
    __syncthreads();
    hidden_forward(p, dsm);
}

}  // namespace lsb
