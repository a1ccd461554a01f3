// Host side of the C ABI (include/lipsub_b200.h): context construction,
// HBM layout, kernel dispatch and the CUDA graphs that keep the L-BFGS loop
// and whole timesteps on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lipsub_b200.h"
#include "lsb_context.hpp"
#include "lsb_solve.cuh"
#include "lsb_sweep.cuh"

namespace lsb {

thread_local std::string g_last_error;

const char* status_name(lsb_status s) {
    switch (s) {
        case LSB_OK: return "ok";
        case LSB_EINVAL: return "invalid argument";
        case LSB_ENONFINITE: return "non-finite energy";
        case LSB_ECUDA: return "cuda error";
        case LSB_EMESH: return "mesh error";
        case LSB_ESTATE: return "bad state";
    }
    return "?";
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw LsbError(LSB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ dynamics kernels
// qbar - X for the step (reduced_solver.cpp:249-254), warm start z (:256).
__global__ void prep_step_kernel(int n, const int* vfree, const double* u_state, const double* v_state,
                                 const double* a_ext, const double* z_state, int r, DevState* st, double* ut_out,
                                 double* eprow) {
    const double dt = st->dt;
    const int quasi = st->quasi_static;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int f = i / 3, c = i - 3 * f;
        const size_t vi = (size_t)vfree[f] * 3 + c;
        const double ut = u_state[vi] + dt * v_state[vi] + (dt * dt) * a_ext[i];
        ut_out[i] = quasi ? 0.0 : ut;
        eprow[6 * (size_t)i + 5] = quasi ? 0.0 : ut;
    }
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < r; i += blockDim.x) st->zt[i] = z_state[i];
        if (threadIdx.x == 0) {
            st->has_inertia = quasi ? 0 : 1;
            st->inv_dt2 = 1.0 / (dt * dt);
        }
    }
}

// After a step / simulate: put back the objective lsb_set_inertia installed (the step
// objective's qbar lives in the same ut / eprow column 5 slots; reference reduced_step builds a
// fresh ReducedObjective per step and leaves the caller's untouched, reduced_solver.cpp:241-254).
__global__ void restore_objective_kernel(int n, const double* ut_user, double* ut, double* eprow, DevState* st,
                                         int has_inertia, double inv_dt2, double dt) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double v = ut_user ? ut_user[i] : 0.0;
        ut[i] = v;
        eprow[6 * (size_t)i + 5] = v;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->has_inertia = has_inertia;
        st->quasi_static = has_inertia ? 0 : 1;
        st->inv_dt2 = inv_dt2;
        st->dt = dt;
    }
}

void restore_user_objective(Context& c) {
    const bool inert = c.has_qbar && c.d_ut_user;
    restore_objective_kernel<<<std::max(1, std::min((c.n + 255) / 256, 4 * c.num_sms)), 256, 0, c.stream>>>(
        c.n, inert ? c.d_ut_user : nullptr, c.d_ut, c.d_eprow, c.d_state, inert ? 1 : 0, 1.0 / (c.dt * c.dt), c.dt);
    cuda_check(cudaGetLastError(), "restore objective");
}

// x' = unpack(decode(z*)), v' = (x' - x) / dt over all V rows (:266-276), report.
__global__ void finalize_step_kernel(int V, const double* U, const char* vpinned, const double* pin_disp,
                                     double* u_state, double* v_state, double* z_state, int r, DevState* st) {
    lsb_exit_report* reports = static_cast<lsb_exit_report*>(st->reports);
    double* z_traj = st->z_traj;
    const double dt = st->dt;
    const int quasi = st->quasi_static;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        for (int c = 0; c < 3; ++c) {
            const size_t k = (size_t)v * 3 + c;
            double un;
            if (vpinned[v]) un = pin_disp[k];
            else un = U[(size_t)v * 4 + c];
            v_state[k] = quasi ? 0.0 : (un - u_state[k]) / dt;
            u_state[k] = un;
        }
    }
    if (blockIdx.x == 0) {
        const int idx = st->step_idx;
        __syncthreads();
        for (int i = threadIdx.x; i < r; i += blockDim.x) {
            z_state[i] = st->x[i];
            if (z_traj) z_traj[(size_t)idx * r + i] = st->x[i];
        }
        if (threadIdx.x == 0) {
            lsb_exit_report rep;
            rep.code = st->status != kStOk ? -st->status : st->code;
            rep.iterations = (st->code == 4 || (st->code == 1 && st->iter >= st->max_iters)) ? st->max_iters : st->iter;
            rep.final_grad_inf_norm = st->gnorm;
            rep.wall_time_ms = (double)(st->t_end - st->t_start) * 1e-6;
            rep.value_evals = st->value_evals;
            rep.grad_evals = st->grad_evals;
            if (reports) reports[idx] = rep;
            st->step_idx = idx + 1;
            st->t += dt;
        }
    }
}

__global__ void count_loop_kernel(const DevState* st, long long* acc, int per_body) {
    // device-side launch accounting for WHILE-loop bodies: per_body kernels per body
    if (threadIdx.x == 0 && blockIdx.x == 0) acc[0] += (long long)per_body * st->loop_iters;
}

// ------------------------------------------------------------------ Impl<TS>
constexpr int kSolveDefaultMaxRows = 262144;

template <typename TS>
struct KernelSet {
    void (*out_fwd)(const EvalParams<TS>);
    void (*vjp)(const EvalParams<TS>);
    void (*vjp_gather)(const EvalParams<TS>);  // gather folded into the VJP (tv in smem)
    void (*vjp_wgather)(const EvalParams<TS>);  // gather per warp and tile inside the VJP stream
    size_t smem;      // dynamic smem of both streaming kernels (ring + scratch)
    int tile_rows;
    size_t stage_bytes;  // one ring stage (tile + side records)
};

template <typename TS, int HP>
KernelSet<TS> kernels_for() {
    return {out_fwd_tma_kernel<TS, HP>, vjp_tma_kernel<TS, HP>, vjp_gather_tma_kernel<TS, HP>,
            vjp_wgather_tma_kernel<TS, HP>, stream_smem_bytes<TS, HP>(),
            StreamCfg<TS, HP>::TR, (size_t)StreamCfg<TS, HP>::STAGEB};
}

using SolveFnD = void (*)(const EvalParams<double>, const SolveParams);
using SolveFnF = void (*)(const EvalParams<float>, const SolveParams);
template <typename TS>
struct SolveFn {
    using type = void (*)(const EvalParams<TS>, const SolveParams);
};
template <typename TS, int CS>
typename SolveFn<TS>::type select_solve(int hp);
template <>
SolveFn<double>::type select_solve<double, 8>(int hp) {
    switch (hp) {
        case 64: return solve_kernel<double, 64, 8>;
        case 128: return solve_kernel<double, 128, 8>;
        case 256: return solve_kernel<double, 256, 8>;
        case 512: return solve_kernel<double, 512, 8>;
    }
    return nullptr;
}
template <>
SolveFn<double>::type select_solve<double, 16>(int hp) {
    switch (hp) {
        case 64: return solve_kernel<double, 64, 16>;
        case 128: return solve_kernel<double, 128, 16>;
        case 256: return solve_kernel<double, 256, 16>;
        case 512: return solve_kernel<double, 512, 16>;
    }
    return nullptr;
}
template <>
SolveFn<float>::type select_solve<float, 8>(int hp) {
    switch (hp) {
        case 128: return solve_kernel<float, 128, 8>;
        case 256: return solve_kernel<float, 256, 8>;
        case 512: return solve_kernel<float, 512, 8>;
    }
    return nullptr;
}
template <>
SolveFn<float>::type select_solve<float, 16>(int hp) {
    switch (hp) {
        case 128: return solve_kernel<float, 128, 16>;
        case 256: return solve_kernel<float, 256, 16>;
        case 512: return solve_kernel<float, 512, 16>;
    }
    return nullptr;
}

template <typename TS>
KernelSet<TS> select_kernels(int hp);
template <>
KernelSet<float> select_kernels<float>(int hp) {
    switch (hp) {
        case 128: return kernels_for<float, 128>();
        case 256: return kernels_for<float, 256>();
        case 512: return kernels_for<float, 512>();
    }
    throw LsbError(LSB_EINVAL, "decoder: unsupported padded width");
}
template <>
KernelSet<double> select_kernels<double>(int hp) {
    switch (hp) {
        case 64: return kernels_for<double, 64>();
        case 128: return kernels_for<double, 128>();
        case 256: return kernels_for<double, 256>();
        case 512: return kernels_for<double, 512>();
    }
    throw LsbError(LSB_EINVAL, "decoder: unsupported padded width");
}

template <typename TS>
using SweepFn = void (*)(const EvalParams<TS>, const SweepParams);
template <typename TS>
SweepFn<TS> select_sweep(int hp, size_t* smem);
template <>
SweepFn<float> select_sweep<float>(int hp, size_t* smem) {
    switch (hp) {
        case 128: *smem = sweep_smem_bytes<float, 128>(); return sweep_kernel<float, 128>;
        case 256: *smem = sweep_smem_bytes<float, 256>(); return sweep_kernel<float, 256>;
        case 512: *smem = sweep_smem_bytes<float, 512>(); return sweep_kernel<float, 512>;
    }
    return nullptr;
}
template <>
SweepFn<double> select_sweep<double>(int hp, size_t* smem) {
    switch (hp) {
        case 64: *smem = sweep_smem_bytes<double, 64>(); return sweep_kernel<double, 64>;
        case 128: *smem = sweep_smem_bytes<double, 128>(); return sweep_kernel<double, 128>;
        case 256: *smem = sweep_smem_bytes<double, 256>(); return sweep_kernel<double, 256>;
    }
    return nullptr;
}

using CtrlFn = void (*)(int, int, int);  // placeholder type for table entries

template <typename TS>
struct Impl final : ImplBase {
    EvalParams<TS> p{};
    KernelSet<TS> ks{};
    void (*ctrl)(const EvalParams<TS>, int, int, int) = nullptr;
    size_t vjp_smem = 0, ctrl_smem = 0, out_smem = 0, vjpg_smem = 0;
    bool fuse_gather = false;
    int ctrl_threads = 256;
    int grid_gather = 1;
    // persistent solve kernel (cooperative launch of thread-block clusters)
    typename SolveFn<TS>::type solve = nullptr;
    size_t solve_smem = 0;
    unsigned launch_seq = 0;
    int solve_spw = 1, solve_spw_ctrl = 1, solve_tv_cap = 0, solve_tv_off = 0, solve_tv_off_ctrl = 0;
    int solve_wsl_words = 0, solve_tv_global = 0;
    int solve_grid = 0;
    float solve_ctrl_tile_w = 0.5f;
    EvalParams<TS> ps{};  // params with solve-sized partial buffers
    SolveShared* d_sh = nullptr;
    int cs = 8;
    cudaGraphExec_t g_min = nullptr, g_step = nullptr, g_eval[2] = {nullptr, nullptr};
    // sweep pass (lsb_sweep.cuh): out_fwd + elem + gather/VJP as one ticketed kernel
    SweepFn<TS> sweep = nullptr;
    SweepParams swp{};
    size_t sweep_smem = 0;
    int sweep_grid = 0;
    bool use_sweep = false;
    std::vector<void*> sweep_bufs;
    EvalParams<TS> pc{};  // params of the control kernels (the sweep's group partials when it runs)
    int pdl_mask = 15;    // programmatic edges inside graph bodies (LSB_PDL bit mask)
    void (*elem_fn)(const EvalParams<TS>) = elem_kernel<TS, 0>;
    cudaGraphConditionalHandle h_min{}, h_step{};

    ~Impl() override {
        if (g_min) cudaGraphExecDestroy(g_min);
        if (g_step) cudaGraphExecDestroy(g_step);
        for (auto& ge : g_eval)
            if (ge) cudaGraphExecDestroy(ge);
    }

    // One evaluation (ctrl start -> [sweep | out_fwd -> elem -> gather/VJP] -> ctrl) as a cached
    // graph per want_grad, with programmatic edges where LSB_PDL enables them.
    cudaGraphExec_t eval_graph(Context& c, bool want_grad) {
        cudaGraphExec_t& ge = g_eval[want_grad ? 1 : 0];
        if (ge) return ge;
        cudaGraph_t g;
        cuda_check(cudaGraphCreate(&g, 0), "graph create");
        int cm = kCtrlStart, mode = kModeEval, want = want_grad ? 1 : 0;
        EvalParams<TS> pg = p;
        EvalParams<TS> pcg = pc;
        SweepParams sw = swp;
        void* sargs[] = {&pcg, &cm, &mode, &want};
        cudaGraphNode_t n0 = add_kernel(g, nullptr, (void*)ctrl, cs, ctrl_smem, sargs, ctrl_threads);
        void* a1[] = {&pg};
        void* asw[] = {&pg, &sw};
        const int pm = c.dev.pdl;
        if (!want_grad && !use_sweep) {
            // value only (lsb_eval without gradient): E is final after the element pass; neither the
            // VJP nor the control kernel after it has anything to do
            cudaGraphNode_t n1 = add_kernel_pdl(g, n0, (void*)ks.out_fwd, p.grid_out, out_smem, a1, kStreamThreads, pm & 1);
            add_kernel_pdl(g, n1, (void*)elem_fn, p.grid_elem, 0, a1, 256, pm & 2);
            cuda_check(cudaGraphInstantiate(&ge, g, 0), "graph instantiate (eval)");
            cudaGraphDestroy(g);
            return ge;
        }
        cudaGraphNode_t n3;
        if (use_sweep) {
            n3 = add_kernel_pdl(g, n0, (void*)sweep, sweep_grid, sweep_smem, asw, kSwThreads, pm & 1);
        } else {
            cudaGraphNode_t n1 = add_kernel_pdl(g, n0, (void*)ks.out_fwd, p.grid_out, out_smem, a1, kStreamThreads, pm & 1);
            cudaGraphNode_t n2 = add_kernel_pdl(g, n1, (void*)elem_fn, p.grid_elem, 0, a1, 256, pm & 2);
            n3 = add_gather_vjp(g, n2, a1, pm & 4);
        }
        int cm2 = kCtrlAfterEval, z0 = 0, z1 = 0;
        void* a4[] = {&pcg, &cm2, &z0, &z1};
        add_kernel_pdl(g, n3, (void*)ctrl, cs, ctrl_smem, a4, ctrl_threads, pm & 8);
        cuda_check(cudaGraphInstantiate(&ge, g, 0), "graph instantiate (eval)");
        cudaGraphDestroy(g);
        return ge;
    }

    void launch_eval_graph(Context& c, bool want_grad) {
        cuda_check(cudaGraphLaunch(eval_graph(c, want_grad), c.stream), "graph launch (eval)");
        if (!want_grad && !use_sweep) c.launches += 3;  // ctrl, out_fwd, elem
        else c.launches += use_sweep ? 3 : (fuse_gather ? 5 : 6);  // ctrl, [sweep | out_fwd, elem, [gather,] vjp], ctrl
    }

    int eval_timed(Context& c, cudaEvent_t* ev, bool want_grad) override {
        cuda_check(cudaEventRecord(ev[0], c.stream), "ev");
        if (solve && c.use_solve) launch_solve(c, 0, 0, want_grad ? 1 : 0);
        else launch_eval_graph(c, want_grad);
        cuda_check(cudaEventRecord(ev[3], c.stream), "ev");
        return 2;
    }

    void setup(Context& c) override {
        const HostMesh& m = c.mesh;
        p.n = c.n;
        p.n_free = m.n_free;
        p.V = m.V;
        p.E = m.E;
        p.r = c.r;
        p.nhid = c.nhid;
        p.h = c.h;
        p.hp = c.hp;
        p.out_act = c.out_act;
        p.elem_f32 = std::is_same<TS, float>::value && c.dev.elem_f32 ? 1 : 0;
        p.l2_pf_tiles = c.dev.l2_pf;
        p.l2_pf_elem = c.dev.l2_pf_elem;
        elem_fn = p.elem_f32 ? elem_kernel<TS, 1> : elem_kernel<TS, 0>;
        p.Wout = static_cast<const TS*>(c.d_Wout);
        p.bout = c.d_bout;
        p.sout = c.d_sout;
        p.cout = c.d_cout;
        p.dsout = c.d_dsout;
        p.mass = c.d_mass;
        p.ut = c.d_ut;
        p.rin = c.d_rin;
        p.eprow = c.d_eprow;
        p.tv = c.d_tv;
        p.vfree = c.d_vfree;
        p.tets = reinterpret_cast<const int4*>(c.d_tets);
        p.rec = static_cast<const TS*>(c.d_rec);
        p.U = c.d_U;
        p.forces = c.d_forces;
        p.csr_ptr = c.d_csr_ptr;
        p.csr_ent = c.d_csr_ent;
        p.fpos = reinterpret_cast<const int4*>(c.d_fpos);
        p.Wh = c.d_Wh;
        p.Wh_s = std::is_same<TS, double>::value ? reinterpret_cast<const TS*>(c.d_Wh)
                                                  : reinterpret_cast<const TS*>(c.d_Wh_f);
        p.bh = c.d_bh;
        for (int l = 0; l < c.nhid; ++l) {
            p.hoff[l] = c.hoff[l];
            p.boff[l] = c.boff[l];
            p.hrows[l] = c.hrows[l];
            p.hcols[l] = c.hcols[l];
            p.hact[l] = c.hact[l];
        }
        p.a_hid = c.d_a_hid;
        p.y_last = c.d_y_last;
        p.st = c.d_state;
        ks = select_kernels<TS>(c.hp);
        // W_out stays L2-resident when it fits in ~60% of L2, else it is streamed
        const size_t wbytes = (size_t)c.n * c.hp * sizeof(TS);
        p.w_resident = wbytes <= (size_t)(0.6 * c.l2_bytes) ? 1 : 0;
        if (c.dev.w_resident >= 0) p.w_resident = c.dev.w_resident;  // developer override
        p.w_keep_tiles = p.w_resident ? 0 : c.dev.w_keep;
        // grid sizing: persistent grids of (SMs x resident blocks)
        int occ = 0;
        p.vpb = 64;  // 192 rows per slab: a multiple of every tile height
        out_smem = ks.smem;
        vjp_smem = ks.smem + 8 * (size_t)c.hp * sizeof(double);
        cuda_check(cudaFuncSetAttribute(ks.out_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)out_smem),
                   "smem attr out_fwd");
        cuda_check(cudaFuncSetAttribute(ks.vjp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vjp_smem),
                   "smem attr vjp");
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ks.out_fwd, kStreamThreads, out_smem),
                   "occupancy out_fwd");
        const int ntiles = (c.n + ks.tile_rows - 1) / ks.tile_rows;
        p.grid_out = std::max(1, std::min(ntiles, c.num_sms * std::max(1, occ)));
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, elem_fn, 256, 0), "occupancy elem");
        c.grid_elem_cap = c.num_sms * std::max(1, occ);
        p.grid_elem = std::max(1, std::min((m.E + 255) / 256, c.grid_elem_cap));
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ks.vjp, kStreamThreads, vjp_smem),
                   "occupancy vjp");
        p.grid_vjp = std::max(1, std::min(ntiles, c.num_sms * std::max(1, occ)));
        // fused gather + VJP: tv for a CTA's rows in shared memory; W-only stages, column sums in
        // the drained ring.  Grid: two CTAs per SM (measured on config 3: 4.70K evals/s vs 4.27K with
        // three, whose per-CTA gather prologues cost more than the extra stages gain), fewer if
        // the tv scratch does not fit.
        {
            fuse_gather = c.dev.fuse_gather != 0;
            bool ok = false;
            if (fuse_gather && c.dev.vjp_wg) {  // per-warp gather: no tv scratch, up to 3 CTAs per SM
                const size_t sm = 512 + (size_t)(kStreamThreads / 32) * kStreamSpw * ks.tile_rows * c.hp * sizeof(TS);
                int occ2 = 0;
                if (cudaFuncSetAttribute(ks.vjp_wgather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) ==
                        cudaSuccess &&
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, ks.vjp_wgather, kStreamThreads, sm) ==
                        cudaSuccess &&
                    occ2 >= 1) {
                    ks.vjp_gather = ks.vjp_wgather;
                    vjpg_smem = sm;
                    p.grid_vjp = std::max(1, std::min(ntiles, c.num_sms * std::min(occ2, c.dev.vjp_wg_cta)));
                    ok = true;
                }
                cudaGetLastError();
            }
#ifndef LSB_VJP_MAXCTA
#define LSB_VJP_MAXCTA 2
#endif
            for (int want = LSB_VJP_MAXCTA; fuse_gather && want >= 1 && !ok; --want) {  // CTA-wide gather
                const int grid = std::max(1, std::min(ntiles, c.num_sms * want));
                const size_t tvb = ((size_t)((ntiles + grid - 1) / grid) * ks.tile_rows * sizeof(double) + 127) &
                                   ~(size_t)127;
                const size_t sm = 512 + (size_t)(kStreamThreads / 32) * kStreamSpw * ks.tile_rows * c.hp * sizeof(TS) + tvb;
                int occ2 = 0;
                if (cudaFuncSetAttribute(ks.vjp_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) !=
                        cudaSuccess ||
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, ks.vjp_gather, kStreamThreads, sm) !=
                        cudaSuccess) {
                    cudaGetLastError();
                    continue;
                }
                if (occ2 * c.num_sms >= grid) {
                    vjpg_smem = sm;
                    p.grid_vjp = grid;
                    ok = true;
                }
            }
            if (!ok) fuse_gather = false;  // keep the VJP grid; fall back to the separate gather kernel
            c.body_kernels = fuse_gather ? 4 : 5;
        }
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_kernel<TS>, 256, 0), "occupancy gather");
        grid_gather = std::max(1, std::min((m.n_free + 255) / 256, c.num_sms * std::max(1, occ)));
        p.group = 16;
        p.n_groups = (p.grid_vjp + p.group - 1) / p.group;
        // control cluster: hidden weights split in row slices over cs CTAs
        size_t wtot = 0;
        int maxrows = 0;
        for (int l = 0; l < c.nhid; ++l) {
            wtot += (size_t)c.hrows[l] * c.hcols[l];
            maxrows = std::max(maxrows, c.hrows[l]);
        }
        const size_t fixed = (3 * kMaxHidden + 128 + 2 * kMaxLayers * 64) * sizeof(double) + sizeof(DevState) + 64;
        auto slice_words = [&](int k) {  // 8-byte words of the staged slices (stored as TS)
            size_t e = 0;
            for (int l = 0; l < c.nhid; ++l) e += (((size_t)((c.hrows[l] + k - 1) / k) * c.hcols[l] + 3) & ~(size_t)3);
            return (e * sizeof(TS) + 7) / 8;
        };
        cs = 8;
        if (slice_words(8) * 8 + fixed > 200 * 1024 || (maxrows + 7) / 8 > 64) cs = 16;
        // wide decoders on the multi-kernel path (config 3): 16-CTA control clusters (config 3: 4.69K
        // vs 4.66K evals/s device-timed, 4.68K vs 4.49K through lsb_eval)
        if (c.hp >= 256 && c.n > kSolveDefaultMaxRows) cs = 16;
        if (c.dev.ctrl_cluster16) cs = 16;  // developer override
        if (slice_words(cs) * 8 + fixed > 220 * 1024 || (maxrows + cs - 1) / cs > 64)
            throw LsbError(LSB_EINVAL, "decoder: hidden layers too large for the control cluster");
        p.cs = cs;
        p.ctrl_smem_w = (int)slice_words(cs);
        ctrl_smem = p.ctrl_smem_w * sizeof(double) + fixed;
        ctrl = cs == 8 ? ctrl_kernel<TS, 8> : ctrl_kernel<TS, 16>;
        ctrl_threads = 256;
        // uniform-width decoders: the fast-path control kernel (static row partition, st.async
        // layer exchange); LSB_CTRL_FAST=0 keeps the generic kernel
        {
            bool uniform = c.nhid >= 1 && c.r >= 1 && c.r <= 64 && (c.hp == 128 || c.hp == 256);
            for (int l = 0; l < c.nhid && uniform; ++l)
                uniform = c.hrows[l] == c.hp && c.hcols[l] == (l == 0 ? c.r : c.hp);
            if (uniform && c.dev.ctrl_fast) {
                const size_t fsm = ctrl_fast_smem<TS>(c.nhid, c.hcols, c.hp / cs);
                if (fsm + 1024 <= 227 * 1024) {
                    if (c.hp == 128) ctrl = cs == 8 ? ctrl_fast_kernel<TS, 128, 8> : ctrl_fast_kernel<TS, 128, 16>;
                    else ctrl = cs == 8 ? ctrl_fast_kernel<TS, 256, 8> : ctrl_fast_kernel<TS, 256, 16>;
                    ctrl_smem = fsm;
                    ctrl_threads = kSolveThreads;
                }
            }
        }
        if (cs == 16)
            cuda_check(cudaFuncSetAttribute(ctrl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1), "cluster 16");
        cuda_check(cudaFuncSetAttribute(ctrl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctrl_smem),
                   "smem attr ctrl");
        (void)wtot;
        c.grid_out = p.grid_out;
        c.grid_elem = p.grid_elem;
        c.grid_vjp = p.grid_vjp;
        c.alloc_partials(p.grid_out, p.grid_elem, p.grid_vjp, p.n_groups);
        p.e_part_out = c.d_e_part_out;
        p.e_part_elem = c.d_e_part_elem;
        p.ybar_part = c.d_ybar_part;
        p.ybar_grp = c.d_ybar_grp;
        p.grp_cnt = c.d_grp_cnt;
        p.in_graph = 0;
        pdl_mask = c.dev.pdl;
        setup_sweep(c);
        setup_solve(c);
    }

    // Work-item plan of the sweep pass over the current element set (lsb_sweep.cuh).
    void setup_sweep(Context& c) {
        for (void* b : sweep_bufs) c.dfree(b);
        sweep_bufs.clear();
        use_sweep = false;
        pc = p;
        c.body_kernels = fuse_gather ? 4 : 5;
        if (!c.dev.sweep) return;
        sweep = select_sweep<TS>(c.hp, &sweep_smem);
        if (!sweep || sweep_smem > 227 * 1024) return;
        if (cudaFuncSetAttribute(sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sweep_smem) != cudaSuccess) {
            cudaGetLastError();
            return;
        }
        int occ = 0;
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep, kSwThreads, sweep_smem),
                   "occupancy sweep");
        if (occ < 1) return;
        sweep_grid = c.num_sms * occ;
        const HostMesh& m = c.mesh;
        const int TR = ks.tile_rows, RI = kSwItemTiles * TR;
        const int ntiles = (c.n + TR - 1) / TR;
        const int nf = (ntiles + kSwItemTiles - 1) / kSwItemTiles, nv = nf;
        const int ne = (m.E + kSwTets - 1) / kSwTets;
        const int ng = (c.n + kSwGatherRows - 1) / kSwGatherRows;
        std::vector<int> depF(ne, -1), depG(ng, -1), depV(nv, 0);
        for (int e = 0; e < m.E; ++e)
            for (int k = 0; k < 4; ++k) {
                const int slot = m.free_index[m.T[4 * (size_t)e + k]];
                if (slot >= 0) depF[e / kSwTets] = std::max(depF[e / kSwTets], (3 * slot + 2) / RI);
            }
        for (int g = 0; g < ng; ++g) {
            const int R0 = g * kSwGatherRows, R1 = std::min(c.n, R0 + kSwGatherRows);
            for (int f = R0 / 3; f <= (R1 - 1) / 3; ++f)
                for (int k = m.csr_ptr[f]; k < m.csr_ptr[f + 1]; ++k)
                    depG[g] = std::max(depG[g], (m.csr_ent[k] / 4) / kSwTets);
        }
        for (int v = 0; v < nv; ++v) depV[v] = (std::min(c.n, (v + 1) * RI) - 1) / kSwGatherRows;
        // element queue: E items in order; a G item follows its last E dependency by `lag`
        // tickets (about one grid of element groups), or as soon as nothing else can be emitted
        const int lag = (int)(c.dev.sweep_lag * sweep_grid);
        const int etotal = ne + ng;
        std::vector<int> order;
        order.reserve(etotal);
        std::vector<int> posE(ne, 0);
        int ei = 0, gi = 0;
        auto g_ready = [&](bool use_lag) {
            const int d = depG[gi];
            return d < 0 || (d < ei && (!use_lag || posE[d] + lag <= (int)order.size()));
        };
        while ((int)order.size() < etotal) {
            bool prog = false;
            if (ei < ne) {
                posE[ei] = (int)order.size();
                order.push_back((kSwE << 28) | ei);
                ++ei;
                prog = true;
            }
            while (gi < ng && g_ready(true)) order.push_back((kSwG << 28) | gi++), prog = true;
            if (!prog) {
                if (gi < ng && g_ready(false)) order.push_back((kSwG << 28) | gi++);
                else throw LsbError(LSB_EMESH, "sweep plan: unsatisfiable dependency");
            }
        }
        auto up = [&](const void* src, size_t bytes) {
            void* d = c.dmalloc(std::max<size_t>(bytes, 16));
            sweep_bufs.push_back(d);
            if (src) c.copy(d, src, bytes, cudaMemcpyHostToDevice, "sweep plan");
            else cuda_check(cudaMemsetAsync(d, 0, std::max<size_t>(bytes, 16), c.stream), "sweep zero");
            return d;
        };
        const int ngroups = (nv + kSwGroup - 1) / kSwGroup;
        swp = SweepParams{};
        swp.eorder = static_cast<const int*>(up(order.data(), 4 * order.size()));
        swp.etotal = etotal;
        swp.nf = nf;
        swp.ne = ne;
        swp.ng = ng;
        swp.nv = nv;
        swp.ngroups = ngroups;
        swp.depF = static_cast<const int*>(up(depF.data(), 4 * depF.size()));
        swp.depG = static_cast<const int*>(up(depG.data(), 4 * depG.size()));
        swp.depV = static_cast<const int*>(up(depV.data(), 4 * depV.size()));
        swp.f_done = static_cast<unsigned*>(up(nullptr, 4 * (size_t)nf));
        swp.e_done = static_cast<unsigned*>(up(nullptr, 4 * (size_t)ne));
        swp.g_done = static_cast<unsigned*>(up(nullptr, 4 * (size_t)ng));
        swp.e_f = static_cast<double*>(up(nullptr, 8 * (size_t)nf));
        swp.e_e = static_cast<double*>(up(nullptr, 8 * (size_t)ne));
        swp.ybar_item = static_cast<double*>(up(nullptr, 8 * (size_t)nv * c.hp));
        swp.ybar_grp = static_cast<double*>(up(nullptr, 8 * (size_t)ngroups * c.hp));
        swp.grp_cnt = static_cast<unsigned*>(up(nullptr, 4 * (size_t)ngroups));
        SweepCounters ctr0{};
        ctr0.seq = 1;
        swp.ctr = static_cast<SweepCounters*>(up(&ctr0, sizeof(SweepCounters)));
        swp.trace_cap = nf + nv + etotal;
        swp.trace = c.dev.trace ? static_cast<unsigned long long*>(up(nullptr, 32 * (size_t)swp.trace_cap)) : nullptr;
        c.d_sweep_trace = swp.trace;
        c.sweep_tickets = swp.trace_cap;
        cuda_check(cudaStreamSynchronize(c.stream), "sweep plan sync");
        use_sweep = true;
        pc.n_groups = ngroups;
        pc.ybar_grp = swp.ybar_grp;
        c.body_kernels = 2;  // sweep, ctrl
    }

    void launch_sweep(cudaStream_t s) { sweep<<<sweep_grid, kSwThreads, sweep_smem, s>>>(p, swp); }

    void setup_solve(Context& c) {
        if (c.dev.disable_solve) {
            c.solve_reason = "disabled by LSB_DISABLE_SOLVE_KERNEL";
            return;
        }
        solve = cs == 8 ? select_solve<TS, 8>(c.hp) : select_solve<TS, 16>(c.hp);
        if (!solve) {
            c.solve_reason = "no solve kernel instantiated for this width";
            return;
        }
        // control-area weights in storage precision: per-layer row slices, 16-byte aligned
        {
            size_t w = 0;
            for (int l = 0; l < c.nhid; ++l)
                w += ((size_t)((c.hrows[l] + cs - 1) / cs) * c.hcols[l] + 3) & ~(size_t)3;
            solve_wsl_words = (int)((w * sizeof(TS) + 7) / 8);
        }
        // self-issued rings: 9 warps x spw stages each, as many as fit (control CTAs: their
        // control area follows the ring), then the tv / partials scratch -- or, when that does
        // not fit, tv in global memory streamed with the VJP tiles
        const size_t cap = 227 * 1024 - 2048;  // static smem of the kernel (barriers, flags) + margin
        const size_t ctrl_area = ((size_t)solve_wsl_words + ctrl_fixed_words()) * sizeof(double);
        const int nw = kSolveThreads / 32;
        for (int tvg = c.dev.solve_tv_global; tvg < 2; ++tvg) {
            solve_tv_global = tvg;
            if (tvg == 0) {
                const int ntiles = (c.n + ks.tile_rows - 1) / ks.tile_rows;
                const int g_min = 96;  // clusters of 8/16 on 148 SMs give >= 112 CTAs
                solve_tv_cap = std::max((ntiles + g_min - 1) / g_min * ks.tile_rows, c.hp);
            } else {
                solve_tv_cap = c.hp;  // partials only
            }
            const size_t tvb = ((size_t)solve_tv_cap * sizeof(double) + 127) & ~(size_t)127;
            solve_spw_ctrl = 0;
            for (int k = 1; k * nw <= kSolveMaxStages && k <= 3; ++k)
                if (kSolveBarBytes + k * nw * ks.stage_bytes + ctrl_area + tvb <= cap) solve_spw_ctrl = k;
            solve_spw = std::max(solve_spw_ctrl, 1);
            for (int k = 1; k * nw <= kSolveMaxStages && k <= 2; ++k)
                if (kSolveBarBytes + k * nw * ks.stage_bytes + tvb <= cap) solve_spw = std::max(solve_spw, k);
            solve_tv_off_ctrl = (int)(kSolveBarBytes + solve_spw_ctrl * nw * ks.stage_bytes + ctrl_area);
            solve_tv_off = (int)(kSolveBarBytes + solve_spw * nw * ks.stage_bytes);
            solve_smem = std::max((size_t)solve_tv_off_ctrl, (size_t)solve_tv_off) + tvb;
            if (solve_spw_ctrl == 0) solve_smem = SIZE_MAX;  // no ring stage fits beside the control area
            if (solve_smem <= cap) break;
        }
        if (solve_smem > cap || solve_spw_ctrl < 1 || solve_spw < 1) {
            c.solve_reason = "shared memory: no ring fits beside the control area within 227 KB";
            solve = nullptr;
            return;
        }
        if (cudaFuncSetAttribute(solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)solve_smem) != cudaSuccess ||
            (cs == 16 && cudaFuncSetAttribute(solve, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)) {
            c.solve_reason = std::string("attribute: ") + cudaGetErrorString(cudaGetLastError()) + " (smem " +
                             std::to_string(solve_smem) + " B)";
            solve = nullptr;
            return;
        }
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kSolveThreads);
        cfg.dynamicSmemBytes = solve_smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, (void*)solve, &cfg) != cudaSuccess || nclusters < 1) {
            c.solve_reason = std::string("occupancy: ") + cudaGetErrorString(cudaGetLastError());
            solve = nullptr;
            return;
        }
        if (c.dev.solve_clusters > 0) nclusters = std::min(nclusters, c.dev.solve_clusters);  // developer override
        solve_grid = nclusters * cs;
        if (solve_grid > kSolveMaxGrid) {  // the control cluster sums the per-CTA partials with 5 x 32 lanes
            c.solve_reason = "grid of " + std::to_string(solve_grid) + " CTAs exceeds " + std::to_string(kSolveMaxGrid);
            solve = nullptr;
            return;
        }
        if (c.dev.ctrl_tile_w >= 0.f) solve_ctrl_tile_w = c.dev.ctrl_tile_w;  // developer tuning
        solve_ctrl_tile_w = std::min(1.0f, std::max(0.0f, solve_ctrl_tile_w));
        if (!solve_tv_global) {
            const int ntiles = (c.n + ks.tile_rows - 1) / ks.tile_rows;
            int share = 0;  // largest per-CTA tile share
            for (int k = 0; k < solve_grid; ++k)
                share = std::max(share, solve_tile_start(ntiles, k + 1, solve_grid, cs, solve_ctrl_tile_w) -
                                            solve_tile_start(ntiles, k, solve_grid, cs, solve_ctrl_tile_w));
            if (share * ks.tile_rows > solve_tv_cap) {
                c.solve_reason = "tv scratch too small for " + std::to_string(solve_grid) + " CTAs";
                solve = nullptr;
                return;
            }
        }
        ps = p;
        ps.e_part_out = static_cast<double*>(c.dmalloc(sizeof(double) * solve_grid));
        ps.e_part_elem = static_cast<double*>(c.dmalloc(sizeof(double) * solve_grid));
        ps.ybar_part = static_cast<double*>(c.dmalloc(sizeof(double) * (size_t)solve_grid * c.hp));
        d_sh = static_cast<SolveShared*>(c.dmalloc(sizeof(SolveShared)));
        c.solve_grid = solve_grid;
        // Default path: the persistent kernel wins where an evaluation is latency-bound (configs
        // 1-2); for very large n (config 3) the multi-kernel path, which streams on all SMs with
        // several CTAs each, is faster (measured 275 vs 337 us per c3 evaluation), so it stays
        // the default there.  lsb_set_solve_kernel(ctx, 1) selects the persistent kernel anyway.
        if (c.n > kSolveDefaultMaxRows) c.use_solve = false;
        c.solve_reason = "ring stages/warp " + std::to_string(solve_spw) + " (control CTAs " +
                         std::to_string(solve_spw_ctrl) + "), smem " + std::to_string(solve_smem) + " B, cluster " +
                         std::to_string(cs) + (solve_tv_global ? ", tv in global memory" : "");
    }

    SolveParams solve_params(Context& c, int task, int quasi, int want_grad = 1) {
        SolveParams sp{};
        sp.task = task;
        sp.quasi = quasi;
        sp.spw = solve_spw;
        sp.spw_ctrl = solve_spw_ctrl;
        sp.tv_off = solve_tv_off;
        sp.tv_off_ctrl = solve_tv_off_ctrl;
        sp.tv_cap = solve_tv_cap;
        sp.ctrl_tile_w = solve_ctrl_tile_w;
        sp.pf_frac = c.dev.pf_frac;
        sp.tv_global = solve_tv_global;
        sp.wsl_words = solve_wsl_words;
        sp.exp = c.dev.solve_exp;
        sp.seq = ++launch_seq;
        sp.want_grad = want_grad;
        sp.u_state = c.d_u_state;
        sp.v_state = c.d_v_state;
        sp.a_ext = c.d_a_ext;
        sp.z_state = c.d_z_state;
        sp.u_state_w = c.d_u_state;
        sp.v_state_w = c.d_v_state;
        sp.vpinned = c.d_vpinned;
        sp.pin_disp = c.d_pin_disp;
        sp.sh = d_sh;
        sp.launch_acc = nullptr;
        sp.trace = c.d_trace;
        return sp;
    }

    bool eval_direct(Context& c, const double* z, bool want_grad, double* out_dev) override {
        if (!(solve && c.use_solve) || c.r > kMaxLatent) return false;
        launch_solve(c, 0, 0, want_grad ? 1 : 0, z, out_dev);
        return true;
    }

    void launch_solve(Context& c, int task, int quasi, int want_grad = 1, const double* z = nullptr,
                      double* out_dev = nullptr) {
        SolveParams sp = solve_params(c, task, quasi, want_grad);
        sp.out_map = out_dev;
        sp.z_in = z ? 1 : 0;
        if (z)
            for (int i = 0; i < c.r; ++i) sp.z[i] = z[i];
        cudaLaunchConfig_t cfg = {};
        // cooperative cluster launch: the kernel's own grid barrier (grid_barrier) needs every
        // CTA co-resident, which the cooperative attribute makes the driver guarantee (or
        // refuse the launch) even when other contexts or processes share the GPU.
        // LSB_NONCOOP=1 (profiling only) drops the attribute so ncu can replay the kernel.
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.gridDim = dim3(solve_grid);
        cfg.blockDim = dim3(kSolveThreads);
        cfg.dynamicSmemBytes = solve_smem;
        cfg.stream = c.stream;
        cfg.attrs = at;
        cfg.numAttrs = c.dev.noncoop ? 1 : 2;
        cuda_check(cudaLaunchKernelEx(&cfg, solve, ps, sp), "solve kernel launch");
        c.launches += 1;
    }

    bool has_solve() const override { return solve != nullptr; }
    void solve_eval(Context& c) override { launch_solve(c, 0, 0, 1); }
    void solve_minimize(Context& c) override { launch_solve(c, 1, 0); }
    void solve_step(Context& c, int quasi) override { launch_solve(c, 2, quasi); }

    void launch_gather_vjp(cudaStream_t s) {
        if (fuse_gather) {
            ks.vjp_gather<<<p.grid_vjp, kStreamThreads, vjpg_smem, s>>>(p);
        } else {
            gather_kernel<TS><<<grid_gather, 256, 0, s>>>(p);
            ks.vjp<<<p.grid_vjp, kStreamThreads, vjp_smem, s>>>(p);
        }
    }
    // graph form: returns the last node
    cudaGraphNode_t add_gather_vjp(cudaGraph_t g, cudaGraphNode_t dep, void** args, bool pdl = false) {
        if (fuse_gather)
            return add_kernel_pdl(g, dep, (void*)ks.vjp_gather, p.grid_vjp, vjpg_smem, args, kStreamThreads, pdl);
        cudaGraphNode_t n = add_kernel(g, dep, (void*)gather_kernel<TS>, grid_gather, 0, args);
        return add_kernel(g, n, (void*)ks.vjp, p.grid_vjp, vjp_smem, args, kStreamThreads);
    }

    void launch_ctrl(cudaStream_t s, int cmode, int smode, int want) {
        ctrl<<<cs, ctrl_threads, ctrl_smem, s>>>(pc, cmode, smode, want);
    }

    // One evaluation body, stream-launched (non-graph path).
    void launch_eval_body(cudaStream_t s, Context& c) {
        if (use_sweep) {
            launch_sweep(s);
            launch_ctrl(s, kCtrlAfterEval, 0, 0);
            c.launches += 2;
            return;
        }
        ks.out_fwd<<<p.grid_out, kStreamThreads, out_smem, s>>>(p);
        elem_fn<<<p.grid_elem, 256, 0, s>>>(p);
        launch_gather_vjp(s);
        launch_ctrl(s, kCtrlAfterEval, 0, 0);
        c.launches += fuse_gather ? 4 : 5;
    }

    void eval(Context& c, bool want_grad) override {
        if (solve && c.use_solve) {
            launch_solve(c, 0, 0, want_grad ? 1 : 0);
            return;
        }
        launch_eval_graph(c, want_grad);
    }

    void profile(Context& c, int reps, float* ms) override {
        cudaStream_t s = c.stream;
        cudaEvent_t ev[6];
        for (auto& e : ev) cuda_check(cudaEventCreate(&e), "event");
        double acc[5] = {0, 0, 0, 0, 0};
        for (int it = 0; it < reps; ++it) {
            cudaEventRecord(ev[0], s);
            launch_ctrl(s, kCtrlStart, kModeEval, 1);
            cudaEventRecord(ev[1], s);
            if (use_sweep) {
                launch_sweep(s);
                cudaEventRecord(ev[2], s);
                cudaEventRecord(ev[3], s);
                cudaEventRecord(ev[4], s);
            } else {
                ks.out_fwd<<<p.grid_out, kStreamThreads, out_smem, s>>>(p);
                cudaEventRecord(ev[2], s);
                elem_fn<<<p.grid_elem, 256, 0, s>>>(p);
                cudaEventRecord(ev[3], s);
                launch_gather_vjp(s);
                cudaEventRecord(ev[4], s);
            }
            launch_ctrl(s, kCtrlAfterEval, 0, 0);
            cudaEventRecord(ev[5], s);
            c.launches += use_sweep ? 3 : (fuse_gather ? 4 : 5);
            cuda_check(cudaEventSynchronize(ev[5]), "profile sync");
            float t;
            cudaEventElapsedTime(&t, ev[1], ev[2]);
            acc[0] += t;
            cudaEventElapsedTime(&t, ev[2], ev[3]);
            acc[1] += t;
            cudaEventElapsedTime(&t, ev[3], ev[4]);
            acc[2] += t;
            cudaEventElapsedTime(&t, ev[4], ev[5]);
            acc[3] += t;
            cudaEventElapsedTime(&t, ev[0], ev[5]);
            acc[4] += t;
        }
        for (int k = 0; k < 5; ++k) ms[k] = (float)(acc[k] / reps);
        for (auto& e : ev) cudaEventDestroy(e);
    }

    cudaGraphNode_t add_kernel(cudaGraph_t g, cudaGraphNode_t dep, void* fn, int grid, size_t smem, void** args,
                               int threads = 256) {
        cudaKernelNodeParams kp = {};
        kp.func = fn;
        kp.gridDim = dim3(grid);
        kp.blockDim = dim3(threads);
        kp.sharedMemBytes = (unsigned)smem;
        kp.kernelParams = args;
        cudaGraphNode_t nd;
        cuda_check(cudaGraphAddKernelNode(&nd, g, dep ? &dep : nullptr, dep ? 1 : 0, &kp), "kernel node");
        return nd;
    }
    // Kernel node whose edge from the kernel node `dep` is programmatic (PDL): its CTAs may start
    // once every CTA of `dep` has executed griddepcontrol.launch_dependents, and it orders its
    // dependent reads behind griddepcontrol.wait (full completion + memory of `dep`).
    cudaGraphNode_t add_kernel_pdl(cudaGraph_t g, cudaGraphNode_t dep, void* fn, int grid, size_t smem, void** args,
                                   int threads, bool pdl) {
        if (!pdl || !dep) return add_kernel(g, dep, fn, grid, smem, args, threads);
        cudaGraphNode_t nd = add_kernel(g, nullptr, fn, grid, smem, args, threads);
        cudaGraphEdgeData ed = {};
        ed.from_port = cudaGraphKernelNodePortProgrammatic;
        ed.type = cudaGraphDependencyTypeProgrammatic;
        cuda_check(cudaGraphAddDependencies_v2(g, &dep, &nd, &ed, 1), "programmatic edge");
        return nd;
    }

    // WHILE(cond){ out_fwd -> elem -> vjp -> ctrl } appended after `dep`.
    cudaGraphNode_t add_while(cudaGraph_t graph, cudaGraphNode_t dep, cudaGraphConditionalHandle* handle) {
        cuda_check(cudaGraphConditionalHandleCreate(handle, graph, 1, cudaGraphCondAssignDefault), "cond handle");
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = *handle;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t wnode;
        cuda_check(cudaGraphAddNode(&wnode, graph, dep ? &dep : nullptr, dep ? 1 : 0, &cp), "while node");
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        EvalParams<TS> pg = p;
        pg.in_graph = 1;
        pg.cond = *handle;
        EvalParams<TS> pcg = pc;
        pcg.in_graph = 1;
        pcg.cond = *handle;
        SweepParams sw = swp;
        void* a1[] = {&pg};
        void* asw[] = {&pg, &sw};
        int cm = kCtrlAfterEval, z0 = 0, z1 = 0;
        void* a4[] = {&pcg, &cm, &z0, &z1};
        cudaGraphNode_t n3;
        const int pm = pdl_mask;
        if (use_sweep) {
            n3 = add_kernel(body, nullptr, (void*)sweep, sweep_grid, sweep_smem, asw, kSwThreads);
        } else {
            cudaGraphNode_t n1 = add_kernel(body, nullptr, (void*)ks.out_fwd, p.grid_out, out_smem, a1, kStreamThreads);
            cudaGraphNode_t n2 = add_kernel_pdl(body, n1, (void*)elem_fn, p.grid_elem, 0, a1, 256, pm & 2);
            n3 = add_gather_vjp(body, n2, a1, pm & 4);
        }
        add_kernel_pdl(body, n3, (void*)ctrl, cs, ctrl_smem, a4, ctrl_threads, pm & 8);
        return wnode;
    }

    cudaGraphNode_t add_start(cudaGraph_t graph, cudaGraphNode_t dep) {
        int cm = kCtrlStart, mode = kModeLbfgs, want = 1;
        EvalParams<TS> pg = pc;
        void* args[] = {&pg, &cm, &mode, &want};
        return add_kernel(graph, dep, (void*)ctrl, cs, ctrl_smem, args, ctrl_threads);
    }

    void build_min_graph(Context& c) {
        cudaGraph_t g;
        cuda_check(cudaGraphCreate(&g, 0), "graph create");
        cudaGraphNode_t st = add_start(g, nullptr);
        add_while(g, st, &h_min);
        cuda_check(cudaGraphInstantiate(&g_min, g, 0), "graph instantiate (minimize)");
        cudaGraphDestroy(g);
    }

    void build_step_graph(Context& c) {
        cudaGraph_t g;
        cuda_check(cudaGraphCreate(&g, 0), "graph create");
        const int threads = 256;
        const int grid_n = std::max(1, std::min((p.n + threads - 1) / threads, c.num_sms * 8));
        const int grid_v = std::max(1, std::min((p.V + threads - 1) / threads, c.num_sms * 8));
        int n = p.n, r = p.r, V = p.V;
        const int* vfree = p.vfree;
        const double* u_state = c.d_u_state;
        const double* v_state = c.d_v_state;
        const double* a_ext = c.d_a_ext;
        const double* z_state = c.d_z_state;
        DevState* st = c.d_state;
        double* ut = c.d_ut;
        double* eprow = c.d_eprow;
        void* a_prep[] = {&n, &vfree, &u_state, &v_state, &a_ext, &z_state, &r, &st, &ut, &eprow};
        cudaGraphNode_t n_prep = add_kernel(g, nullptr, (void*)prep_step_kernel, grid_n, 0, a_prep);
        cudaGraphNode_t n_start = add_start(g, n_prep);
        cudaGraphNode_t n_while = add_while(g, n_start, &h_step);
        const double* U = c.d_U;
        const char* vpinned = c.d_vpinned;
        const double* pin_disp = c.d_pin_disp;
        double* u_st = c.d_u_state;
        double* v_st = c.d_v_state;
        double* z_st = c.d_z_state;
        void* a_fin[] = {&V, &U, &vpinned, &pin_disp, &u_st, &v_st, &z_st, &r, &st};
        cudaGraphNode_t n_fin = add_kernel(g, n_while, (void*)finalize_step_kernel, grid_v, 0, a_fin);
        long long* acc = c.d_launch_acc;
        const DevState* cst = c.d_state;
        int per_body = c.body_kernels;
        void* a_cnt[] = {&cst, &acc, &per_body};
        cudaKernelNodeParams kp = {};
        kp.func = (void*)count_loop_kernel;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(32);
        kp.kernelParams = a_cnt;
        cudaGraphNode_t n_cnt;
        cuda_check(cudaGraphAddKernelNode(&n_cnt, g, &n_fin, 1, &kp), "node count");
        cuda_check(cudaGraphInstantiate(&g_step, g, 0), "graph instantiate (step)");
        cudaGraphDestroy(g);
    }

    void minimize(Context& c) override {
        if (solve && c.use_solve) {
            launch_solve(c, 1, 0);
            return;
        }
        if (!g_min) build_min_graph(c);
        cuda_check(cudaGraphLaunch(g_min, c.stream), "graph launch (minimize)");
        c.launches += 1;  // start; loop bodies are counted from st->loop_iters
    }

    void step(Context& c) override {
        if (solve && c.use_solve) {
            launch_solve(c, 2, c.h_state->quasi_static);
            return;
        }
        if (!g_step) {
            c.ensure_step_buffers(1);
            build_step_graph(c);
        }
        cuda_check(cudaGraphLaunch(g_step, c.stream), "graph launch (step)");
        c.launches += 4;  // prep, start, finalize, count (bodies via device accumulator)
    }

    void rebind_elements(Context& c) override {
        for (EvalParams<TS>* q : {&p, &ps}) {
            q->E = c.mesh.E;
            q->tets = reinterpret_cast<const int4*>(c.d_tets);
            q->rec = static_cast<const TS*>(c.d_rec);
            q->forces = c.d_forces;
            q->csr_ptr = c.d_csr_ptr;
            q->csr_ent = c.d_csr_ent;
            q->fpos = reinterpret_cast<const int4*>(c.d_fpos);
        }
        p.grid_elem = std::max(1, std::min((c.mesh.E + 255) / 256, c.grid_elem_cap));
        c.grid_elem = p.grid_elem;
        ps.grid_elem = p.grid_elem;
        setup_sweep(c);
        invalidate_graphs();
    }

    void invalidate_graphs() override {
        if (g_min) cudaGraphExecDestroy(g_min);
        if (g_step) cudaGraphExecDestroy(g_step);
        for (auto& ge : g_eval) {
            if (ge) cudaGraphExecDestroy(ge);
            ge = nullptr;
        }
        g_min = g_step = nullptr;
    }
};

std::unique_ptr<ImplBase> make_impl(int precision) {
    if (precision == LSB_FP64) return std::unique_ptr<ImplBase>(new Impl<double>());
    return std::unique_ptr<ImplBase>(new Impl<float>());
}

}  // namespace lsb
