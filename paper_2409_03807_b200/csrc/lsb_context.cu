// Host side of the C ABI (include/lipsub_b200.h): context construction,
// HBM layout, kernel dispatch and the CUDA graphs that keep the L-BFGS loop
// and whole timesteps on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lipsub_b200.h"
#include "lsb_context.hpp"

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
                                 const double* a_ext, const double* z_state, int r, DevState* st, void* ut_out,
                                 int fp32) {
    const double dt = st->dt;
    const int quasi = st->quasi_static;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int f = i / 3, c = i - 3 * f;
        const size_t vi = (size_t)vfree[f] * 3 + c;
        const double ut = u_state[vi] + dt * v_state[vi] + (dt * dt) * a_ext[i];
        if (fp32) static_cast<float*>(ut_out)[i] = quasi ? 0.f : (float)ut;
        else static_cast<double*>(ut_out)[i] = quasi ? 0.0 : ut;
    }
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < r; i += blockDim.x) st->zt[i] = z_state[i];
        if (threadIdx.x == 0) {
            st->has_inertia = quasi ? 0 : 1;
            st->inv_dt2 = 1.0 / (dt * dt);
        }
    }
}

// x' = unpack(decode(z*)), v' = (x' - x) / dt over all V rows (:266-276), report.
__global__ void finalize_step_kernel(int V, const void* U, int fp32, const char* vpinned, const double* pin_disp,
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
            else un = fp32 ? (double)static_cast<const float*>(U)[(size_t)v * 4 + c]
                           : static_cast<const double*>(U)[(size_t)v * 4 + c];
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

__global__ void count_loop_kernel(const DevState* st, long long* acc) {
    // device-side launch accounting for WHILE-loop bodies: 3 kernels per body
    if (threadIdx.x == 0 && blockIdx.x == 0) acc[0] += 3LL * st->loop_iters;
}

// ------------------------------------------------------------------ Impl<T>
template <typename T>
struct KernelSet {
    void (*out_fwd)(const EvalParams<T>);
    void (*vjp)(const EvalParams<T>);
};

template <typename T, int HP>
KernelSet<T> kernels_for() {
    return {out_fwd_kernel<T, HP>, vjp_ctrl_kernel<T, HP>};
}

template <typename T>
KernelSet<T> select_kernels(int hp) {
    switch (hp) {
        case 32: return kernels_for<T, 32>();
        case 64: return kernels_for<T, 64>();
        case 128: return kernels_for<T, 128>();
        case 256: return kernels_for<T, 256>();
        case 512: return kernels_for<T, 512>();
    }
    throw LsbError(LSB_EINVAL, "decoder: unsupported padded width");
}

template <typename T>
struct Impl final : ImplBase {
    EvalParams<T> p{};
    KernelSet<T> ks{};
    size_t vjp_smem = 0, start_smem = 0;
    cudaGraphExec_t g_min = nullptr, g_step = nullptr;
    cudaGraphConditionalHandle h_min{}, h_step{};

    ~Impl() override {
        if (g_min) cudaGraphExecDestroy(g_min);
        if (g_step) cudaGraphExecDestroy(g_step);
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
        p.Wout = static_cast<const T*>(c.d_Wout);
        p.bout = static_cast<const T*>(c.d_bout);
        p.sout = static_cast<const T*>(c.d_sout);
        p.cout = static_cast<const T*>(c.d_cout);
        p.dsout = static_cast<T*>(c.d_dsout);
        p.mass = static_cast<const T*>(c.d_mass);
        p.ut = static_cast<const T*>(c.d_ut);
        p.rin = static_cast<T*>(c.d_rin);
        p.vfree = c.d_vfree;
        p.tets = reinterpret_cast<const int4*>(c.d_tets);
        p.rec = static_cast<const T*>(c.d_rec);
        p.U = static_cast<T*>(c.d_U);
        p.forces = static_cast<T*>(c.d_forces);
        p.csr_ptr = c.d_csr_ptr;
        p.csr_ent = c.d_csr_ent;
        p.Wh = c.d_Wh;
        p.WhT = c.d_WhT;
        p.bh = c.d_bh;
        for (int l = 0; l < c.nhid; ++l) {
            p.hoff[l] = c.hoff[l];
            p.boff[l] = c.boff[l];
            p.hrows[l] = c.hrows[l];
            p.hcols[l] = c.hcols[l];
            p.hact[l] = c.hact[l];
        }
        p.a_hid = c.d_a_hid;
        p.y_last = static_cast<T*>(c.d_y_last);
        p.st = c.d_state;
        ks = select_kernels<T>(c.hp);
        // grid sizing: persistent grids of (SMs x resident blocks)
        int occ = 0;
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ks.out_fwd, 256, 0), "occupancy out_fwd");
        p.grid_out = std::max(1, c.num_sms * std::max(1, occ));
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, elem_kernel<T>, 256, 0), "occupancy elem");
        p.grid_elem = std::max(1, std::min((m.E + 255) / 256, c.num_sms * std::max(1, occ)));
        p.vpb = 64;
        vjp_smem = std::max<size_t>(8 * (size_t)c.hp * sizeof(double) + 3 * p.vpb * sizeof(T),
                                    2 * kMaxHidden * sizeof(double));
        cuda_check(cudaFuncSetAttribute(ks.vjp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vjp_smem),
                   "smem attr vjp");
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ks.vjp, 256, vjp_smem), "occupancy vjp");
        const int nslab = (m.n_free + p.vpb - 1) / p.vpb;
        p.grid_vjp = std::max(1, std::min(nslab, c.num_sms * std::max(1, occ)));
        p.group = 16;
        p.n_groups = (p.grid_vjp + p.group - 1) / p.group;
        start_smem = 2 * kMaxHidden * sizeof(double);
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
    }

    // One evaluation body, stream-launched (non-graph path).
    void launch_eval_body(cudaStream_t s, Context& c) {
        ks.out_fwd<<<p.grid_out, 256, 0, s>>>(p);
        elem_kernel<T><<<p.grid_elem, 256, 0, s>>>(p);
        ks.vjp<<<p.grid_vjp, 256, vjp_smem, s>>>(p);
        c.launches += 3;
    }

    void eval(Context& c, bool want_grad) override {
        cudaStream_t s = c.stream;
        start_kernel<T><<<1, 256, start_smem, s>>>(p, kModeEval, want_grad ? 1 : 0);
        c.launches += 1;
        launch_eval_body(s, c);
        cuda_check(cudaGetLastError(), "eval launch");
    }

    void profile(Context& c, int reps, float* ms) override {
        cudaStream_t s = c.stream;
        cudaEvent_t ev[5];
        for (auto& e : ev) cuda_check(cudaEventCreate(&e), "event");
        double acc[4] = {0, 0, 0, 0};
        for (int it = 0; it < reps; ++it) {
            cudaEventRecord(ev[0], s);
            start_kernel<T><<<1, 256, start_smem, s>>>(p, kModeEval, 1);
            cudaEventRecord(ev[1], s);
            ks.out_fwd<<<p.grid_out, 256, 0, s>>>(p);
            cudaEventRecord(ev[2], s);
            elem_kernel<T><<<p.grid_elem, 256, 0, s>>>(p);
            cudaEventRecord(ev[3], s);
            ks.vjp<<<p.grid_vjp, 256, vjp_smem, s>>>(p);
            cudaEventRecord(ev[4], s);
            c.launches += 4;
            cuda_check(cudaEventSynchronize(ev[4]), "profile sync");
            float t;
            cudaEventElapsedTime(&t, ev[1], ev[2]);
            acc[0] += t;
            cudaEventElapsedTime(&t, ev[2], ev[3]);
            acc[1] += t;
            cudaEventElapsedTime(&t, ev[3], ev[4]);
            acc[2] += t;
            cudaEventElapsedTime(&t, ev[0], ev[4]);
            acc[3] += t;
        }
        for (int k = 0; k < 4; ++k) ms[k] = (float)(acc[k] / reps);
        for (auto& e : ev) cudaEventDestroy(e);
    }

    // WHILE(cond){ out_fwd -> elem -> vjp_ctrl } appended after `dep`.
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
        EvalParams<T> pg = p;
        pg.in_graph = 1;
        pg.cond = *handle;
        // kernel params are copied at node creation
        void* args[] = {&pg};
        cudaKernelNodeParams kp = {};
        kp.kernelParams = args;
        kp.blockDim = dim3(256);
        cudaGraphNode_t n1, n2, n3;
        kp.func = (void*)ks.out_fwd;
        kp.gridDim = dim3(p.grid_out);
        kp.sharedMemBytes = 0;
        cuda_check(cudaGraphAddKernelNode(&n1, body, nullptr, 0, &kp), "node out_fwd");
        kp.func = (void*)elem_kernel<T>;
        kp.gridDim = dim3(p.grid_elem);
        cuda_check(cudaGraphAddKernelNode(&n2, body, &n1, 1, &kp), "node elem");
        kp.func = (void*)ks.vjp;
        kp.gridDim = dim3(p.grid_vjp);
        kp.sharedMemBytes = (unsigned)vjp_smem;
        cuda_check(cudaGraphAddKernelNode(&n3, body, &n2, 1, &kp), "node vjp");
        return wnode;
    }

    cudaGraphNode_t add_start(cudaGraph_t graph, cudaGraphNode_t dep) {
        int mode = kModeLbfgs, want = 1;
        EvalParams<T> pg = p;
        void* args[] = {&pg, &mode, &want};
        cudaKernelNodeParams kp = {};
        kp.func = (void*)start_kernel<T>;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(256);
        kp.sharedMemBytes = (unsigned)start_smem;
        kp.kernelParams = args;
        cudaGraphNode_t nd;
        cuda_check(cudaGraphAddKernelNode(&nd, graph, dep ? &dep : nullptr, dep ? 1 : 0, &kp), "node start");
        return nd;
    }

    void build_min_graph(Context& c) {
        cudaGraph_t g;
        cuda_check(cudaGraphCreate(&g, 0), "graph create");
        cudaGraphNode_t st = add_start(g, nullptr);
        cudaGraphNode_t w = add_while(g, st, &h_min);
        (void)w;
        cuda_check(cudaGraphInstantiate(&g_min, g, 0), "graph instantiate (minimize)");
        cudaGraphDestroy(g);
    }

    void build_step_graph(Context& c) {
        cudaGraph_t g;
        cuda_check(cudaGraphCreate(&g, 0), "graph create");
        const int threads = 256;
        const int grid_n = std::max(1, std::min((p.n + threads - 1) / threads, c.num_sms * 8));
        const int grid_v = std::max(1, std::min((p.V + threads - 1) / threads, c.num_sms * 8));
        // prep
        int n = p.n, r = p.r, fp32 = sizeof(T) == 4 ? 1 : 0, V = p.V;
        const int* vfree = p.vfree;
        const double* u_state = c.d_u_state;
        const double* v_state = c.d_v_state;
        const double* a_ext = c.d_a_ext;
        const double* z_state = c.d_z_state;
        DevState* st = c.d_state;
        void* ut = c.d_ut;
        void* a_prep[] = {&n, &vfree, &u_state, &v_state, &a_ext, &z_state, &r, &st, &ut, &fp32};
        cudaKernelNodeParams kp = {};
        kp.func = (void*)prep_step_kernel;
        kp.gridDim = dim3(grid_n);
        kp.blockDim = dim3(threads);
        kp.kernelParams = a_prep;
        cudaGraphNode_t n_prep;
        cuda_check(cudaGraphAddKernelNode(&n_prep, g, nullptr, 0, &kp), "node prep");
        cudaGraphNode_t n_start = add_start(g, n_prep);
        cudaGraphNode_t n_while = add_while(g, n_start, &h_step);
        // finalize
        const void* U = c.d_U;
        const char* vpinned = c.d_vpinned;
        const double* pin_disp = c.d_pin_disp;
        double* u_st = c.d_u_state;
        double* v_st = c.d_v_state;
        double* z_st = c.d_z_state;
        void* a_fin[] = {&V, &U, &fp32, &vpinned, &pin_disp, &u_st, &v_st, &z_st, &r, &st};
        kp.func = (void*)finalize_step_kernel;
        kp.gridDim = dim3(grid_v);
        kp.kernelParams = a_fin;
        cudaGraphNode_t n_fin;
        cuda_check(cudaGraphAddKernelNode(&n_fin, g, &n_while, 1, &kp), "node finalize");
        long long* acc = c.d_launch_acc;
        const DevState* cst = c.d_state;
        void* a_cnt[] = {&cst, &acc};
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
        if (!g_min) build_min_graph(c);
        cuda_check(cudaGraphLaunch(g_min, c.stream), "graph launch (minimize)");
        c.launches += 1;  // start kernel; loop bodies are counted from st->loop_iters
    }

    void step(Context& c) override {
        if (!g_step) {
            c.ensure_step_buffers(1);
            build_step_graph(c);
        }
        cuda_check(cudaGraphLaunch(g_step, c.stream), "graph launch (step)");
        c.launches += 4;  // prep, start, finalize, count (bodies via device accumulator)
    }

    void invalidate_graphs() override {
        if (g_min) cudaGraphExecDestroy(g_min);
        if (g_step) cudaGraphExecDestroy(g_step);
        g_min = g_step = nullptr;
    }
};

std::unique_ptr<ImplBase> make_impl(int precision) {
    if (precision == LSB_FP64) return std::unique_ptr<ImplBase>(new Impl<double>());
    return std::unique_ptr<ImplBase>(new Impl<float>());
}

}  // namespace lsb
