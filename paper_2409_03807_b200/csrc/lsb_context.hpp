// Context object behind the opaque lsb_context handle: host mesh/decoder
// copies, the HBM layout of every device buffer and the precision-specific
// kernel implementation.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lipsub_b200.h"
#include "lsb_kernels.cuh"
#include "lsb_setup.hpp"

namespace lsb {

extern thread_local std::string g_last_error;

struct LsbError : std::runtime_error {
    lsb_status code;
    LsbError(lsb_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void cuda_check(cudaError_t e, const char* what);

struct Context;

// Developer switches (A/B experiments, tests, profiling).  Read from the environment exactly
// once, when a context is created (lsb_create) -- never per launch -- and reported by
// lsb_get_dev_flags so a bench line records any that were set.  None changes results except
// LSB_SOLVE_EXP bits 1 and 4 (timing-only experiments that skip work), which are rejected
// unless the library is built with -DLSB_TIMING_EXPERIMENTS.
struct DevFlags {
    int tc = 1;               // LSB_TC=0: batched GEMMs on the CUDA-core SGEMM instead of tcgen05
    int fuse_gather = 1;      // LSB_FUSE_GATHER=0: separate vertex-gather kernel (multi-kernel path)
    int ctrl_cluster16 = 0;   // LSB_CTRL_CLUSTER=16: 16-CTA control clusters
    int ctrl_fast = 1;        // LSB_CTRL_FAST=0: generic control-cluster kernel
    int disable_solve = 0;    // LSB_DISABLE_SOLVE_KERNEL=1: multi-kernel path only
    int solve_tv_global = 0;  // LSB_SOLVE_TV_GLOBAL=1: persistent kernel's tv in global memory
    float ctrl_tile_w = -1.f; // LSB_CTRL_TILE_W: control CTAs' W_out tile share (<0: default)
    float pf_frac = 1.f;      // LSB_PREFETCH_FRAC: cold-start L2 prefetch fraction
    int solve_exp = 0;        // LSB_SOLVE_EXP: persistent-kernel A/B bits (lsb_solve.cuh SolveParams::exp)
    int trace = 0;            // LSB_TRACE=1: persistent-kernel phase timestamps
    int fuse_tangent_out = 1; // LSB_FUSE_TOUT=0: tangent output as its own kernel after the output GEMM (Hessian path)
    int hess3 = 1;            // LSB_HESS3=0: the D^T M' element Hessian kernel instead of the edge-space chained-MMA form
    int elem_f2 = 1;          // LSB_ELEM_F2=0: scalar batched element kernel instead of the packed fp32x2 one
    int theta_tb = 24;        // LSB_THETA_TB: tets per block of the theta element pass
    int noncoop = 0;          // LSB_NONCOOP=1: persistent kernel as a plain cluster launch (ncu replay)
    int elem_f32 = 1;         // LSB_ELEM_F32=0: fp64 element arithmetic in fp32-storage mode (multi-kernel path)
    int pdl = 5;              // LSB_PDL bit mask of programmatic edges (1 ctrl->out_fwd, 2 out_fwd->elem, 4 elem->vjp,
                              // 8 vjp->ctrl); 0: plain full-completion edges
    int l2_pf_elem = 0;       // LSB_L2PF_ELEM: VJP head tiles prefetched into L2 by the element pass (measured: slower)
    int l2_pf = 8;            // LSB_L2PF: W tiles per out_fwd CTA prefetched into L2 during the control kernel (PDL); 8 and 16
                              // measured 208.7 and 209.4 us per c3 evaluation, 0: 214.0, 32: 213.6 (tools/l2pf_ab.sh)
    int vjp_wg = 0;           // LSB_VJP_WG=1: per-warp, per-tile gather in the fused VJP (measured 1% slower than the prologue)
    int vjp_wg_cta = 3;       // LSB_VJP_WG_CTA: CTAs per SM of the per-warp-gather VJP
    int w_keep = 8;           // LSB_W_KEEP: W tiles at the end of every out_fwd CTA range kept in L2 (evict_last) for the VJP's
                              // re-read (c3: 29 MB; measured 212.8 -> 211.1 us per evaluation, 16+ tiles lose it again)
    int w_resident = -1;      // LSB_W_RESIDENT=0/1: force the W_out L2 policy (evict_first / evict_last)
    int solve_clusters = 0;   // LSB_SOLVE_CLUSTERS: cap on the persistent kernel's clusters (0: all that fit)
    int sweep = 0;            // LSB_SWEEP=1: fused warp-specialised sweep pass instead of out_fwd, elem, vjp (measured slower)
    float sweep_lag = 1.5f;   // LSB_SWEEP_LAG: ticket lag between an item and its dependencies, in grids
    std::string active;       // "NAME=value ..." of every switch found set
};
DevFlags read_dev_flags();

struct ImplBase {
    virtual ~ImplBase() = default;
    virtual void setup(Context& c) = 0;
    virtual void eval(Context& c, bool want_grad) = 0;
    virtual void minimize(Context& c) = 0;
    virtual void step(Context& c) = 0;
    virtual void profile(Context& c, int reps, float* ms) = 0;
    virtual void invalidate_graphs() = 0;
    // the element set changed (runtime cubature): re-point the element arrays, regrid
    virtual void rebind_elements(Context& c) = 0;
    // One evaluation at st->zt as a graph with event-record nodes:
    // ev[0] | ctrl(start) | ev[1] | out_fwd | ev[2] | elem, vjp, ctrl | ev[3]
    // Records ev[0] .. ev[3] around one evaluation (ev[1] .. ev[2]: the output-layer kernel)
    // and returns 4, or records only ev[0] and ev[3] around a single-launch evaluation and
    // returns 2 (every event record costs ~2.7 us of GPU time inside the bracket).
    virtual int eval_timed(Context& c, cudaEvent_t* ev, bool want_grad = true) = 0;
    // One evaluation at z with z passed by value and {E, status, grad} written by the kernel into
    // host-mapped memory out (device view out_dev); false when this path is unavailable.
    virtual bool eval_direct(Context& c, const double* z, bool want_grad, double* out_dev) = 0;
    // persistent solve kernel (one cooperative cluster launch per eval / solve / step)
    virtual bool has_solve() const = 0;
    virtual void solve_eval(Context& c) = 0;
    virtual void solve_minimize(Context& c) = 0;
    virtual void solve_step(Context& c, int quasi) = 0;
};
std::unique_ptr<ImplBase> make_impl(int precision);
void restore_user_objective(Context& c);

// Batched / second-order engines (lsb_batched.cu, lsb_hessian.cu).
struct BatchedBase {
    virtual ~BatchedBase() = default;
};

struct Context {
    int precision = LSB_FP64, device = 0, num_sms = 148;
    size_t wsize = 8;
    cudaStream_t stream = nullptr;
    int body_kernels = 5;  // kernels per multi-kernel evaluation body (out_fwd, elem, [gather,] vjp, ctrl)
    HostMesh mesh;
    std::vector<double> mass;        // n
    double total_mass = 0.0;
    std::vector<double> mu, lambda;  // E
    double density = 0.0;
    // decoder (host copy, fp64)
    int r = 0, n = 0, nhid = 0, h = 0, hp = 0, out_act = 0;
    std::vector<HostLayer> layers;   // all layers incl. output
    std::vector<double> shift, scale;
    int hoff[kMaxLayers] = {}, boff[kMaxLayers] = {}, hrows[kMaxLayers] = {}, hcols[kMaxLayers] = {},
        hact[kMaxLayers] = {};
    // objective host mirror
    std::vector<double> pin_positions;  // V*3
    int pins_version = 0;               // bumped by lsb_set_pin_positions: the batched engine re-lays its pinned rows
    bool has_qbar = false;
    double dt = 0.05;

    // ---- device buffers: W_out and rec in the storage precision (wsize), rest fp64 ----
    void* d_Wout = nullptr;  // n x hp
    double *d_bout = nullptr, *d_sout = nullptr, *d_cout = nullptr, *d_dsout = nullptr;
    double *d_mass = nullptr, *d_ut = nullptr, *d_rin = nullptr;
    double* d_ut_user = nullptr;  // qbar - X of the lsb_set_inertia objective (restored after steps)
    double* d_eprow = nullptr;  // n x 6 {b, s, shift - X, m, U slot, qbar - X}
    std::vector<double> h_eprow;
    double* d_tv = nullptr;     // n
    int* d_vfree = nullptr;
    int* d_tets = nullptr;
    void* d_rec = nullptr;
    double* d_U = nullptr;
    double* d_forces = nullptr;
    int *d_csr_ptr = nullptr, *d_csr_ent = nullptr;
    int* d_fpos = nullptr;  // E x 4 CSR positions of tet-slot forces
    double *d_Wh = nullptr, *d_bh = nullptr;
    float* d_Wh_f = nullptr;  // hidden weights in fp32 (solve kernel, fp32 mode)
    double* d_a_hid = nullptr;
    double* d_y_last = nullptr;
    size_t l2_bytes = 126u << 20;
    double *d_e_part_out = nullptr, *d_e_part_elem = nullptr, *d_ybar_part = nullptr, *d_ybar_grp = nullptr;
    unsigned int* d_grp_cnt = nullptr;
    DevState* d_state = nullptr;
    DevState* h_state = nullptr;  // pinned mirror
    double* h_out = nullptr;      // host-mapped {E, status, grad[kMaxLatent]} (direct evaluation)
    double* d_out = nullptr;      // its device view
    // dynamics
    double *d_u_state = nullptr, *d_v_state = nullptr, *d_z_state = nullptr, *d_a_ext = nullptr;
    double* d_pin_disp = nullptr;
    char* d_vpinned = nullptr;
    lsb_exit_report* d_reports = nullptr;
    double* d_z_traj = nullptr;
    int step_capacity = 0;
    bool state_set = false;
    long long* d_launch_acc = nullptr;
    long long launches = 0;
    int grid_out = 0, grid_elem = 0, grid_vjp = 0, solve_grid = 0;
    bool use_solve = true;
    std::string solve_reason;
    unsigned long long* d_sweep_trace = nullptr;  // sweep-pass item trace (LSB_TRACE=1), 4 words per ticket
    int sweep_tickets = 0;
    unsigned long long* d_trace = nullptr;  // solve-kernel phase trace (LSB_TRACE=1)  // route eval/minimize/step through the persistent kernel when available

    DevFlags dev;

    std::unique_ptr<ImplBase> impl;
    std::unique_ptr<BatchedBase> batched;
    std::unique_ptr<BatchedBase> refops;  // scratch of the reference-primitive operations (lsb_refops.cu)
    long long batched_launches = 0;
    std::vector<void*> allocations;
    void dfree(void* p);
    // runtime cubature (SolverConfig::runtime_cubature, reduced_solver.hpp:23): the full mesh and
    // material are kept here while `mesh`, `mu`, `lambda` hold the active (weighted) subset
    bool has_full = false;
    HostMesh mesh_full;
    std::vector<double> mu_full, lambda_full;
    int grid_elem_cap = 1;

    ~Context();
    void* dmalloc(size_t bytes);
    void copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, const char* what) const;
    void alloc_partials(int g_out, int g_elem, int g_vjp, int n_groups);
    void ensure_step_buffers(int steps);
    void upload_real(void* dst, const double* src, size_t count);  // converts to wsize
};

}  // namespace lsb

struct lsb_context {
    lsb::Context c;
};
