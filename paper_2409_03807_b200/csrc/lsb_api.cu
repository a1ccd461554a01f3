// extern "C" entry points of include/lipsub_b200.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <chrono>
#include <cstddef>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/lipsub_b200.h"
#include "lsb_batched.hpp"
#include "lsb_context.hpp"
#include "lsb_newton.hpp"
#include "lsb_refops.hpp"

namespace lsb {
void bench_evals(Context& c, int K, const double* Z, size_t flush_bytes, double* eval_ms, double* out_ms, double* E,
                 bool want_grad);
void bench_call(Context& c, int reps, size_t flush_bytes, double* ms, const std::function<void()>& call);
void bench_steps(Context& c, int K, size_t flush_bytes, double* step_ms, lsb_exit_report* reps);
}  // namespace lsb

using namespace lsb;

namespace lsb {

Context::~Context() {
    if (stream) cudaStreamSynchronize(stream);
    impl.reset();
    batched.reset();
    for (void* p : allocations) cudaFree(p);
    if (h_state) cudaFreeHost(h_state);
    if (h_out) cudaFreeHost(h_out);
    if (stream) cudaStreamDestroy(stream);
}

void* Context::dmalloc(size_t bytes) {
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc");
    cuda_check(cudaMemsetAsync(p, 0, std::max<size_t>(bytes, 16), stream), "cudaMemset");
    allocations.push_back(p);
    return p;
}

// Every host<->device copy of a context goes through its (non-blocking) stream and
// waits for it: copies are then ordered after the allocation memsets and kernels
// queued on that stream (a legacy-stream cudaMemcpy is not).
void Context::dfree(void* p) {
    if (!p) return;
    for (size_t i = 0; i < allocations.size(); ++i)
        if (allocations[i] == p) {
            cudaFree(p);
            allocations.erase(allocations.begin() + (long)i);
            return;
        }
}

void Context::copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, const char* what) const {
    cuda_check(cudaMemcpyAsync(dst, src, bytes, kind, stream), what);
    cuda_check(cudaStreamSynchronize(stream), what);
}

void Context::upload_real(void* dst, const double* src, size_t count) {
    if (wsize == 8) {
        copy(dst, src, count * 8, cudaMemcpyHostToDevice, "upload");
    } else {
        std::vector<float> tmp(count);
        for (size_t i = 0; i < count; ++i) tmp[i] = static_cast<float>(src[i]);
        copy(dst, tmp.data(), count * 4, cudaMemcpyHostToDevice, "upload");
    }
}

void Context::alloc_partials(int g_out, int g_elem, int g_vjp, int n_groups) {
    d_e_part_out = static_cast<double*>(dmalloc(sizeof(double) * g_out));
    d_e_part_elem = static_cast<double*>(dmalloc(sizeof(double) * g_elem));
    d_ybar_part = static_cast<double*>(dmalloc(sizeof(double) * (size_t)g_vjp * hp));
    d_ybar_grp = static_cast<double*>(dmalloc(sizeof(double) * (size_t)n_groups * hp));
    d_grp_cnt = static_cast<unsigned int*>(dmalloc(sizeof(unsigned int) * n_groups));
}

void Context::ensure_step_buffers(int steps) {
    if (steps <= step_capacity) return;
    const int cap = std::max(steps, 2 * step_capacity);
    d_reports = static_cast<lsb_exit_report*>(dmalloc(sizeof(lsb_exit_report) * cap));
    d_z_traj = static_cast<double*>(dmalloc(sizeof(double) * (size_t)cap * r));
    step_capacity = cap;
    void* rp = d_reports;
    double* zp = d_z_traj;
    cuda_check(cudaMemcpyAsync(&d_state->reports, &rp, sizeof(void*), cudaMemcpyHostToDevice, stream), "reports ptr");
    cuda_check(cudaMemcpyAsync(&d_state->z_traj, &zp, sizeof(double*), cudaMemcpyHostToDevice, stream), "ztraj ptr");
    cuda_check(cudaStreamSynchronize(stream), "sync");
}

}  // namespace lsb

namespace {

lsb_status run(const std::function<void()>& f) {
    try {
        f();
        return LSB_OK;
    } catch (const LsbError& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return LSB_EINVAL;
    } catch (const std::bad_alloc& e) {
        g_last_error = "out of host memory";
        return LSB_ECUDA;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return LSB_EMESH;
    }
}

void require(bool ok, const std::string& msg, lsb_status code = LSB_EINVAL) {
    if (!ok) throw LsbError(code, msg);
}

void check_ctx(const lsb_context* ctx) { require(ctx != nullptr, "null context"); }

void sync(Context& c) { cuda_check(cudaStreamSynchronize(c.stream), "stream sync"); }

// Write a field of the device state from the host (async on the context stream).
template <typename F>
void put_state(Context& c, F DevState::*field, const F& value) {
    static thread_local F tmp;
    tmp = value;
    cuda_check(cudaMemcpyAsync(&(c.d_state->*field), &tmp, sizeof(F), cudaMemcpyHostToDevice, c.stream), "state put");
    sync(c);
}

void put_config(Context& c, const lsb_solver_config* cfg) {
    require(cfg != nullptr, "solver: null config");
    // reference SolverConfig::validate (reduced_solver.cpp:14-20)
    require(cfg->epsilon > 0.0, "solver: epsilon must be > 0");
    require(cfg->max_iters >= 1 && cfg->max_linesearch >= 1, "solver: iteration caps must be >= 1");
    require(cfg->dt > 0.0, "solver: dt must be > 0");
    require(cfg->lbfgs_history >= 1, "solver: lbfgs history must be >= 1");
    require(cfg->lbfgs_history <= kMaxHistory, "solver: lbfgs history exceeds device maximum 16");
    DevState* h = c.h_state;
    cuda_check(cudaMemcpyAsync(h, c.d_state, sizeof(DevState), cudaMemcpyDeviceToHost, c.stream), "state get");
    sync(c);
    h->eps = cfg->epsilon;
    h->max_iters = cfg->max_iters;
    h->max_ls = cfg->max_linesearch;
    h->hist_cap = cfg->lbfgs_history;
    h->dt = cfg->dt;
    cuda_check(cudaMemcpyAsync(c.d_state, h, sizeof(DevState), cudaMemcpyHostToDevice, c.stream), "state put");
    sync(c);
}

void get_state(Context& c) {
    cuda_check(cudaMemcpyAsync(c.h_state, c.d_state, sizeof(DevState), cudaMemcpyDeviceToHost, c.stream), "state get");
    sync(c);
}

void fill_report(const DevState* s, lsb_exit_report* rep) {
    if (!rep) return;
    rep->code = s->code;
    rep->iterations = s->iter;
    rep->final_grad_inf_norm = s->gnorm;
    rep->wall_time_ms = (double)(s->t_end - s->t_start) * 1e-6;
    rep->value_evals = s->value_evals;
    rep->grad_evals = s->grad_evals;
}

void upload_pins(Context& c) {
    // pinned rows of U get pin - X; free rows are overwritten by every decode
    const HostMesh& m = c.mesh;
    std::vector<double> disp(3 * (size_t)m.V, 0.0);
    for (int v : m.pinned)
        for (int k = 0; k < 3; ++k) disp[3 * (size_t)v + k] = c.pin_positions[3 * (size_t)v + k] - m.X[3 * (size_t)v + k];
    c.copy(c.d_pin_disp, disp.data(), disp.size() * 8, cudaMemcpyHostToDevice, "pins");
    std::vector<double> U4(4 * (size_t)m.V, 0.0);
    for (int v : m.pinned)
        for (int k = 0; k < 3; ++k) U4[4 * (size_t)v + k] = disp[3 * (size_t)v + k];
    // free rows: keep whatever the last decode wrote (re-uploading zeros is harmless
    // because every evaluation rewrites them before the element pass).
    c.copy(c.d_U, U4.data(), U4.size() * 8, cudaMemcpyHostToDevice, "U pins");
}

}  // namespace

namespace lsb {
DevFlags read_dev_flags() {
    DevFlags f;
    auto get = [&](const char* name) -> const char* {
        const char* v = getenv(name);
        if (v && *v) f.active += std::string(f.active.empty() ? "" : " ") + name + "=" + v;
        return (v && *v) ? v : nullptr;
    };
    if (const char* v = get("LSB_TC")) f.tc = v[0] != '0';
    if (const char* v = get("LSB_FUSE_GATHER")) f.fuse_gather = v[0] != '0';
    if (const char* v = get("LSB_CTRL_CLUSTER")) f.ctrl_cluster16 = atoi(v) == 16;
    if (const char* v = get("LSB_CTRL_FAST")) f.ctrl_fast = v[0] != '0';
    if (const char* v = get("LSB_DISABLE_SOLVE_KERNEL")) f.disable_solve = v[0] == '1';
    if (const char* v = get("LSB_SOLVE_TV_GLOBAL")) f.solve_tv_global = v[0] == '1';
    if (const char* v = get("LSB_CTRL_TILE_W")) f.ctrl_tile_w = (float)atof(v);
    if (const char* v = get("LSB_PREFETCH_FRAC")) f.pf_frac = std::min(1.0f, std::max(0.0f, (float)atof(v)));
    if (const char* v = get("LSB_SOLVE_EXP")) f.solve_exp = atoi(v);
    if (const char* v = get("LSB_TRACE")) f.trace = v[0] == '1';
    if (const char* v = get("LSB_FUSE_TOUT")) f.fuse_tangent_out = v[0] != '0';
    if (const char* v = get("LSB_HESS3")) f.hess3 = v[0] != '0';
    if (const char* v = get("LSB_ELEM_F2")) f.elem_f2 = v[0] != '0';
    if (const char* v = get("LSB_THETA_TB")) f.theta_tb = std::max(1, std::min(48, atoi(v)));
    if (const char* v = get("LSB_NONCOOP")) f.noncoop = v[0] == '1';
    if (const char* v = get("LSB_SWEEP")) f.sweep = v[0] == '1';
    if (const char* v = get("LSB_PDL")) f.pdl = atoi(v) & 15;
    if (const char* v = get("LSB_VJP_WG")) f.vjp_wg = v[0] != '0';
    if (const char* v = get("LSB_SOLVE_CLUSTERS")) f.solve_clusters = std::max(0, atoi(v));
    if (const char* v = get("LSB_W_RESIDENT")) f.w_resident = v[0] == '1' ? 1 : 0;
    if (const char* v = get("LSB_VJP_WG_CTA")) f.vjp_wg_cta = std::max(1, std::min(4, atoi(v)));
    if (const char* v = get("LSB_L2PF")) f.l2_pf = std::max(0, std::min(256, atoi(v)));
    if (const char* v = get("LSB_W_KEEP")) f.w_keep = std::max(0, std::min(4096, atoi(v)));
    if (const char* v = get("LSB_L2PF_ELEM")) f.l2_pf_elem = std::max(0, std::min(256, atoi(v)));
    if (const char* v = get("LSB_ELEM_F32")) f.elem_f32 = v[0] != '0';
    if (const char* v = get("LSB_SWEEP_LAG")) f.sweep_lag = std::min(8.0f, std::max(0.0f, (float)atof(v)));
#ifndef LSB_TIMING_EXPERIMENTS
    // bits 1 / 4 skip the tile math / the tv gather: results invalid, timing builds only
    if (f.solve_exp & (1 | 4))
        throw LsbError(LSB_EINVAL, "LSB_SOLVE_EXP bits 1/4 (results invalid) need a -DLSB_TIMING_EXPERIMENTS build");
#endif
    return f;
}
}  // namespace lsb

extern "C" {

const char* lsb_last_error(void) { return g_last_error.c_str(); }
const char* lsb_version(void) { return "lipsub_b200 0.1 (sm_100a)"; }

lsb_status lsb_bar_mesh_size(int nx, int ny, int nz, int pin_left, int* V, int* E, int* num_pinned) {
    return run([&] {
        require(nx >= 1 && ny >= 1 && nz >= 1, "bar: grid sizes must be >= 1");
        if (V) *V = (nx + 1) * (ny + 1) * (nz + 1);
        if (E) *E = 6 * nx * ny * nz;
        if (num_pinned) *num_pinned = pin_left ? (ny + 1) * (nz + 1) : 0;
    });
}

lsb_status lsb_make_bar_mesh(int nx, int ny, int nz, double width, double height, double depth, double jitter_frac,
                             uint64_t seed, int pin_left, double* rest_positions, int32_t* tets, int32_t* pinned) {
    return run([&] {
        const HostMesh m = make_bar_mesh(nx, ny, nz, width, height, depth, jitter_frac, seed, pin_left != 0);
        if (rest_positions) std::memcpy(rest_positions, m.X.data(), m.X.size() * 8);
        if (tets) std::memcpy(tets, m.T.data(), m.T.size() * 4);
        if (pinned) std::memcpy(pinned, m.pinned.data(), m.pinned.size() * 4);
    });
}

lsb_status lsb_make_bar_decoder(int V, const double* rest_positions, int num_pinned, const int32_t* pinned,
                                int latent_dim, int hidden_layers, int width, int act, uint64_t seed, double out_scale,
                                double* weights_packed, double* norm_shift, double* norm_scale) {
    return run([&] {
        require(V > 0 && rest_positions != nullptr, "decoder: mesh required");
        HostMesh m;
        m.V = V;
        m.X.assign(rest_positions, rest_positions + 3 * (size_t)V);
        m.pinned.assign(pinned, pinned + num_pinned);
        // free numbering only (no elements needed)
        std::vector<char> pin(V, 0);
        for (int v : m.pinned) {
            require(v >= 0 && v < V, "decoder: pinned vertex out of range");
            pin[v] = 1;
        }
        m.free_index.assign(V, -1);
        for (int v = 0; v < V; ++v)
            if (!pin[v]) {
                m.free_index[v] = (int)m.free_vertex.size();
                m.free_vertex.push_back(v);
            }
        m.n_free = (int)m.free_vertex.size();
        const HostDecoder d = make_bar_decoder(m, latent_dim, hidden_layers, width, act, seed, out_scale);
        size_t off = 0;
        for (const HostLayer& L : d.layers) {
            if (weights_packed) std::memcpy(weights_packed + off, L.W.data(), L.W.size() * 8);
            off += L.W.size();
        }
        if (norm_shift) std::memcpy(norm_shift, d.shift.data(), d.shift.size() * 8);
        if (norm_scale) std::memcpy(norm_scale, d.scale.data(), d.scale.size() * 8);
    });
}

lsb_status lsb_lame_from_young(int num_tets, double E_lo, double E_hi, double nu, uint64_t seed, double* mu,
                               double* lambda) {
    return run([&] {
        require(num_tets >= 0 && mu && lambda, "material: bad arguments");
        require(E_lo > 0.0 && E_hi >= E_lo, "material: Young's modulus range must be positive");
        require(nu > -1.0 && nu < 0.5, "material: Poisson ratio must be in (-1, 0.5)");
        Rng rng = substream(seed, 2);
        for (int e = 0; e < num_tets; ++e) {
            const double E = E_hi > E_lo ? E_lo + (E_hi - E_lo) * randu(rng) : E_lo;
            mu[e] = E / (2.0 * (1.0 + nu));
            lambda[e] = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
        }
    });
}

lsb_status lsb_gaussian_stream(uint64_t seed, uint64_t tag, int count, double std_dev, double* out) {
    return run([&] {
        require(count >= 0 && (count == 0 || out), "gaussian_stream: bad arguments");
        Rng rng = substream(seed, tag);
        for (int i = 0; i < count; ++i) out[i] = std_dev * randn(rng);
    });
}

// Element-set device arrays (tets, records {Dm^-1, vol, mu, lambda}, CSR-ordered force
// slots, fpos, CSR) from c.mesh / c.mu / c.lambda; previous buffers are released.
static void upload_elements(Context& c) {
    const HostMesh& m = c.mesh;
    const size_t w = c.wsize;
    for (void* q : {(void*)c.d_tets, c.d_rec, (void*)c.d_forces, (void*)c.d_fpos, (void*)c.d_csr_ptr, (void*)c.d_csr_ent})
        c.dfree(q);
    c.d_tets = static_cast<int*>(c.dmalloc(sizeof(int) * 4 * std::max<size_t>(1, (size_t)m.E)));
    if (m.E) c.copy(c.d_tets, m.T.data(), sizeof(int) * 4 * (size_t)m.E, cudaMemcpyHostToDevice, "tets");
    {
        std::vector<double> rec(12 * std::max<size_t>(1, (size_t)m.E), 0.0);
        for (int e = 0; e < m.E; ++e) {
            double* o = &rec[12 * (size_t)e];
            std::copy(&m.Dminv[9 * (size_t)e], &m.Dminv[9 * (size_t)e] + 9, o);
            o[9] = m.vol[e];
            o[10] = c.mu[e];
            o[11] = c.lambda[e];
        }
        c.d_rec = c.dmalloc(rec.size() * w);
        c.upload_real(c.d_rec, rec.data(), rec.size());
    }
    c.d_forces = static_cast<double*>(c.dmalloc(4 * std::max<size_t>(1, m.csr_ent.size()) * 8));
    {  // CSR position of each (tet, slot) force; -1 for pinned vertices
        std::vector<int> fpos(4 * std::max<size_t>(1, (size_t)m.E), -1);
        for (int f = 0; f < m.n_free; ++f)
            for (int k = m.csr_ptr[f]; k < m.csr_ptr[f + 1]; ++k) fpos[m.csr_ent[k]] = k;
        c.d_fpos = static_cast<int*>(c.dmalloc(fpos.size() * 4));
        c.copy(c.d_fpos, fpos.data(), fpos.size() * 4, cudaMemcpyHostToDevice, "fpos");
    }
    c.d_csr_ptr = static_cast<int*>(c.dmalloc(sizeof(int) * (m.n_free + 1)));
    c.copy(c.d_csr_ptr, m.csr_ptr.data(), sizeof(int) * (m.n_free + 1), cudaMemcpyHostToDevice, "csr");
    c.d_csr_ent = static_cast<int*>(c.dmalloc(sizeof(int) * std::max<size_t>(1, m.csr_ent.size())));
    if (!m.csr_ent.empty())
        c.copy(c.d_csr_ent, m.csr_ent.data(), sizeof(int) * m.csr_ent.size(), cudaMemcpyHostToDevice, "csr");
}

lsb_status lsb_create(const lsb_mesh_desc* mesh, const lsb_decoder_desc* dec, int precision, int device,
                      lsb_context** out) {
    return run([&] {
        require(mesh && dec && out, "create: null argument");
        require(precision == LSB_FP64 || precision == LSB_FP32, "create: precision must be LSB_FP64 or LSB_FP32");
        *out = nullptr;
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw LsbError(LSB_ECUDA, "no CUDA device available (the B200 path has no CPU fallback)");
        require(device >= 0 && device < ndev, "create: device index out of range");
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        cuda_check(cudaGetDeviceProperties(&prop, device), "device props");
        if (prop.major < 10)
            throw LsbError(LSB_ECUDA, std::string("device ") + prop.name + " is not sm_100 (built for sm_100a only)");

        auto holder = std::make_unique<lsb_context>();
        Context& c = holder->c;
        c.precision = precision;
        c.device = device;
        c.num_sms = prop.multiProcessorCount;
        c.l2_bytes = (size_t)prop.l2CacheSize;
        c.wsize = precision == LSB_FP64 ? 8 : 4;
        c.dev = read_dev_flags();
        cuda_check(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking), "stream");

        // ---- mesh (build_mesh semantics) ----
        require(mesh->num_vertices > 0 && mesh->num_tets > 0, "mesh: empty mesh");
        require(mesh->rest_positions && mesh->tets, "mesh: null arrays");
        require(mesh->num_pinned >= 0 && (mesh->num_pinned == 0 || mesh->pinned), "mesh: bad pin list");
        HostMesh& m = c.mesh;
        m.V = mesh->num_vertices;
        m.E = mesh->num_tets;
        m.X.assign(mesh->rest_positions, mesh->rest_positions + 3 * (size_t)m.V);
        m.T.assign(mesh->tets, mesh->tets + 4 * (size_t)m.E);
        m.pinned.assign(mesh->pinned, mesh->pinned + mesh->num_pinned);
        try {
            precompute(m);
        } catch (const std::invalid_argument& e) {
            throw LsbError(LSB_EINVAL, e.what());
        } catch (const std::runtime_error& e) {
            throw LsbError(LSB_EMESH, e.what());
        }
        require(m.n_free > 0, "mesh: every vertex is pinned");
        require(mesh->mu && mesh->lambda, "material: null mu/lambda");
        c.mu.assign(mesh->mu, mesh->mu + m.E);
        c.lambda.assign(mesh->lambda, mesh->lambda + m.E);
        for (int e = 0; e < m.E; ++e) {  // MaterialParams::validate (mesh.cpp:12-18)
            require(c.mu[e] > 0.0, "material: mu must be > 0");
            require(c.lambda[e] >= 0.0, "material: lambda must be >= 0");
        }
        c.density = mesh->density;
        c.mass = lump_mass(m, mesh->density, &c.total_mass);
        c.n = 3 * m.n_free;
        c.pin_positions = m.X;

        // ---- decoder (SubspaceModel::validate, net.cpp:66-88) ----
        require(dec->latent_dim >= 1 && dec->latent_dim <= kMaxLatent, "model: latent dim must be in [1, 64]");
        require(dec->num_layers >= 1 && dec->num_layers - 1 <= kMaxLayers, "model: bad layer count");
        require(dec->rows && dec->cols && dec->activations && dec->weights && dec->biases, "model: null arrays");
        require(dec->norm_shift && dec->norm_scale, "model: normalization vectors required");
        c.r = dec->latent_dim;
        const int L = dec->num_layers;
        int width = c.r;
        for (int l = 0; l < L; ++l) {
            require(dec->cols[l] == width, "model: decoder layer shapes do not chain");
            require(dec->rows[l] >= 1, "model: empty layer");
            require(dec->activations[l] >= 0 && dec->activations[l] <= 3, "activation: unknown tag");
            require(dec->weights[l] && dec->biases[l], "model: null layer arrays");
            HostLayer hl;
            hl.rows = dec->rows[l];
            hl.cols = dec->cols[l];
            hl.act = dec->activations[l];
            hl.W.assign(dec->weights[l], dec->weights[l] + (size_t)hl.rows * hl.cols);
            hl.b.assign(dec->biases[l], dec->biases[l] + hl.rows);
            c.layers.push_back(std::move(hl));
            width = dec->rows[l];
        }
        require(width == c.n, "model: decoder output width != n (3 x free vertices)");
        c.shift.assign(dec->norm_shift, dec->norm_shift + c.n);
        c.scale.assign(dec->norm_scale, dec->norm_scale + c.n);
        for (double s : c.scale) require(s > 0.0, "model: norm_scale entries must be positive");
        c.nhid = L - 1;
        c.h = c.layers[L - 1].cols;
        require(c.h <= kMaxHidden, "model: hidden width exceeds device maximum 512");
        for (int l = 0; l < c.nhid; ++l) require(c.layers[l].rows <= kMaxHidden, "model: hidden width exceeds 512");
        c.out_act = c.layers[L - 1].act;
        c.hp = 32;
        while (c.hp < c.h) c.hp *= 2;
        if (precision == LSB_FP64) c.hp = std::max(c.hp, 64);  // >= 32 lanes x double2
        else c.hp = std::max(c.hp, 128);                          // >= 32 lanes x float4

        const size_t w = c.wsize;
        const int n = c.n;
        // ---- HBM layout ----
        // output layer, rows padded to hp
        {
            std::vector<double> Wp((size_t)n * c.hp, 0.0);
            const HostLayer& o = c.layers[L - 1];
            for (int i = 0; i < n; ++i)
                std::copy(&o.W[(size_t)i * c.h], &o.W[(size_t)i * c.h] + c.h, &Wp[(size_t)i * c.hp]);
            c.d_Wout = c.dmalloc(Wp.size() * w);
            c.upload_real(c.d_Wout, Wp.data(), Wp.size());
            c.d_bout = static_cast<double*>(c.dmalloc(n * 8));
            c.copy(c.d_bout, o.b.data(), n * 8, cudaMemcpyHostToDevice, "bout");
        }
        c.d_sout = static_cast<double*>(c.dmalloc(n * 8));
        c.copy(c.d_sout, c.scale.data(), n * 8, cudaMemcpyHostToDevice, "sout");
        {
            std::vector<double> cs(n);
            for (int f = 0; f < m.n_free; ++f)
                for (int k = 0; k < 3; ++k)
                    cs[3 * f + k] = c.shift[3 * f + k] - m.X[3 * (size_t)m.free_vertex[f] + k];
            c.d_cout = static_cast<double*>(c.dmalloc(n * 8));
            c.copy(c.d_cout, cs.data(), n * 8, cudaMemcpyHostToDevice, "cout");
        }
        c.d_dsout = static_cast<double*>(c.dmalloc(n * 8));
        c.d_mass = static_cast<double*>(c.dmalloc(n * 8));
        c.copy(c.d_mass, c.mass.data(), n * 8, cudaMemcpyHostToDevice, "mass");
        c.d_ut = static_cast<double*>(c.dmalloc((n + 2) * 8));  // +2: 16-byte TMA tails
        c.d_rin = static_cast<double*>(c.dmalloc(n * 8));
        c.d_tv = static_cast<double*>(c.dmalloc((n + 2) * 8));
        {  // per-row side data staged with every W_out tile
            std::vector<double> ep(6 * (size_t)n, 0.0);
            const HostLayer& o = c.layers[L - 1];
            for (int f = 0; f < m.n_free; ++f)
                for (int k = 0; k < 3; ++k) {
                    const int i = 3 * f + k;
                    ep[6 * (size_t)i + 0] = o.b[i];
                    ep[6 * (size_t)i + 1] = c.scale[i];
                    ep[6 * (size_t)i + 2] = c.shift[i] - m.X[3 * (size_t)m.free_vertex[f] + k];
                    ep[6 * (size_t)i + 3] = c.mass[i];
                    ep[6 * (size_t)i + 4] = (double)(4 * m.free_vertex[f] + k);
                }
            c.h_eprow = ep;
            c.d_eprow = static_cast<double*>(c.dmalloc(ep.size() * 8));
            c.copy(c.d_eprow, ep.data(), ep.size() * 8, cudaMemcpyHostToDevice, "eprow");
        }
        c.d_vfree = static_cast<int*>(c.dmalloc(sizeof(int) * m.n_free));
        c.copy(c.d_vfree, m.free_vertex.data(), sizeof(int) * m.n_free, cudaMemcpyHostToDevice, "vfree");
        upload_elements(c);
        c.d_U = static_cast<double*>(c.dmalloc(4 * (size_t)m.V * 8));
        {  // hidden layers, fp64, row-major and transposed
            std::vector<double> Wh, bh;
            for (int l = 0; l < c.nhid; ++l) {
                const HostLayer& hl = c.layers[l];
                // offsets multiple of 4 elements: 16-byte aligned layer starts for the bulk-copy
                // staging in both fp64 and fp32 copies
                while (Wh.size() & 3) Wh.push_back(0.0);
                while (bh.size() & 3) bh.push_back(0.0);
                c.hoff[l] = (int)Wh.size();
                c.boff[l] = (int)bh.size();
                c.hrows[l] = hl.rows;
                c.hcols[l] = hl.cols;
                c.hact[l] = hl.act;
                Wh.insert(Wh.end(), hl.W.begin(), hl.W.end());
                bh.insert(bh.end(), hl.b.begin(), hl.b.end());
            }
            c.d_Wh = static_cast<double*>(c.dmalloc(8 * std::max<size_t>(1, Wh.size())));
            c.d_bh = static_cast<double*>(c.dmalloc(8 * std::max<size_t>(1, bh.size())));
            {  // storage-precision copy for the solve kernel's control cluster (fp32 mode)
                std::vector<float> wf(Wh.begin(), Wh.end());
                c.d_Wh_f = static_cast<float*>(c.dmalloc(4 * std::max<size_t>(1, wf.size())));
                if (!wf.empty()) c.copy(c.d_Wh_f, wf.data(), 4 * wf.size(), cudaMemcpyHostToDevice, "Wh f32");
            }
            if (!Wh.empty()) {
                c.copy(c.d_Wh, Wh.data(), 8 * Wh.size(), cudaMemcpyHostToDevice, "Wh");
                c.copy(c.d_bh, bh.data(), 8 * bh.size(), cudaMemcpyHostToDevice, "bh");
            }
        }
        c.d_a_hid = static_cast<double*>(c.dmalloc(sizeof(double) * kMaxHidden * std::max(1, c.nhid)));
        c.d_y_last = static_cast<double*>(c.dmalloc(c.hp * 8));
        c.d_state = static_cast<DevState*>(c.dmalloc(sizeof(DevState)));
        cuda_check(cudaMallocHost(&c.h_state, sizeof(DevState)), "pinned state");
        if (cudaHostAlloc(&c.h_out, sizeof(double) * (2 + kMaxLatent), cudaHostAllocMapped) == cudaSuccess) {
            if (cudaHostGetDevicePointer(&c.d_out, c.h_out, 0) != cudaSuccess) {
                cudaFreeHost(c.h_out);
                c.h_out = nullptr;
                c.d_out = nullptr;
            }
        } else {
            c.h_out = nullptr;
        }
        cudaGetLastError();
        std::memset(c.h_state, 0, sizeof(DevState));
        // dynamics
        c.d_u_state = static_cast<double*>(c.dmalloc(sizeof(double) * 3 * (size_t)m.V));
        c.d_v_state = static_cast<double*>(c.dmalloc(sizeof(double) * 3 * (size_t)m.V));
        c.d_z_state = static_cast<double*>(c.dmalloc(sizeof(double) * c.r));
        c.d_a_ext = static_cast<double*>(c.dmalloc(sizeof(double) * n));
        c.d_pin_disp = static_cast<double*>(c.dmalloc(sizeof(double) * 3 * (size_t)m.V));
        {
            std::vector<char> vp(m.V, 0);
            for (int v : m.pinned) vp[v] = 1;
            c.d_vpinned = static_cast<char*>(c.dmalloc(m.V));
            c.copy(c.d_vpinned, vp.data(), m.V, cudaMemcpyHostToDevice, "vpinned");
        }
        c.d_launch_acc = static_cast<long long*>(c.dmalloc(sizeof(long long)));
        cuda_check(cudaStreamSynchronize(c.stream), "sync");
        upload_pins(c);
        if (c.dev.trace) c.d_trace = static_cast<unsigned long long*>(c.dmalloc(8 * 2048));
        c.impl = make_impl(precision);
        c.impl->setup(c);
        // defaults: dt 0.05 (SolverConfig), history 8, no inertia
        DevState* h = c.h_state;
        std::memset(h, 0, sizeof(DevState));
        h->dt = 0.05;
        h->inv_dt2 = 1.0 / (0.05 * 0.05);
        h->has_inertia = 0;
        h->eps = 1e-5;
        h->max_iters = 1024;
        h->max_ls = 128;
        h->hist_cap = 8;
        h->phase = kPhaseDone;
        c.copy(c.d_state, h, sizeof(DevState), cudaMemcpyHostToDevice, "state init");
        c.ensure_step_buffers(16);
        cuda_check(cudaDeviceSynchronize(), "create sync");
        *out = holder.release();
    });
}

void lsb_destroy(lsb_context* ctx) { delete ctx; }

lsb_status lsb_get_info(const lsb_context* ctx, int* n, int* r, int* V, int* E, int* h, int* precision) {
    return run([&] {
        check_ctx(ctx);
        const Context& c = ctx->c;
        if (n) *n = c.n;
        if (r) *r = c.r;
        if (V) *V = c.mesh.V;
        if (E) *E = c.mesh.E;
        if (h) *h = c.h;
        if (precision) *precision = c.precision;
    });
}

lsb_status lsb_get_mass(const lsb_context* ctx, double* mass_diag, double* total_mass) {
    return run([&] {
        check_ctx(ctx);
        if (mass_diag) std::memcpy(mass_diag, ctx->c.mass.data(), ctx->c.mass.size() * 8);
        if (total_mass) *total_mass = ctx->c.total_mass;
    });
}

lsb_status lsb_set_pin_positions(lsb_context* ctx, const double* pin_positions) {
    return run([&] {
        check_ctx(ctx);
        require(pin_positions != nullptr, "pins: null array");
        Context& c = ctx->c;
        sync(c);
        c.pin_positions.assign(pin_positions, pin_positions + 3 * (size_t)c.mesh.V);
        ++c.pins_version;
        upload_pins(c);
    });
}

lsb_status lsb_set_inertia(lsb_context* ctx, const double* qbar, double dt) {
    return run([&] {
        check_ctx(ctx);
        Context& c = ctx->c;
        require(dt > 0.0, "solver: dt must be > 0");
        sync(c);
        get_state(c);
        DevState* h = c.h_state;
        h->dt = dt;
        h->inv_dt2 = 1.0 / (dt * dt);
        h->has_inertia = qbar ? 1 : 0;
        h->quasi_static = qbar ? 0 : 1;
        if (qbar) {
            std::vector<double> ut(c.n);
            for (int f = 0; f < c.mesh.n_free; ++f)
                for (int k = 0; k < 3; ++k)
                    ut[3 * f + k] = qbar[3 * f + k] - c.mesh.X[3 * (size_t)c.mesh.free_vertex[f] + k];
            c.copy(c.d_ut, ut.data(), ut.size() * 8, cudaMemcpyHostToDevice, "ut");
            if (!c.d_ut_user) c.d_ut_user = static_cast<double*>(c.dmalloc(sizeof(double) * c.n));
            c.copy(c.d_ut_user, ut.data(), ut.size() * 8, cudaMemcpyHostToDevice, "ut (user)");
            for (int i = 0; i < c.n; ++i) c.h_eprow[6 * (size_t)i + 5] = ut[i];
            c.copy(c.d_eprow, c.h_eprow.data(), c.h_eprow.size() * 8, cudaMemcpyHostToDevice, "eprow");
        }
        c.has_qbar = qbar != nullptr;
        c.dt = dt;
        c.copy(c.d_state, h, sizeof(DevState), cudaMemcpyHostToDevice, "state put");
    });
}

static void put_zt(Context& c, const double* z) {
    // staged through the pinned host mirror: a truly asynchronous DMA (pageable sources are
    // copied synchronously by the driver)
    if (z != c.h_state->zt) std::memcpy(c.h_state->zt, z, sizeof(double) * c.r);
    cuda_check(cudaMemcpyAsync(c.d_state->zt, c.h_state->zt, sizeof(double) * c.r, cudaMemcpyHostToDevice, c.stream),
               "z upload");
}

// The evaluation result only (configuration + current-evaluation block of DevState:
// f_eval, status, zt, gz; ~1 KB of the ~20 KB state).
static void get_eval_result(Context& c) {
    cuda_check(cudaMemcpyAsync(c.h_state, c.d_state, offsetof(DevState, phase), cudaMemcpyDeviceToHost, c.stream),
               "eval result");
    sync(c);
}

lsb_status lsb_eval(lsb_context* ctx, const double* z, double* value, double* grad) {
    return run([&] {
        check_ctx(ctx);
        require(z && value, "eval: null argument");
        Context& c = ctx->c;
        // direct path (persistent kernel): z travels with the launch and the kernel writes
        // {E, status, grad} into host-mapped memory -- no separate copies
        if (c.h_out && c.impl->eval_direct(c, z, grad != nullptr, c.d_out)) {
            sync(c);
            // keep the host mirror's evaluation block current (as get_eval_result does)
            std::memcpy(c.h_state->zt, z, sizeof(double) * c.r);
            c.h_state->f_eval = c.h_out[0];
            c.h_state->status = (int)c.h_out[1];
            if (grad) std::memcpy(c.h_state->gz, c.h_out + 2, sizeof(double) * c.r);
            if (c.h_state->status == kStNonFinite) throw LsbError(LSB_ENONFINITE, "reduced objective: non-finite energy");
            *value = c.h_out[0];
            if (grad) std::memcpy(grad, c.h_out + 2, sizeof(double) * c.r);
            return;
        }
        put_zt(c, z);
        c.impl->eval(c, grad != nullptr);
        get_eval_result(c);
        const DevState* s = c.h_state;
        if (s->status == kStNonFinite) throw LsbError(LSB_ENONFINITE, "reduced objective: non-finite energy");
        *value = s->f_eval;
        if (grad) std::memcpy(grad, s->gz, sizeof(double) * c.r);
    });
}

lsb_status lsb_decode(lsb_context* ctx, const double* z, double* q) {
    return run([&] {
        check_ctx(ctx);
        require(z && q, "decode: null argument");
        Context& c = ctx->c;
        put_zt(c, z);
        c.impl->eval(c, false);
        sync(c);
        const HostMesh& m = c.mesh;
        std::vector<double> U(4 * (size_t)m.V);
        c.copy(U.data(), c.d_U, U.size() * 8, cudaMemcpyDeviceToHost, "U");
        for (int f = 0; f < m.n_free; ++f)
            for (int k = 0; k < 3; ++k)
                q[3 * f + k] = m.X[3 * (size_t)m.free_vertex[f] + k] + U[4 * (size_t)m.free_vertex[f] + k];
    });
}

lsb_status lsb_lbfgs(lsb_context* ctx, double* z, const lsb_solver_config* cfg, lsb_exit_report* report) {
    return run([&] {
        check_ctx(ctx);
        require(z != nullptr, "lbfgs: null z");
        Context& c = ctx->c;
        put_config(c, cfg);
        put_zt(c, z);
        c.impl->minimize(c);
        get_state(c);
        const DevState* s = c.h_state;
        if (!(c.use_solve && c.impl->has_solve())) c.launches += (long long)c.body_kernels * s->loop_iters;
        if (s->status == kStNonFinite) throw LsbError(LSB_ENONFINITE, "reduced objective: non-finite energy");
        std::memcpy(z, s->x, sizeof(double) * c.r);
        fill_report(s, report);
    });
}

lsb_status lsb_set_state(lsb_context* ctx, const double* positions, const double* velocities, const double* z) {
    return run([&] {
        check_ctx(ctx);
        require(positions && velocities && z, "state: null argument");
        Context& c = ctx->c;
        sync(c);
        const HostMesh& m = c.mesh;
        std::vector<double> u(3 * (size_t)m.V);
        for (size_t i = 0; i < u.size(); ++i) u[i] = positions[i] - m.X[i];
        c.copy(c.d_u_state, u.data(), u.size() * 8, cudaMemcpyHostToDevice, "state u");
        c.copy(c.d_v_state, velocities, u.size() * 8, cudaMemcpyHostToDevice, "state v");
        c.copy(c.d_z_state, z, c.r * 8, cudaMemcpyHostToDevice, "state z");
        put_state(c, &DevState::t, 0.0);
        c.state_set = true;
    });
}

lsb_status lsb_get_state(lsb_context* ctx, double* positions, double* velocities, double* z, double* t) {
    return run([&] {
        check_ctx(ctx);
        Context& c = ctx->c;
        require(c.state_set, "state: lsb_set_state has not been called", LSB_ESTATE);
        sync(c);
        const HostMesh& m = c.mesh;
        if (positions) {
            c.copy(positions, c.d_u_state, 24 * (size_t)m.V, cudaMemcpyDeviceToHost, "state u");
            for (size_t i = 0; i < 3 * (size_t)m.V; ++i) positions[i] += m.X[i];
        }
        if (velocities) c.copy(velocities, c.d_v_state, 24 * (size_t)m.V, cudaMemcpyDeviceToHost, "state v");
        if (z) c.copy(z, c.d_z_state, 8 * (size_t)c.r, cudaMemcpyDeviceToHost, "state z");
        if (t) {
            get_state(c);
            *t = c.h_state->t;
        }
    });
}

lsb_status lsb_set_external_force(lsb_context* ctx, const double* force) {
    return run([&] {
        check_ctx(ctx);
        require(force != nullptr, "force: null array");
        Context& c = ctx->c;
        sync(c);
        std::vector<double> a(c.n);
        for (int i = 0; i < c.n; ++i) a[i] = force[i] / c.mass[i];  // f / m (reduced_solver.cpp:253)
        c.copy(c.d_a_ext, a.data(), a.size() * 8, cudaMemcpyHostToDevice, "force");
    });
}

static void prepare_steps(Context& c, int steps, const lsb_solver_config* cfg, int quasi_static) {
    require(c.state_set, "step: lsb_set_state has not been called", LSB_ESTATE);
    require(steps >= 0, "simulate: negative step count");
    put_config(c, cfg);
    get_state(c);
    c.h_state->quasi_static = quasi_static ? 1 : 0;
    c.h_state->step_idx = 0;
    c.copy(c.d_state, c.h_state, sizeof(DevState), cudaMemcpyHostToDevice, "state put");
    c.ensure_step_buffers(std::max(1, steps));
}

lsb_status lsb_step(lsb_context* ctx, const lsb_solver_config* cfg, int quasi_static, lsb_exit_report* report) {
    return run([&] {
        check_ctx(ctx);
        Context& c = ctx->c;
        prepare_steps(c, 1, cfg, quasi_static);
        c.impl->step(c);
        restore_user_objective(c);
        get_state(c);
        if (c.h_state->status == kStNonFinite) throw LsbError(LSB_ENONFINITE, "reduced objective: non-finite energy");
        if (report) c.copy(report, c.d_reports, sizeof(lsb_exit_report), cudaMemcpyDeviceToHost, "report");
    });
}

lsb_status lsb_simulate(lsb_context* ctx, int steps, const lsb_solver_config* cfg, int quasi_static,
                        lsb_exit_report* reports, double* z_traj) {
    return run([&] {
        check_ctx(ctx);
        Context& c = ctx->c;
        prepare_steps(c, steps, cfg, quasi_static);
        for (int s = 0; s < steps; ++s) c.impl->step(c);
        restore_user_objective(c);
        sync(c);
        get_state(c);
        if (reports) c.copy(reports, c.d_reports, sizeof(lsb_exit_report) * steps, cudaMemcpyDeviceToHost, "reports");
        if (z_traj) c.copy(z_traj, c.d_z_traj, sizeof(double) * (size_t)steps * c.r, cudaMemcpyDeviceToHost, "z traj");
        std::vector<lsb_exit_report> tmp(steps);
        c.copy(tmp.data(), c.d_reports, sizeof(lsb_exit_report) * steps, cudaMemcpyDeviceToHost, "reports");
        for (int s = 0; s < steps; ++s)
            if (tmp[s].code == -kStNonFinite) throw LsbError(LSB_ENONFINITE, "reduced objective: non-finite energy");
    });
}

lsb_status lsb_get_solve_info(const lsb_context* ctx, int* solve_grid, int* use_solve) {
    return run([&] {
        check_ctx(ctx);
        if (solve_grid) *solve_grid = ctx->c.impl->has_solve() ? ctx->c.solve_grid : 0;
        g_last_error = ctx->c.solve_reason;
        if (use_solve) *use_solve = (ctx->c.use_solve && ctx->c.impl->has_solve()) ? 1 : 0;
    });
}

lsb_status lsb_set_solve_kernel(lsb_context* ctx, int enable) {
    return run([&] {
        check_ctx(ctx);
        ctx->c.use_solve = enable != 0;
    });
}

lsb_status lsb_get_trace_raw(const lsb_context* ctx, unsigned long long* out) {
    return run([&] {
        check_ctx(ctx);
        require(ctx->c.d_trace != nullptr, "trace: LSB_TRACE=1 not set at create");
        ctx->c.copy(out, ctx->c.d_trace, 8 * 2048, cudaMemcpyDeviceToHost, "trace");
    });
}

lsb_status lsb_get_sweep_trace(const lsb_context* ctx, unsigned long long* out, int cap, int* count) {
    return run([&] {
        check_ctx(ctx);
        require(count != nullptr, "sweep trace: null count");
        *count = ctx->c.d_sweep_trace ? ctx->c.sweep_tickets : 0;
        if (!ctx->c.d_sweep_trace || !out) return;
        const size_t words = std::min<size_t>((size_t)cap, 4 * (size_t)ctx->c.sweep_tickets);
        ctx->c.copy(out, ctx->c.d_sweep_trace, 8 * words, cudaMemcpyDeviceToHost, "sweep trace");
    });
}

lsb_status lsb_get_trace(const lsb_context* ctx, unsigned long long* out, int cap, int* count) {
    return run([&] {
        check_ctx(ctx);
        *count = 0;
        if (!ctx->c.d_trace) return;
        std::vector<unsigned long long> t(512);
        ctx->c.copy(t.data(), ctx->c.d_trace, 8 * 512, cudaMemcpyDeviceToHost, "trace");
        const int n = (int)std::min<unsigned long long>(t[0], 255);
        for (int i = 0; i < n && 2 * i + 1 < cap; ++i) {
            out[2 * i] = t[1 + 2 * i];
            out[2 * i + 1] = t[2 + 2 * i];
        }
        *count = n;
    });
}

lsb_status lsb_get_dev_flags(const lsb_context* ctx, char* buf, int cap) {
    return run([&] {
        check_ctx(ctx);
        require(buf && cap > 0, "dev flags: null buffer");
        const std::string& a = ctx->c.dev.active;
        const size_t k = std::min(a.size(), (size_t)cap - 1);
        std::memcpy(buf, a.data(), k);
        buf[k] = 0;
    });
}

lsb_status lsb_get_launch_count(const lsb_context* ctx, long long* launches) {
    return run([&] {
        check_ctx(ctx);
        const Context& c = ctx->c;
        long long dev = 0;
        c.copy(&dev, c.d_launch_acc, sizeof(long long), cudaMemcpyDeviceToHost, "launch acc");
        *launches = c.launches + dev + c.batched_launches;
    });
}

lsb_status lsb_profile_eval(lsb_context* ctx, const double* z, int reps, double* ms_out_fwd, double* ms_elem,
                            double* ms_vjp, double* ms_total) {
    return run([&] {
        check_ctx(ctx);
        require(z && reps > 0, "profile: bad arguments");
        Context& c = ctx->c;
        put_zt(c, z);
        float ms[4];
        c.impl->profile(c, reps, ms);
        if (ms_out_fwd) *ms_out_fwd = ms[0];
        if (ms_elem) *ms_elem = ms[1];
        if (ms_vjp) *ms_vjp = ms[2];
        if (ms_total) *ms_total = ms[3];
    });
}

lsb_status lsb_bench_evals(lsb_context* ctx, int K, const double* Z, size_t flush_bytes, double* eval_ms,
                           double* out_fwd_ms, double* E) {
    return lsb_bench_evals_ex(ctx, K, Z, flush_bytes, 1, eval_ms, out_fwd_ms, E);
}

lsb_status lsb_bench_evals_ex(lsb_context* ctx, int K, const double* Z, size_t flush_bytes, int want_grad,
                              double* eval_ms, double* out_fwd_ms, double* E) {
    return run([&] {
        check_ctx(ctx);
        require(K >= 1 && Z && eval_ms && out_fwd_ms, "bench: bad arguments");
        bench_evals(ctx->c, K, Z, flush_bytes, eval_ms, out_fwd_ms, E, want_grad != 0);
    });
}

lsb_status lsb_bench_batched(lsb_context* ctx, int kind, int B, const double* Z1, const double* Z2, int reps,
                             size_t flush_bytes, double* ms, double* E, double* G, double* loss) {
    return run([&] {
        check_ctx(ctx);
        require(reps >= 1 && B >= 1 && Z1 && ms, "bench batched: bad arguments");
        Context& c = ctx->c;
        if (kind == 0) {
            require(E != nullptr, "bench batched: E required");
            bench_call(c, reps, flush_bytes, ms, [&] { batched_eval(c, B, Z1, E, G); });
        } else if (kind == 1) {
            require(Z2 && loss, "bench batched: Z2 and loss required");
            for (int p = 0; p < B; ++p) {  // losses.cpp:202-204
                double dz2 = 0.0;
                for (int k = 0; k < c.r; ++k)
                    dz2 += (Z1[p * c.r + k] - Z2[p * c.r + k]) * (Z1[p * c.r + k] - Z2[p * c.r + k]);
                require(dz2 > 0.0, "lipschitz loss: coincident pair");
            }
            bench_call(c, reps, flush_bytes, ms, [&] { *loss = lipschitz_loss(c, B, Z1, Z2); });
        } else {
            throw LsbError(LSB_EINVAL, "bench batched: kind must be 0 (eval_batched) or 1 (lipschitz loss)");
        }
    });
}

lsb_status lsb_bench_e2e(lsb_context* ctx, int K, const double* Z, double* E, double* G, double* seconds) {
    return run([&] {
        check_ctx(ctx);
        require(K >= 1 && Z && E && G && seconds, "bench e2e: bad arguments");
        const int r = ctx->c.r;
        const auto t0 = std::chrono::steady_clock::now();
        for (int k = 0; k < K; ++k) {
            const lsb_status st = lsb_eval(ctx, Z + (size_t)k * r, E + k, G + (size_t)k * r);
            if (st != LSB_OK) throw LsbError(st, "bench e2e: lsb_eval failed");
        }
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

lsb_status lsb_bench_steps(lsb_context* ctx, int K, const lsb_solver_config* cfg, int quasi_static,
                           size_t flush_bytes, double* step_ms, lsb_exit_report* reports) {
    return run([&] {
        check_ctx(ctx);
        require(K >= 1 && step_ms, "bench: bad arguments");
        Context& c = ctx->c;
        prepare_steps(c, K, cfg, quasi_static);
        bench_steps(c, K, flush_bytes, step_ms, reports);
        restore_user_objective(c);
        get_state(c);
    });
}

lsb_status lsb_assemble(lsb_context* ctx, const double* q, double* value, double* grad) {
    return run([&] {
        check_ctx(ctx);
        require(q && value, "assemble: null argument");
        refops_assemble(ctx->c, q, value, grad);
    });
}

lsb_status lsb_element_snh(lsb_context* ctx, int count, const int* ids, const double* positions, double* energy,
                           double* grad, double* hess) {
    return run([&] {
        check_ctx(ctx);
        require(count >= 0 && (count == 0 || (ids && positions && energy && grad)), "element_snh: bad arguments");
        if (count == 0) return;
        for (int k = 0; k < count; ++k)
            require(ids[k] >= 0 && ids[k] < ctx->c.mesh.E, "element_snh: element id out of range");
        refops_element_snh(ctx->c, count, ids, positions, energy, grad, hess);
    });
}

lsb_status lsb_elastic_hessian_apply(lsb_context* ctx, const double* q, int k, const double* in, double* out) {
    return run([&] {
        check_ctx(ctx);
        require(k >= 0 && q && (k == 0 || (in && out)), "elastic_hessian_apply: bad arguments");
        if (k == 0) return;
        refops_elastic_hessian_apply(ctx->c, q, k, in, out);
    });
}

lsb_status lsb_decode_jacobian(lsb_context* ctx, const double* z, double* J) {
    return run([&] {
        check_ctx(ctx);
        require(z && J, "decode_jacobian: null argument");
        refops_decode_jacobian(ctx->c, z, J);
    });
}

lsb_status lsb_decode_second_directional(lsb_context* ctx, const double* z, const double* u, const double* v,
                                         double* out) {
    return run([&] {
        check_ctx(ctx);
        require(z && u && v && out, "decode_second_directional: null argument");
        refops_decode_second_directional(ctx->c, z, u, v, out);
    });
}

lsb_status lsb_eval_batched(lsb_context* ctx, int B, const double* Z, double* E, double* G) {
    return run([&] {
        check_ctx(ctx);
        require(B >= 0 && (B == 0 || (Z && E)), "eval_batched: bad arguments");
        if (B == 0) return;
        batched_eval(ctx->c, B, Z, E, G);
    });
}

lsb_status lsb_hessian_batched(lsb_context* ctx, int B, const double* Z, double* H) {
    return run([&] {
        check_ctx(ctx);
        require(B >= 0 && (B == 0 || (Z && H)), "hessian_batched: bad arguments");
        if (B == 0) return;
        batched_hessian(ctx->c, B, Z, H);
    });
}

// Runtime cubature (SolverConfig::runtime_cubature / ReducedObjective::runtime_cubature,
// reduced_solver.hpp:23,67; assemble over an ElementSubset, energy.cpp:418-432): the elastic
// term sums w_k E_{ids[k]}.  Linear in the element volume, so the active element set is the
// subset with vol * w; count == 0 (or ids NULL) restores the full set.
lsb_status lsb_set_cubature(lsb_context* ctx, int count, const int* ids, const double* weights) {
    return run([&] {
        check_ctx(ctx);
        Context& c = ctx->c;
        if (!c.has_full) {
            c.mesh_full = c.mesh;
            c.mu_full = c.mu;
            c.lambda_full = c.lambda;
            c.has_full = true;
        }
        const HostMesh& F = c.mesh_full;
        HostMesh m = F;
        std::vector<double> mu = c.mu_full, lam = c.lambda_full;
        if (count > 0 && ids) {
            require(weights != nullptr, "cubature: weights required with ids");
            m.E = count;
            m.T.assign(4 * (size_t)count, 0);
            m.Dminv.assign(9 * (size_t)count, 0.0);
            m.vol.assign(count, 0.0);
            mu.assign(count, 0.0);
            lam.assign(count, 0.0);
            for (int k = 0; k < count; ++k) {
                const int e = ids[k];
                require(e >= 0 && e < F.E, "cubature: element id out of range");
                require(std::isfinite(weights[k]), "cubature: non-finite weight");
                std::copy(&F.T[4 * (size_t)e], &F.T[4 * (size_t)e] + 4, &m.T[4 * (size_t)k]);
                std::copy(&F.Dminv[9 * (size_t)e], &F.Dminv[9 * (size_t)e] + 9, &m.Dminv[9 * (size_t)k]);
                m.vol[k] = F.vol[e] * weights[k];
                mu[k] = c.mu_full[e];
                lam[k] = c.lambda_full[e];
            }
            // vertex (free slot) -> incident (element k * 4 + corner), ascending k
            std::vector<int> cnt(m.n_free + 1, 0);
            for (int k = 0; k < count; ++k)
                for (int s = 0; s < 4; ++s) {
                    const int f = m.free_index[m.T[4 * (size_t)k + s]];
                    if (f >= 0) cnt[f + 1]++;
                }
            m.csr_ptr.assign(m.n_free + 1, 0);
            for (int f = 0; f < m.n_free; ++f) m.csr_ptr[f + 1] = m.csr_ptr[f] + cnt[f + 1];
            m.csr_ent.assign(m.csr_ptr[m.n_free], 0);
            std::vector<int> fill(m.csr_ptr.begin(), m.csr_ptr.end() - 1);
            for (int k = 0; k < count; ++k)
                for (int s = 0; s < 4; ++s) {
                    const int f = m.free_index[m.T[4 * (size_t)k + s]];
                    if (f >= 0) m.csr_ent[fill[f]++] = 4 * k + s;
                }
        }
        sync(c);
        c.mesh = std::move(m);
        c.mu = std::move(mu);
        c.lambda = std::move(lam);
        upload_elements(c);
        c.impl->rebind_elements(c);
        c.batched.reset();  // rebuilt lazily over the new element set
    });
}

lsb_status lsb_objective_hessian(lsb_context* ctx, int B, const double* Z, double* H) {
    return run([&] {
        check_ctx(ctx);
        require(B >= 0 && (B == 0 || (Z && H)), "objective_hessian: bad arguments");
        if (B == 0) return;
        batched_objective_hessian(ctx->c, B, Z, H);
    });
}

// projective_newton_minimize(objective, hessian, z, cfg) (reduced_solver.cpp:133-182) on this
// context's objective: device E / grad E and device objective Hessians, host d x d algebra.
lsb_status lsb_projective_newton(lsb_context* ctx, double* z, const lsb_solver_config* cfg, lsb_exit_report* report) {
    return run([&] {
        check_ctx(ctx);
        require(z != nullptr && cfg != nullptr, "projective newton: null argument");
        require(cfg->epsilon > 0 && cfg->max_iters > 0 && cfg->max_linesearch > 0, "solver config: invalid");
        Context& c = ctx->c;
        const auto t0 = std::chrono::steady_clock::now();
        const int r = c.r;
        int value_evals = 0, grad_evals = 0;
        auto objective = [&](const std::vector<double>& x, std::vector<double>* g) {
            put_zt(c, x.data());
            c.impl->eval(c, g != nullptr);
            get_eval_result(c);
            const DevState* s = c.h_state;
            if (s->status == kStNonFinite) throw LsbError(LSB_ENONFINITE, "reduced objective: non-finite energy");
            if (g) {
                g->assign(s->gz, s->gz + r);
                ++grad_evals;
            } else {
                ++value_evals;
            }
            return s->f_eval;
        };
        auto inf_norm = [](const std::vector<double>& v) {
            double m = 0.0;
            for (double x : v) m = std::max(m, std::fabs(x));
            return m;
        };
        std::vector<double> x(z, z + r), g(r), H((size_t)r * r);
        double f = objective(x, &g);
        lsb_exit_report rep{};
        rep.code = 4;
        bool done = false;
        for (int iter = 0; iter < cfg->max_iters && !done; ++iter) {
            rep.iterations = iter;
            rep.final_grad_inf_norm = inf_norm(g);
            if (rep.final_grad_inf_norm < cfg->epsilon) {
                rep.code = 1;
                done = true;
                break;
            }
            batched_objective_hessian(c, 1, x.data(), H.data());
            const std::vector<double> Hp = newton::project_spd(H, r);
            std::vector<double> mg(r), d;
            for (int k = 0; k < r; ++k) mg[k] = -g[k];
            if (!newton::ldlt_solve(Hp, r, mg, d)) throw LsbError(LSB_ENONFINITE, "projective newton: factorization failed");
            for (double v : d)
                if (!std::isfinite(v)) throw LsbError(LSB_ENONFINITE, "projective newton: singular system");
            double gtd = 0.0;
            for (int k = 0; k < r; ++k) gtd += g[k] * d[k];
            if (!(gtd < 0.0)) {
                rep.code = 2;
                done = true;
                break;
            }
            std::vector<double> trial(r);
            bool ok = false;
            double a = 1.0;
            for (int ls = 0; ls < cfg->max_linesearch; ++ls) {  // armijo (reduced_solver.cpp:43-54)
                for (int k = 0; k < r; ++k) trial[k] = x[k] + a * d[k];
                const double ft = objective(trial, nullptr);
                if (std::isfinite(ft) && ft <= f + 1e-4 * a * gtd) {
                    ok = true;
                    break;
                }
                a *= 0.5;
            }
            if (!ok) {
                rep.code = 3;
                done = true;
                break;
            }
            x = trial;
            f = objective(x, &g);
        }
        if (!done) {
            rep.iterations = cfg->max_iters;
            rep.final_grad_inf_norm = inf_norm(g);
            rep.code = rep.final_grad_inf_norm < cfg->epsilon ? 1 : 4;
        }
        std::memcpy(z, x.data(), sizeof(double) * r);
        rep.wall_time_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        rep.value_evals = value_evals;
        rep.grad_evals = grad_evals;
        if (report) *report = rep;
    });
}

lsb_status lsb_lipschitz_loss(lsb_context* ctx, int P, const double* Z1, const double* Z2, double* loss) {
    return run([&] {
        check_ctx(ctx);
        require(P > 0, "lipschitz loss: no pairs");  // losses.cpp:199
        require(Z1 && Z2 && loss, "lipschitz loss: null argument");
        const int r = ctx->c.r;
        for (int p = 0; p < P; ++p) {  // losses.cpp:202-204
            double dz2 = 0.0;
            for (int k = 0; k < r; ++k) dz2 += (Z1[p * r + k] - Z2[p * r + k]) * (Z1[p * r + k] - Z2[p * r + k]);
            require(dz2 > 0.0, "lipschitz loss: coincident pair");
        }
        *loss = lipschitz_loss(ctx->c, P, Z1, Z2);
    });
}

lsb_status lsb_lipschitz_loss_grad(lsb_context* ctx, int P, const double* Z1, const double* Z2, double* loss,
                                   double* grad) {
    return run([&] {
        check_ctx(ctx);
        require(P > 0, "lipschitz loss: no pairs");  // losses.cpp:199
        require(Z1 && Z2 && loss && grad, "lipschitz loss: null argument");
        const int r = ctx->c.r;
        for (int p = 0; p < P; ++p) {  // losses.cpp:202-204
            double dz2 = 0.0;
            for (int k = 0; k < r; ++k) dz2 += (Z1[p * r + k] - Z2[p * r + k]) * (Z1[p * r + k] - Z2[p * r + k]);
            require(dz2 > 0.0, "lipschitz loss: coincident pair");
        }
        *loss = lipschitz_loss_grad(ctx->c, P, Z1, Z2, grad);
    });
}

}  // extern "C"
