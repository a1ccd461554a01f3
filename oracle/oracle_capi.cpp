// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.  ctypes-facing C API of the
// CPU oracle (oracle.hpp).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load this library.
#include <chrono>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <algorithm>
#include <string>
#include <thread>

#include "oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e) {
    g_err = e.what();
    return -1;
}
struct Ctx {  // one problem instance: mesh + material + decoder + mass
    Mesh mesh;
    Material mat;
    Model model;
    std::vector<double> mass;
    double total_mass = 0.0;
    std::vector<double> pins;  // V*3 pin positions (rest)
    bool has_cub = false;      // runtime cubature (ElementSubset) for the objective calls
    std::vector<int> cub_ids;
    std::vector<double> cub_w;
};
// ReducedObjective over the context (+ its runtime cubature when set)
void bind_objective(ReducedObjective& obj, Ctx* c) {
    obj.model = &c->model;
    obj.mesh = &c->mesh;
    obj.mat = &c->mat;
    obj.pin_positions = c->pins;
    obj.mass = c->mass;
    if (c->has_cub) {
        obj.cub_ids = &c->cub_ids;
        obj.cub_w = &c->cub_w;
    }
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

double orc_randu_seq(std::uint64_t seed, std::uint64_t tag, int count, double* out) {
    Rng r = substream(seed, tag);
    for (int i = 0; i < count; ++i) out[i] = randu(r);
    return 0.0;
}
void orc_randn_seq(std::uint64_t seed, std::uint64_t tag, int count, double* out) {
    Rng r = substream(seed, tag);
    for (int i = 0; i < count; ++i) out[i] = randn(r);
}
double orc_activation_eval(int act, double x, int order) {
    try {
        return activation_eval(act, x, order);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 0.0 / 0.0;
    }
}

// ---- problem context ---------------------------------------------------------
// mesh_kind: 0 = explicit (V, X, E, T, pins), 1 = Kuhn bar (grid args).
void* orc_ctx_bar(int nx, int ny, int nz, double w, double h, double d, double jitter_frac,
                  std::uint64_t mesh_seed, int pin_left) {
    try {
        auto* c = new Ctx;
        c->mesh = make_bar_kuhn(nx, ny, nz, w, h, d, jitter_frac, mesh_seed, pin_left != 0);
        c->pins = c->mesh.X;
        return c;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void* orc_ctx_mesh(int V, const double* X, int E, const int* T, int npins, const int* pins) {
    try {
        auto* c = new Ctx;
        c->mesh = build_mesh(V, X, E, T, std::vector<int>(pins, pins + npins));
        c->pins = c->mesh.X;
        return c;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void orc_ctx_free(void* p) { delete static_cast<Ctx*>(p); }

void orc_ctx_info(void* p, int* V, int* E, int* n_free, int* npinned) {
    auto* c = static_cast<Ctx*>(p);
    *V = c->mesh.V;
    *E = c->mesh.E;
    *n_free = c->mesh.n_free;
    *npinned = static_cast<int>(c->mesh.pinned.size());
}
void orc_ctx_mesh_arrays(void* p, double* X, int* T, double* Dminv, double* vol, int* free_index) {
    auto* c = static_cast<Ctx*>(p);
    const Mesh& m = c->mesh;
    if (X) std::memcpy(X, m.X.data(), m.X.size() * 8);
    if (T) std::memcpy(T, m.T.data(), m.T.size() * 4);
    if (Dminv) std::memcpy(Dminv, m.Dminv.data(), m.Dminv.size() * 8);
    if (vol) std::memcpy(vol, m.vol.data(), m.vol.size() * 8);
    if (free_index) std::memcpy(free_index, m.free_index.data(), m.free_index.size() * 4);
}

// Material: mu/lambda arrays of length E; density.
int orc_ctx_set_material(void* p, const double* mu, const double* lambda, double density) {
    try {
        auto* c = static_cast<Ctx*>(p);
        if (!(density > 0.0)) throw std::invalid_argument("material: density must be > 0");
        for (int e = 0; e < c->mesh.E; ++e) {
            if (!(mu[e] > 0.0)) throw std::invalid_argument("material: mu must be > 0");
            if (!(lambda[e] >= 0.0)) throw std::invalid_argument("material: lambda must be >= 0");
        }
        c->mat.mu.assign(mu, mu + c->mesh.E);
        c->mat.lambda.assign(lambda, lambda + c->mesh.E);
        c->mat.density = density;
        c->mass = lump_mass(c->mesh, density, &c->total_mass);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
void orc_ctx_mass(void* p, double* diag, double* total) {
    auto* c = static_cast<Ctx*>(p);
    std::memcpy(diag, c->mass.data(), c->mass.size() * 8);
    *total = c->total_mass;
}
void orc_ctx_set_pins(void* p, const double* pin_positions) {
    auto* c = static_cast<Ctx*>(p);
    c->pins.assign(pin_positions, pin_positions + 3 * static_cast<size_t>(c->mesh.V));
}

// Decoder: explicit layers (row-major W), or Xavier bar decoder.
int orc_ctx_set_decoder(void* p, int r, int L, const int* rows, const int* cols, const double* const* W,
                        const double* const* b, const int* acts, const double* shift, const double* scale) {
    try {
        auto* c = static_cast<Ctx*>(p);
        Model m;
        m.r = r;
        m.n = rows[L - 1];
        int width = r;
        for (int l = 0; l < L; ++l) {
            if (cols[l] != width) throw std::invalid_argument("model: decoder layer shapes do not chain");
            Layer ly;
            ly.rows = rows[l];
            ly.cols = cols[l];
            ly.W.assign(W[l], W[l] + static_cast<size_t>(rows[l]) * cols[l]);
            ly.b.assign(b[l], b[l] + rows[l]);
            ly.act = acts[l];
            m.dec.push_back(std::move(ly));
            width = rows[l];
        }
        if (m.n != c->mesh.num_dofs()) throw std::invalid_argument("model: decoder output width != n");
        m.shift.assign(shift, shift + m.n);
        m.scale.assign(scale, scale + m.n);
        c->model = std::move(m);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
int orc_ctx_bar_decoder(void* p, int r, int hidden_layers, int width, int act, std::uint64_t seed,
                        double out_scale) {
    try {
        auto* c = static_cast<Ctx*>(p);
        c->model = make_bar_decoder(c->mesh, r, hidden_layers, width, act, seed, out_scale);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
// Copy decoder layer l out (W row-major, b), plus shift/scale when l < 0.
void orc_ctx_decoder_layer(void* p, int l, int* rows, int* cols, int* act, double* W, double* b) {
    auto* c = static_cast<Ctx*>(p);
    const Layer& ly = c->model.dec[l];
    *rows = ly.rows;
    *cols = ly.cols;
    *act = ly.act;
    if (W) std::memcpy(W, ly.W.data(), ly.W.size() * 8);
    if (b) std::memcpy(b, ly.b.data(), ly.b.size() * 8);
}
int orc_ctx_decoder_layers(void* p) { return static_cast<int>(static_cast<Ctx*>(p)->model.dec.size()); }
void orc_ctx_decoder_norm(void* p, double* shift, double* scale) {
    auto* c = static_cast<Ctx*>(p);
    std::memcpy(shift, c->model.shift.data(), c->model.shift.size() * 8);
    std::memcpy(scale, c->model.scale.data(), c->model.scale.size() * 8);
}

// ---- element / assembly ----------------------------------------------------------
int orc_element_snh(void* p, int e, double mu, double lambda, const double* positions, int want_hess,
                    double* energy, double* grad, double* hess) {
    try {
        auto* c = static_cast<Ctx*>(p);
        ElementDerivatives ed;
        element_snh(c->mesh, mu, lambda, e, positions, want_hess != 0, ed);
        *energy = ed.energy;
        if (grad) std::memcpy(grad, ed.grad, sizeof(ed.grad));
        if (hess && want_hess) std::memcpy(hess, ed.hess, sizeof(ed.hess));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
// subset: nsub < 0 means the full unit-weight set.
int orc_assemble(void* p, const double* q, int nsub, const int* ids, const double* w, double* value,
                 double* grad) {
    try {
        auto* c = static_cast<Ctx*>(p);
        std::vector<double> qq(q, q + c->mesh.num_dofs());
        std::vector<int> sid;
        std::vector<double> sw;
        if (nsub >= 0) {
            sid.assign(ids, ids + nsub);
            sw.assign(w, w + nsub);
        }
        const Assembled a = assemble(c->mesh, c->mat, qq, c->pins, nsub >= 0 ? &sid : nullptr,
                                     nsub >= 0 ? &sw : nullptr);
        *value = a.value;
        if (grad) std::memcpy(grad, a.gradient.data(), a.gradient.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
int orc_elastic_hessian_apply(void* p, const double* q, int k, const double* in, double* out) {
    try {
        auto* c = static_cast<Ctx*>(p);
        const int n = c->mesh.num_dofs();
        std::vector<double> qq(q, q + n), vin(in, in + static_cast<size_t>(n) * k), vout(static_cast<size_t>(n) * k, 0.0);
        elastic_hessian_apply(c->mesh, c->mat, dof_unpack(c->mesh, qq, c->pins), vin, k, vout);
        std::memcpy(out, vout.data(), vout.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- decoder -------------------------------------------------------------------------
int orc_decode(void* p, const double* z, double* q) {
    try {
        auto* c = static_cast<Ctx*>(p);
        const auto out = decode(c->model, std::vector<double>(z, z + c->model.r));
        std::memcpy(q, out.data(), out.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
int orc_decode_jacobian(void* p, const double* z, double* J) {
    try {
        auto* c = static_cast<Ctx*>(p);
        const auto out = decode_jacobian(c->model, std::vector<double>(z, z + c->model.r));
        std::memcpy(J, out.data(), out.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
int orc_decode_second_directional(void* p, const double* z, const double* u, const double* v, double* out) {
    try {
        auto* c = static_cast<Ctx*>(p);
        const int r = c->model.r;
        const auto o = decode_second_directional(c->model, std::vector<double>(z, z + r),
                                                 std::vector<double>(u, u + r), std::vector<double>(v, v + r));
        std::memcpy(out, o.data(), o.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- reduced objective -------------------------------------------------------------------
// qbar may be NULL (quasi-static: no inertia term).
int orc_objective_eval(void* p, const double* qbar, double dt, const double* z, double* value, double* grad) {
    try {
        auto* c = static_cast<Ctx*>(p);
        ReducedObjective obj;
        bind_objective(obj, c);
        obj.dt = dt;
        if (qbar) {
            obj.has_qbar = true;
            obj.qbar.assign(qbar, qbar + c->model.n);
        }
        std::vector<double> g;
        *value = obj.eval(std::vector<double>(z, z + c->model.r), grad ? &g : nullptr);
        if (grad) std::memcpy(grad, g.data(), g.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
int orc_objective_hessian(void* p, const double* qbar, double dt, const double* z, double* H) {
    try {
        auto* c = static_cast<Ctx*>(p);
        ReducedObjective obj;
        bind_objective(obj, c);
        obj.dt = dt;
        if (qbar) {
            obj.has_qbar = true;
            obj.qbar.assign(qbar, qbar + c->model.n);
        }
        const auto h = obj.hessian(std::vector<double>(z, z + c->model.r));
        std::memcpy(H, h.data(), h.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
// Batched objective (config 4 oracle): B independent evals, nthreads host threads.
int orc_objective_eval_batch(void* p, const double* qbar, double dt, int B, const double* Z, double* E,
                             double* G, int nthreads) {
    try {
        auto* c = static_cast<Ctx*>(p);
        const int r = c->model.r;
        ReducedObjective obj;
        bind_objective(obj, c);
        obj.dt = dt;
        if (qbar) {
            obj.has_qbar = true;
            obj.qbar.assign(qbar, qbar + c->model.n);
        }
        std::string err;
        auto work = [&](int b0, int b1) {
            try {
                for (int b = b0; b < b1; ++b) {
                    std::vector<double> g;
                    E[b] = obj.eval(std::vector<double>(Z + b * r, Z + (b + 1) * r), G ? &g : nullptr);
                    if (G) std::memcpy(G + static_cast<size_t>(b) * r, g.data(), r * 8);
                }
            } catch (const std::exception& e) {
                err = e.what();
            }
        };
        nthreads = std::max(1, std::min(nthreads, B));
        std::vector<std::thread> th;
        for (int k = 0; k < nthreads; ++k) th.emplace_back(work, (B * k) / nthreads, (B * (k + 1)) / nthreads);
        for (auto& t : th) t.join();
        if (!err.empty()) throw std::runtime_error(err);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- L-BFGS on a ctypes callback (reduced_solver tests) ------------------------------------
typedef double (*orc_objective_cb)(const double* x, double* g /*nullable*/, int n, void* user);
int orc_lbfgs_minimize(orc_objective_cb cb, void* user, int n, double* x, double epsilon, int max_iters,
                       int max_ls, int history, int* code, int* iterations, double* gnorm) {
    try {
        SolverConfig cfg;
        cfg.epsilon = epsilon;
        cfg.max_iters = max_iters;
        cfg.max_linesearch = max_ls;
        cfg.lbfgs_history = history;
        std::vector<double> xx(x, x + n);
        const ExitReport r = lbfgs_minimize(
            [&](const std::vector<double>& v, std::vector<double>* g) {
                if (g) g->resize(n);
                return cb(v.data(), g ? g->data() : nullptr, n, user);
            },
            xx, cfg);
        std::memcpy(x, xx.data(), n * 8);
        *code = r.code;
        *iterations = r.iterations;
        *gnorm = r.final_grad_inf_norm;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}


// Runtime cubature for the objective calls of this context (count 0 = full set).
int orc_set_cubature(void* p, int count, const int* ids, const double* w) {
    try {
        auto* c = static_cast<Ctx*>(p);
        c->has_cub = count > 0 && ids;
        c->cub_ids.assign(ids, ids + (c->has_cub ? count : 0));
        c->cub_w.assign(w, w + (c->has_cub ? count : 0));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- project_spd / projective Newton (energy.cpp:370-380, reduced_solver.cpp:133-182) ----------
int orc_project_spd(const double* H, int n, double* out) {
    try {
        const auto P = project_spd(std::vector<double>(H, H + (size_t)n * n), n);
        std::memcpy(out, P.data(), P.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
typedef void (*orc_hessian_cb)(const double* x, double* H, int n, void* user);
int orc_projective_newton(orc_objective_cb cb, orc_hessian_cb hcb, void* user, int n, double* x, double epsilon,
                          int max_iters, int max_ls, int* code, int* iterations, double* gnorm) {
    try {
        SolverConfig cfg;
        cfg.epsilon = epsilon;
        cfg.max_iters = max_iters;
        cfg.max_linesearch = max_ls;
        std::vector<double> xx(x, x + n);
        const ExitReport r = projective_newton_minimize(
            [&](const std::vector<double>& v, std::vector<double>* g) {
                if (g) g->resize(n);
                return cb(v.data(), g ? g->data() : nullptr, n, user);
            },
            [&](const std::vector<double>& v) {
                std::vector<double> H((size_t)n * n);
                hcb(v.data(), H.data(), n, user);
                return H;
            },
            xx, cfg);
        std::memcpy(x, xx.data(), n * 8);
        *code = r.code;
        *iterations = r.iterations;
        *gnorm = r.final_grad_inf_norm;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
// Projective Newton on the problem's reduced objective (qbar nullable = quasi-static).
int orc_objective_projective_newton(void* p, const double* qbar, double dt, double* z, double epsilon,
                                    int max_iters, int max_ls, int* code, int* iterations, double* gnorm,
                                    int* evals, int* value_evals) {
    try {
        auto* c = static_cast<Ctx*>(p);
        ReducedObjective obj;
        bind_objective(obj, c);
        obj.dt = dt;
        if (qbar) {
            obj.has_qbar = true;
            obj.qbar.assign(qbar, qbar + c->model.n);
        }
        SolverConfig cfg;
        cfg.epsilon = epsilon;
        cfg.max_iters = max_iters;
        cfg.max_linesearch = max_ls;
        const int r = c->model.r;
        std::vector<double> zz(z, z + r);
        const ExitReport rep = projective_newton_minimize(
            [&](const std::vector<double>& v, std::vector<double>* g) { return obj.eval(v, g); },
            [&](const std::vector<double>& v) { return obj.hessian(v); }, zz, cfg);
        std::memcpy(z, zz.data(), r * 8);
        *code = rep.code;
        *iterations = rep.iterations;
        *gnorm = rep.final_grad_inf_norm;
        if (evals) *evals = rep.evals;
        if (value_evals) *value_evals = rep.value_evals;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- dynamics ---------------------------------------------------------------------------------
// Runs `steps` implicit-Euler reduced steps from (positions, velocities, z),
// gravity force f = m g, static pins at rest.  State arrays are in/out.
// Per-step outputs (may be NULL): codes[steps], iters[steps], gnorm[steps],
// wall_ms[steps], evals[steps] (gradient evals), value_evals[steps], z_traj[steps*r].
int orc_simulate(void* p, const double* gravity, double epsilon, int max_iters, int max_ls, int history,
                 double dt, int quasi_static, int steps, double* positions, double* velocities, double* z,
                 int* codes, int* iters, double* gnorm, double* wall_ms, int* evals, int* value_evals,
                 double* z_traj) {
    try {
        auto* c = static_cast<Ctx*>(p);
        SolverConfig cfg;
        cfg.epsilon = epsilon;
        cfg.max_iters = max_iters;
        cfg.max_linesearch = max_ls;
        cfg.lbfgs_history = history;
        cfg.dt = dt;
        const int V = c->mesh.V, r = c->model.r;
        SimState st;
        st.positions.assign(positions, positions + 3 * V);
        st.velocities.assign(velocities, velocities + 3 * V);
        st.z.assign(z, z + r);
        const std::vector<double> f = gravity_force(c->mesh, c->mass, gravity);
        for (int s = 0; s < steps; ++s) {
            const ExitReport rep = reduced_step(st, c->pins, f, c->model, c->mesh, c->mat, c->mass, cfg,
                                                quasi_static != 0, c->has_cub ? &c->cub_ids : nullptr,
                                                c->has_cub ? &c->cub_w : nullptr);
            if (codes) codes[s] = rep.code;
            if (iters) iters[s] = rep.iterations;
            if (gnorm) gnorm[s] = rep.final_grad_inf_norm;
            if (wall_ms) wall_ms[s] = rep.wall_time_ms;
            if (evals) evals[s] = rep.evals;
            if (value_evals) value_evals[s] = rep.value_evals;
            if (z_traj) std::memcpy(z_traj + static_cast<size_t>(s) * r, st.z.data(), r * 8);
        }
        std::memcpy(positions, st.positions.data(), 3 * V * 8);
        std::memcpy(velocities, st.velocities.data(), 3 * V * 8);
        std::memcpy(z, st.z.data(), r * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// One reduced_step (reduced_solver.cpp:235-277) with an explicit frame: pin positions (V x 3)
// and the external force on the free DOFs (frame_at, scenario.cpp:187-205).
int orc_reduced_step(void* p, const double* pin_positions, const double* force, double epsilon, int max_iters,
                     int max_ls, int history, double dt, int quasi_static, double* positions, double* velocities,
                     double* z, int* code, int* iters) {
    try {
        auto* c = static_cast<Ctx*>(p);
        SolverConfig cfg;
        cfg.epsilon = epsilon;
        cfg.max_iters = max_iters;
        cfg.max_linesearch = max_ls;
        cfg.lbfgs_history = history;
        cfg.dt = dt;
        const int V = c->mesh.V, r = c->model.r, n = c->mesh.num_dofs();
        SimState st;
        st.positions.assign(positions, positions + 3 * V);
        st.velocities.assign(velocities, velocities + 3 * V);
        st.z.assign(z, z + r);
        const std::vector<double> pins(pin_positions, pin_positions + 3 * V), f(force, force + n);
        const ExitReport rep = reduced_step(st, pins, f, c->model, c->mesh, c->mat, c->mass, cfg, quasi_static != 0,
                                            c->has_cub ? &c->cub_ids : nullptr, c->has_cub ? &c->cub_w : nullptr);
        *code = rep.code;
        *iters = rep.iterations;
        std::memcpy(positions, st.positions.data(), 3 * V * 8);
        std::memcpy(velocities, st.velocities.data(), 3 * V * 8);
        std::memcpy(z, st.z.data(), r * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- losses -------------------------------------------------------------------------------------
int orc_reduced_potential_hessian(void* p, const double* z, double* H) {
    try {
        auto* c = static_cast<Ctx*>(p);
        const auto h = reduced_potential_hessian(c->model, c->mesh, c->mat, c->pins,
                                                 std::vector<double>(z, z + c->model.r));
        std::memcpy(H, h.data(), h.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
int orc_lipschitz_loss2(void* p, int P, const double* Z1, const double* Z2, int nthreads, double* loss) {
    try {
        auto* c = static_cast<Ctx*>(p);
        *loss = lipschitz_loss2(c->model, c->mesh, c->mat, c->pins, P, Z1, Z2, nthreads);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
int orc_elastic_third_contraction(void* p, const double* q, int k, const double* A, const double* B, double* qbar) {
    try {
        auto* c = static_cast<Ctx*>(p);
        const int n = c->mesh.num_dofs();
        std::vector<double> qq(q, q + n), va(A, A + static_cast<size_t>(n) * k), vb(B, B + static_cast<size_t>(n) * k),
            out(n, 0.0);
        elastic_third_contraction(c->mesh, c->mat, dof_unpack(c->mesh, qq, c->pins), va, vb, k, out);
        std::memcpy(qbar, out.data(), out.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
// grad: per decoder layer, W (row-major) then b.
int orc_lipschitz_loss2_grad(void* p, int P, const double* Z1, const double* Z2, int nthreads, double* loss,
                             double* grad) {
    try {
        auto* c = static_cast<Ctx*>(p);
        std::vector<std::vector<double>> gW, gb;
        *loss = lipschitz_loss2_grad(c->model, c->mesh, c->mat, c->pins, P, Z1, Z2, gW, gb, nthreads);
        size_t o = 0;
        for (size_t l = 0; l < gW.size(); ++l) {
            std::memcpy(grad + o, gW[l].data(), gW[l].size() * 8);
            o += gW[l].size();
            std::memcpy(grad + o, gb[l].data(), gb[l].size() * 8);
            o += gb[l].size();
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int orc_hardware_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

}  // extern "C"
