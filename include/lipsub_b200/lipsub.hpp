// C++ mirror of the reference `lipsub` hot-path interface over the C ABI
// (include/lipsub_b200.h).  Header-only; link against liblipsub_b200.so.
//
// Names, argument meaning and error behaviour follow the reference headers
// (paths relative to /root/reference/):
//   SolverConfig, ExitReport, exit_code_name  proj/include/lipsub/reduced_solver.hpp:16-39
//   Objective (nullable gradient pointer)     proj/include/lipsub/reduced_solver.hpp:51
//   lbfgs_minimize                            proj/include/lipsub/reduced_solver.hpp:55
//   ReducedObjective::eval / as_objective     proj/include/lipsub/reduced_solver.hpp:59-72
//   SimState, FrameInput, reduced_step        proj/include/lipsub/reduced_solver.hpp:43-48, 75-84
//   reduced_potential_hessian, lipschitz_loss proj/include/lipsub/losses.hpp:111-133
//   HessianFn, projective_newton_minimize     proj/include/lipsub/reduced_solver.hpp:53-57
//   ReducedObjective::hessian                 proj/include/lipsub/reduced_solver.hpp:71
// Eigen::VectorXd is replaced by std::vector<double> (Eigen is not a dependency).
// Errors: LSB_EINVAL -> std::invalid_argument, everything else ->
// std::runtime_error (the reference's exception types); solver outcomes are
// exit codes, never exceptions (reduced_solver.hpp:28-39).
#pragma once

#include <cmath>
#include <chrono>
#include <cstdint>
#include <deque>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../lipsub_b200.h"

namespace lipsub_b200 {

using VectorXd = std::vector<double>;

inline void check(lsb_status s) {
    if (s == LSB_OK) return;
    const std::string msg = lsb_last_error();
    if (s == LSB_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

struct SolverConfig {
    double epsilon = 1e-5;
    int max_iters = 1024;
    int max_linesearch = 128;
    int lbfgs_history = 8;
    double dt = 0.05;

    void validate() const {  // reduced_solver.cpp:14-20
        if (!(epsilon > 0.0)) throw std::invalid_argument("solver: epsilon must be > 0");
        if (max_iters < 1 || max_linesearch < 1) throw std::invalid_argument("solver: iteration caps must be >= 1");
        if (!(dt > 0.0)) throw std::invalid_argument("solver: dt must be > 0");
        if (lbfgs_history < 1) throw std::invalid_argument("solver: lbfgs history must be >= 1");
    }
    lsb_solver_config c() const { return {epsilon, max_iters, max_linesearch, lbfgs_history, dt}; }
};

struct ExitReport {
    enum Code { Converged = 1, Saddle = 2, LinesearchCap = 3, IterationCap = 4 };
    Code code = IterationCap;
    int iterations = 0;
    double final_grad_inf_norm = 0.0;
    double wall_time_ms = 0.0;
    int value_evals = 0, grad_evals = 0;

    static ExitReport from(const lsb_exit_report& r) {
        ExitReport e;
        e.code = static_cast<Code>(r.code);
        e.iterations = r.iterations;
        e.final_grad_inf_norm = r.final_grad_inf_norm;
        e.wall_time_ms = r.wall_time_ms;
        e.value_evals = r.value_evals;
        e.grad_evals = r.grad_evals;
        return e;
    }
};

inline const char* exit_code_name(ExitReport::Code code) {
    switch (code) {
        case ExitReport::Converged: return "I";
        case ExitReport::Saddle: return "II";
        case ExitReport::LinesearchCap: return "III";
        case ExitReport::IterationCap: return "IV";
    }
    return "?";
}

// value + gradient callback; the gradient pointer may be null.
using Objective = std::function<double(const VectorXd&, VectorXd*)>;

// Host L-BFGS + Armijo for an arbitrary objective (reduced_solver.cpp:43-131).
inline ExitReport lbfgs_minimize(const Objective& objective, VectorXd& x, const SolverConfig& cfg) {
    cfg.validate();
    const auto t0 = std::chrono::steady_clock::now();
    auto dot = [](const VectorXd& a, const VectorXd& b) {
        double s = 0.0;
        for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
        return s;
    };
    auto finish = [&](ExitReport r) {
        r.wall_time_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        return r;
    };
    const size_t n = x.size();
    VectorXd g(n);
    double f = objective(x, &g);
    std::deque<std::pair<VectorXd, VectorXd>> hist;
    ExitReport rep;
    for (int iter = 0; iter < cfg.max_iters; ++iter) {
        rep.iterations = iter;
        double gn = 0.0;
        for (double v : g) gn = std::max(gn, std::abs(v));
        rep.final_grad_inf_norm = gn;
        if (gn < cfg.epsilon) {
            rep.code = ExitReport::Converged;
            return finish(rep);
        }
        VectorXd d(n);
        for (size_t i = 0; i < n; ++i) d[i] = -g[i];
        std::vector<double> alpha(hist.size());
        for (long i = (long)hist.size() - 1; i >= 0; --i) {
            alpha[i] = dot(hist[i].first, d) / dot(hist[i].second, hist[i].first);
            for (size_t k = 0; k < n; ++k) d[k] -= alpha[i] * hist[i].second[k];
        }
        if (!hist.empty()) {
            const double gam = dot(hist.back().first, hist.back().second) / dot(hist.back().second, hist.back().second);
            for (double& v : d) v *= gam;
        }
        for (size_t i = 0; i < hist.size(); ++i) {
            const double beta = dot(hist[i].second, d) / dot(hist[i].second, hist[i].first);
            for (size_t k = 0; k < n; ++k) d[k] += (alpha[i] - beta) * hist[i].first[k];
        }
        const double gtd = dot(g, d);
        if (!(gtd < 0.0)) {
            rep.code = ExitReport::Saddle;
            return finish(rep);
        }
        VectorXd trial(n);
        bool ok = false;
        double a = 1.0;
        for (int ls = 0; ls < cfg.max_linesearch; ++ls) {
            for (size_t k = 0; k < n; ++k) trial[k] = x[k] + a * d[k];
            const double ft = objective(trial, nullptr);
            if (std::isfinite(ft) && ft <= f + 1e-4 * a * gtd) {
                ok = true;
                break;
            }
            a *= 0.5;
        }
        if (!ok) {
            rep.code = ExitReport::LinesearchCap;
            return finish(rep);
        }
        VectorXd gn2(n);
        const double fn = objective(trial, &gn2);
        VectorXd s(n), y(n);
        for (size_t k = 0; k < n; ++k) {
            s[k] = trial[k] - x[k];
            y[k] = gn2[k] - g[k];
        }
        if (dot(s, y) > 1e-12 * std::sqrt(dot(s, s)) * std::sqrt(dot(y, y))) {
            hist.emplace_back(s, y);
            if ((int)hist.size() > cfg.lbfgs_history) hist.pop_front();
        }
        x = trial;
        f = fn;
        g = gn2;
    }
    rep.iterations = cfg.max_iters;
    double gn = 0.0;
    for (double v : g) gn = std::max(gn, std::abs(v));
    rep.final_grad_inf_norm = gn;
    rep.code = gn < cfg.epsilon ? ExitReport::Converged : ExitReport::IterationCap;
    return finish(rep);
}

// Mesh + material + decoder resident on one GPU (the reference's
// PotentialContext + MassMatrix + SubspaceModel, energy.hpp:46-60).
class ReducedSystem {
  public:
    ReducedSystem(const lsb_mesh_desc& mesh, const lsb_decoder_desc& dec, int precision = LSB_FP64, int device = 0) {
        check(lsb_create(&mesh, &dec, precision, device, &ctx_));
        int n = 0, r = 0;
        check(lsb_get_info(ctx_, &n, &r, nullptr, nullptr, nullptr, nullptr));
        n_ = n;
        r_ = r;
    }
    ~ReducedSystem() { lsb_destroy(ctx_); }
    ReducedSystem(const ReducedSystem&) = delete;
    ReducedSystem& operator=(const ReducedSystem&) = delete;

    int n() const { return n_; }
    int r() const { return r_; }
    lsb_context* handle() const { return ctx_; }

    void set_inertia(const VectorXd* qbar, double dt) { check(lsb_set_inertia(ctx_, qbar ? qbar->data() : nullptr, dt)); }
    void set_pin_positions(const VectorXd& pins) { check(lsb_set_pin_positions(ctx_, pins.data())); }
    VectorXd decode(const VectorXd& z) {
        if ((int)z.size() != r_) throw std::invalid_argument("decode: z has wrong length");
        VectorXd q(n_);
        check(lsb_decode(ctx_, z.data(), q.data()));
        return q;
    }
    // decode_jacobian (net.hpp:52-53): n x r, row-major.
    VectorXd decode_jacobian(const VectorXd& z) {
        if ((int)z.size() != r_) throw std::invalid_argument("decode: z has wrong length");
        VectorXd J((size_t)n_ * r_);
        check(lsb_decode_jacobian(ctx_, z.data(), J.data()));
        return J;
    }
    // decode_second_directional (net.hpp:57-59).
    VectorXd decode_second_directional(const VectorXd& z, const VectorXd& u, const VectorXd& v) {
        if ((int)z.size() != r_ || (int)u.size() != r_ || (int)v.size() != r_)
            throw std::invalid_argument("decode: z has wrong length");
        VectorXd out(n_);
        check(lsb_decode_second_directional(ctx_, z.data(), u.data(), v.data(), out.data()));
        return out;
    }
    // assemble (energy.hpp:99-101), elastic branch: value and (optionally) the free-DOF gradient.
    double assemble(const VectorXd& q, VectorXd* grad) {
        if ((int)q.size() != n_) throw std::invalid_argument("assemble: q has wrong length");
        double v = 0.0;
        if (grad) grad->resize(n_);
        check(lsb_assemble(ctx_, q.data(), &v, grad ? grad->data() : nullptr));
        return v;
    }
    // elastic_hessian_apply (energy.hpp:109-112): out += H(q) in, n x k row-major.
    void elastic_hessian_apply(const VectorXd& q, int k, const VectorXd& in, VectorXd& out) {
        if ((int)q.size() != n_ || (long long)in.size() != (long long)n_ * k || in.size() != out.size())
            throw std::invalid_argument("elastic_hessian_apply: shape mismatch");
        check(lsb_elastic_hessian_apply(ctx_, q.data(), k, in.data(), out.data()));
    }
    double eval(const VectorXd& z, VectorXd* grad) {
        if ((int)z.size() != r_) throw std::invalid_argument("decode: z has wrong length");
        double v = 0.0;
        if (grad) grad->resize(r_);
        check(lsb_eval(ctx_, z.data(), &v, grad ? grad->data() : nullptr));
        return v;
    }
    // Runtime cubature (ElementSubset, energy.hpp:25-36); empty ids restore the full set.
    void set_cubature(const std::vector<int>& ids, const std::vector<double>& weights) {
        if (ids.size() != weights.size()) throw std::invalid_argument("cubature: ids and weights differ in length");
        check(lsb_set_cubature(ctx_, (int)ids.size(), ids.empty() ? nullptr : ids.data(),
                               weights.empty() ? nullptr : weights.data()));
    }
    // ReducedObjective::hessian (reduced_solver.cpp:204-229) for a batch of points.
    std::vector<double> objective_hessians(const std::vector<double>& Z) {
        const int B = (int)(Z.size() / r_);
        std::vector<double> H((size_t)B * r_ * r_);
        check(lsb_objective_hessian(ctx_, B, Z.data(), H.data()));
        return H;
    }
    // reduced_potential_hessian (losses.cpp:301-316) for a batch of points (B x r row-major).
    std::vector<double> hessians(const std::vector<double>& Z) {
        const int B = (int)(Z.size() / r_);
        std::vector<double> H((size_t)B * r_ * r_);
        check(lsb_hessian_batched(ctx_, B, Z.data(), H.data()));
        return H;
    }

  private:
    lsb_context* ctx_ = nullptr;
    int n_ = 0, r_ = 0;
};

// E(z) = |f(z) - qbar|_M^2 / (2 dt^2) + P(f(z)); without qbar the inertia term is dropped.
struct ReducedObjective {
    ReducedSystem* system = nullptr;
    std::optional<VectorXd> qbar;
    double dt = 0.05;

    void bind() const { system->set_inertia(qbar ? &*qbar : nullptr, dt); }
    double eval(const VectorXd& z, VectorXd* grad) const {
        bind();
        return system->eval(z, grad);
    }
    Objective as_objective() const {
        bind();
        ReducedSystem* s = system;
        return [s](const VectorXd& z, VectorXd* g) { return s->eval(z, g); };
    }
    // d2E/dz2 (row-major r x r), reduced_solver.cpp:204-229
    std::vector<double> hessian(const VectorXd& z) const {
        bind();
        return system->objective_hessians(z);
    }
};

using HessianFn = std::function<std::vector<double>(const VectorXd&)>;  // row-major n x n

// Device overload: evaluations and objective Hessians on the GPU (lsb_projective_newton).
inline ExitReport projective_newton_minimize(const ReducedObjective& obj, VectorXd& z, const SolverConfig& cfg) {
    cfg.validate();
    obj.bind();
    lsb_exit_report rep{};
    const lsb_solver_config c = cfg.c();
    check(lsb_projective_newton(obj.system->handle(), z.data(), &c, &rep));
    return ExitReport::from(rep);
}

// Device-resident overload: the whole L-BFGS loop runs in one CUDA graph.
inline ExitReport lbfgs_minimize(const ReducedObjective& obj, VectorXd& z, const SolverConfig& cfg) {
    cfg.validate();
    obj.bind();
    lsb_exit_report rep{};
    const lsb_solver_config c = cfg.c();
    check(lsb_lbfgs(obj.system->handle(), z.data(), &c, &rep));
    return ExitReport::from(rep);
}

struct SimState {
    VectorXd positions, velocities;  // V*3
    VectorXd z;
    double t = 0.0;
};
struct FrameInput {
    VectorXd pin_positions;   // V*3
    VectorXd external_force;  // n
};

// One implicit-Euler (or quasi-static) reduced step (reduced_solver.cpp:235-277).
inline ExitReport reduced_step(SimState& state, const FrameInput& frame, ReducedSystem& system,
                               const SolverConfig& cfg, bool quasi_static) {
    cfg.validate();
    lsb_context* c = system.handle();
    check(lsb_set_pin_positions(c, frame.pin_positions.data()));
    check(lsb_set_external_force(c, frame.external_force.data()));
    check(lsb_set_state(c, state.positions.data(), state.velocities.data(), state.z.data()));
    lsb_exit_report rep{};
    const lsb_solver_config cc = cfg.c();
    check(lsb_step(c, &cc, quasi_static ? 1 : 0, &rep));
    check(lsb_get_state(c, state.positions.data(), state.velocities.data(), state.z.data(), nullptr));
    state.t += cfg.dt;
    return ExitReport::from(rep);
}

// Order-2 Lipschitz loss over pairs (losses.cpp:196-213, 237-244).
inline double lipschitz_loss(ReducedSystem& system, const std::vector<std::pair<VectorXd, VectorXd>>& pairs) {
    if (pairs.empty()) throw std::invalid_argument("lipschitz loss: no pairs");
    const int r = system.r();
    std::vector<double> Z1, Z2;
    for (const auto& [a, b] : pairs) {
        Z1.insert(Z1.end(), a.begin(), a.end());
        Z2.insert(Z2.end(), b.begin(), b.end());
    }
    double loss = 0.0;
    check(lsb_lipschitz_loss(system.handle(), (int)pairs.size(), Z1.data(), Z2.data(), &loss));
    (void)r;
    return loss;
}

// The same loss and dL/dtheta, flattened per decoder layer as W (row-major) then b
// (build_lipschitz_loss + Tape::backward, losses.cpp:196-213, tape.cpp:46-79).
inline double lipschitz_loss_grad(ReducedSystem& system, const std::vector<std::pair<VectorXd, VectorXd>>& pairs,
                                  std::vector<double>& grad) {
    if (pairs.empty()) throw std::invalid_argument("lipschitz loss: no pairs");
    std::vector<double> Z1, Z2;
    for (const auto& [a, b] : pairs) {
        Z1.insert(Z1.end(), a.begin(), a.end());
        Z2.insert(Z2.end(), b.begin(), b.end());
    }
    double loss = 0.0;
    check(lsb_lipschitz_loss_grad(system.handle(), (int)pairs.size(), Z1.data(), Z2.data(), &loss, grad.data()));
    return loss;
}

}  // namespace lipsub_b200
