// C++ API check (include/lipsub_b200/lipsub.hpp): builds config-1 sized data
// through the setup helpers, checks E/grad against central differences
// (reference test_solvers.cpp:134-146 pattern), device vs host L-BFGS on the same
// objective, reduced_step, and error mapping.  Exit code 0 = pass.
#include <cmath>
#include <cstdio>
#include <vector>

#include "lipsub_b200/lipsub.hpp"

using namespace lipsub_b200;

static int fails = 0;
#define EXPECT(c)                                                        \
    do {                                                                 \
        if (!(c)) {                                                      \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);      \
            ++fails;                                                     \
        }                                                                \
    } while (0)

int main() {
    int V, E, np;
    check(lsb_bar_mesh_size(4, 4, 16, 1, &V, &E, &np));
    std::vector<double> X(3 * V);
    std::vector<int32_t> T(4 * E), pins(np);
    check(lsb_make_bar_mesh(4, 4, 16, 0.25, 0.25, 1.0, 0.0, 0, 1, X.data(), T.data(), pins.data()));
    std::vector<double> mu(E), lam(E);
    check(lsb_lame_from_young(E, 1e5, 1e5, 0.35, 0, mu.data(), lam.data()));
    const int r = 8, h = 64, L = 6, n = 3 * (V - np);
    std::vector<int> rows = {h, h, h, h, h, n}, cols = {r, h, h, h, h, h}, acts = {3, 3, 3, 3, 3, 0};
    size_t tot = 0;
    for (int l = 0; l < L; ++l) tot += (size_t)rows[l] * cols[l];
    std::vector<double> Wp(tot), shift(n), scale(n);
    check(lsb_make_bar_decoder(V, X.data(), np, pins.data(), r, 5, h, 3, 0, 1e-2, Wp.data(), shift.data(), scale.data()));
    std::vector<std::vector<double>> bs(L);
    std::vector<const double*> Wptr(L), bptr(L);
    size_t off = 0;
    for (int l = 0; l < L; ++l) {
        Wptr[l] = Wp.data() + off;
        off += (size_t)rows[l] * cols[l];
        bs[l].assign(rows[l], 0.0);
        bptr[l] = bs[l].data();
    }
    lsb_mesh_desc md{V, X.data(), E, T.data(), np, pins.data(), mu.data(), lam.data(), 1000.0};
    lsb_decoder_desc dd{r, L, rows.data(), cols.data(), acts.data(), Wptr.data(), bptr.data(), shift.data(), scale.data()};
    ReducedSystem sys(md, dd, LSB_FP64, 0);
    EXPECT(sys.n() == n && sys.r() == r);

    std::vector<double> mass(n);
    double tm = 0;
    check(lsb_get_mass(sys.handle(), mass.data(), &tm));
    EXPECT(std::abs(tm - 62.5) < 1e-9);
    const double dt = 1.0 / 60.0;
    VectorXd qbar = shift;
    for (int i = 2; i < n; i += 3) qbar[i] += dt * dt * -9.8;
    ReducedObjective obj{&sys, qbar, dt};

    VectorXd z(r);
    for (int k = 0; k < r; ++k) z[k] = 0.3 * std::sin(1.0 + k);
    VectorXd g;
    const double e = obj.eval(z, &g);
    EXPECT(std::isfinite(e) && (int)g.size() == r);
    double worst = 0.0;
    for (int k = 0; k < r; ++k) {
        VectorXd zp = z, zm = z;
        zp[k] += 1e-6;
        zm[k] -= 1e-6;
        const double fd = (obj.eval(zp, nullptr) - obj.eval(zm, nullptr)) / 2e-6;
        worst = std::max(worst, std::abs(fd - g[k]) / (std::abs(g[k]) + 1e-12));
    }
    EXPECT(worst < 1e-5);

    SolverConfig cfg;
    cfg.lbfgs_history = 5;
    cfg.dt = dt;
    VectorXd zd(r, 0.0), zh(r, 0.0);
    const ExitReport rd = lbfgs_minimize(obj, zd, cfg);               // device-resident
    const ExitReport rh = lbfgs_minimize(obj.as_objective(), zh, cfg);  // host loop, device evals
    EXPECT(rd.code == ExitReport::Converged && rh.code == ExitReport::Converged);
    EXPECT(rd.iterations == rh.iterations);
    double dz = 0.0;
    for (int k = 0; k < r; ++k) dz = std::max(dz, std::abs(zd[k] - zh[k]));
    EXPECT(dz < 1e-9);

    SimState st{X, VectorXd(3 * V, 0.0), VectorXd(r, 0.0), 0.0};
    VectorXd f(n);
    for (int i = 0; i < n; ++i) f[i] = (i % 3 == 2) ? -9.8 * mass[i] : 0.0;
    FrameInput fr{X, f};
    const ExitReport rs = reduced_step(st, fr, sys, cfg, false);
    EXPECT(rs.code == ExitReport::Converged && std::abs(st.t - dt) < 1e-15);
    for (int k = 0; k < r; ++k) dz = std::max(dz, std::abs(st.z[k] - zd[k]));
    EXPECT(dz < 1e-9);  // first step from rest == timestep-0 objective minimiser

    bool threw = false;
    try {
        SolverConfig bad;
        bad.epsilon = 0.0;
        lbfgs_minimize(obj, zd, bad);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw);
    std::printf("%s: E=%.12e |g|=%zu fdworst=%.2e iters=%d/%d\n", fails ? "FAILED" : "ok", e, g.size(), worst,
                rd.iterations, rh.iterations);
    return fails ? 1 : 0;
}
