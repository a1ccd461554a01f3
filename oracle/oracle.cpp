// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.  See oracle.hpp header.
// CPU restatement of the reference hot path; every function cites the
// reference lines it follows (paths relative to /root/reference/).
#include "oracle.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <deque>
#include <set>
#include <stdexcept>
#include <thread>

namespace orc {

// ---------------------------------------------------------------- rng.hpp
double randu(Rng& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
double randu(Rng& rng, double lo, double hi) { return lo + (hi - lo) * randu(rng); }
double randn(Rng& rng) {
    double u1 = 0.0;
    do {
        u1 = randu(rng);
    } while (u1 <= 0.0);
    const double u2 = randu(rng);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}
Rng substream(std::uint64_t seed, std::uint64_t tag) {
    std::uint64_t x = seed + 0x9e3779b97f4a7c15ULL * (tag + 1);
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return Rng(x);
}

// ---------------------------------------------------------------- 3x3 helpers
namespace {

// m[r*3+c]
double det3(const double* m) {
    return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
           m[2] * (m[3] * m[7] - m[4] * m[6]);
}
void inv3(const double* m, double det, double* o) {
    const double id = 1.0 / det;
    o[0] = (m[4] * m[8] - m[5] * m[7]) * id;
    o[1] = (m[2] * m[7] - m[1] * m[8]) * id;
    o[2] = (m[1] * m[5] - m[2] * m[4]) * id;
    o[3] = (m[5] * m[6] - m[3] * m[8]) * id;
    o[4] = (m[0] * m[8] - m[2] * m[6]) * id;
    o[5] = (m[2] * m[3] - m[0] * m[5]) * id;
    o[6] = (m[3] * m[7] - m[4] * m[6]) * id;
    o[7] = (m[1] * m[6] - m[0] * m[7]) * id;
    o[8] = (m[0] * m[4] - m[1] * m[3]) * id;
}
void matmul3(const double* a, const double* b, double* o) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += a[r * 3 + k] * b[k * 3 + c];
            o[r * 3 + c] = s;
        }
}

}  // namespace

// ---------------------------------------------------------------- mesh.cpp
Mesh build_mesh(int V, const double* X, int E, const int* T, const std::vector<int>& pins) {
    // mesh.cpp:90-145 (tetrahedra in 3D only).
    Mesh m;
    m.V = V;
    m.E = E;
    m.X.assign(X, X + 3 * static_cast<size_t>(V));
    m.T.assign(T, T + 4 * static_cast<size_t>(E));
    for (int e = 0; e < E; ++e)
        for (int k = 0; k < 4; ++k) {
            const int v = T[4 * e + k];
            if (v < 0 || v >= V)
                throw std::runtime_error("mesh: element " + std::to_string(e) + " references vertex " +
                                         std::to_string(v) + " out of range [0," + std::to_string(V) + ")");
        }
    m.Dminv.resize(9 * static_cast<size_t>(E));
    m.vol.resize(E);
    for (int e = 0; e < E; ++e) {
        double dm[9];
        const int* t = &T[4 * e];
        for (int c = 0; c < 3; ++c)
            for (int a = 0; a < 3; ++a) dm[a * 3 + c] = X[3 * t[c + 1] + a] - X[3 * t[0] + a];
        const double det = det3(dm);
        if (!(det > 1e-14))  // mesh.cpp:121-125
            throw std::runtime_error("mesh: element " + std::to_string(e) +
                                     " has non-positive rest measure (det Dm = " + std::to_string(det) + ")");
        inv3(dm, det, &m.Dminv[9 * static_cast<size_t>(e)]);
        m.vol[e] = det / 6.0;  // simplex_measure_factor (mesh.cpp:47)
    }
    std::set<int> pin_set(pins.begin(), pins.end());
    for (int v : pin_set)
        if (v < 0 || v >= V) throw std::runtime_error("mesh: pinned vertex " + std::to_string(v) + " out of range");
    m.pinned.assign(pin_set.begin(), pin_set.end());
    m.vertex_pinned.assign(V, 0);
    for (int v : m.pinned) m.vertex_pinned[v] = 1;
    m.free_index.assign(V, -1);
    int slot = 0;
    for (int v = 0; v < V; ++v)
        if (!m.vertex_pinned[v]) m.free_index[v] = slot++;
    m.n_free = slot;
    return m;
}

Mesh make_bar_kuhn(int nx, int ny, int nz, double w, double h, double d, double jitter_frac,
                   std::uint64_t jitter_seed, bool pin_left) {
    const int vx = nx + 1, vy = ny + 1, vz = nz + 1;
    auto vid = [&](int i, int j, int k) { return (i * vy + j) * vz + k; };  // mesh.cpp:359
    const int V = vx * vy * vz;
    std::vector<double> X(3 * static_cast<size_t>(V));
    for (int i = 0; i < vx; ++i)
        for (int j = 0; j < vy; ++j)
            for (int k = 0; k < vz; ++k) {  // mesh.cpp:360-364
                const int v = vid(i, j, k);
                X[3 * v + 0] = w * i / nx;
                X[3 * v + 1] = h * j / ny;
                X[3 * v + 2] = d * k / nz;
            }
    if (jitter_frac > 0.0) {
        // [EXT] config 3: per-vertex N(0, (jitter_frac * cell)^2) per axis, vertex order,
        // stream substream(seed, 1).
        Rng rng = substream(jitter_seed, 1);
        const double cell[3] = {w / nx, h / ny, d / nz};
        for (int v = 0; v < V; ++v)
            for (int c = 0; c < 3; ++c) X[3 * v + c] += jitter_frac * cell[c] * randn(rng);
    }
    // [EXT] Kuhn split: 6 tets per cube around the v000 -> v111 diagonal, one per
    // axis permutation (a, b, c): [v000, v000+e_a, v000+e_a+e_b, v111].
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const int E = 6 * nx * ny * nz;
    std::vector<int> T(4 * static_cast<size_t>(E));
    int e = 0;
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j)
            for (int k = 0; k < nz; ++k)
                for (int p = 0; p < 6; ++p) {
                    int o[3] = {0, 0, 0};
                    int* t = &T[4 * e];
                    t[0] = vid(i, j, k);
                    o[perms[p][0]] = 1;
                    t[1] = vid(i + o[0], j + o[1], k + o[2]);
                    o[perms[p][1]] = 1;
                    t[2] = vid(i + o[0], j + o[1], k + o[2]);
                    t[3] = vid(i + 1, j + 1, k + 1);
                    ++e;
                }
    // Orientation fix (mesh.cpp:386-391): swap the last two vertices when the
    // signed volume is negative.
    for (int t = 0; t < E; ++t) {
        double dm[9];
        int* tt = &T[4 * t];
        for (int c = 0; c < 3; ++c)
            for (int a = 0; a < 3; ++a) dm[a * 3 + c] = X[3 * tt[c + 1] + a] - X[3 * tt[0] + a];
        if (det3(dm) < 0) std::swap(tt[2], tt[3]);
    }
    std::vector<int> pins;
    if (pin_left)  // mesh.cpp:392-395, selected by grid index i == 0
        for (int j = 0; j < vy; ++j)
            for (int k = 0; k < vz; ++k) pins.push_back(vid(0, j, k));
    return build_mesh(V, X.data(), E, T.data(), pins);
}

std::vector<double> lump_mass(const Mesh& m, double density, double* total_mass) {
    // mesh.cpp:417-434
    if (!(density > 0.0)) throw std::invalid_argument("material: density must be > 0");
    std::vector<double> vm(m.V, 0.0);
    for (int e = 0; e < m.E; ++e) {
        const double mm = density * m.vol[e] * 0.25;
        for (int k = 0; k < 4; ++k) vm[m.T[4 * e + k]] += mm;
    }
    double tot = 0.0;
    for (int v = 0; v < m.V; ++v) tot += vm[v];
    if (total_mass) *total_mass = tot;
    std::vector<double> diag(m.num_dofs());
    for (int v = 0; v < m.V; ++v) {
        const int f = m.free_index[v];
        if (f < 0) continue;
        for (int c = 0; c < 3; ++c) diag[3 * f + c] = vm[v];
    }
    return diag;
}

std::vector<double> dof_pack(const Mesh& m, const std::vector<double>& full) {
    std::vector<double> q(m.num_dofs());
    for (int v = 0; v < m.V; ++v) {
        const int f = m.free_index[v];
        if (f < 0) continue;
        for (int c = 0; c < 3; ++c) q[3 * f + c] = full[3 * v + c];
    }
    return q;
}

std::vector<double> dof_unpack(const Mesh& m, const std::vector<double>& q,
                               const std::vector<double>& pin_values) {
    if (static_cast<int>(q.size()) != m.num_dofs())
        throw std::invalid_argument("dof_unpack: q has wrong length");
    std::vector<double> full = pin_values;
    for (int v = 0; v < m.V; ++v) {
        const int f = m.free_index[v];
        if (f < 0) continue;
        for (int c = 0; c < 3; ++c) full[3 * v + c] = q[3 * f + c];
    }
    return full;
}

// ---------------------------------------------------------------- energy.cpp
namespace {

// skew(v) (energy.cpp:17-21), row-major 3x3.
void skew(const double* v, double s, double* out /*3x3 block writer*/, int ld, int r0, int c0) {
    const double m[9] = {0, -v[2], v[1], v[2], 0, -v[0], -v[1], v[0], 0};
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) out[(r0 + r) * ld + c0 + c] = s * m[r * 3 + c];
}

}  // namespace

void element_snh(const Mesh& m, double mu, double lambda, int e, const double* positions,
                 bool want_hessian, ElementDerivatives& out) {
    const int* t = &m.T[4 * e];
    const double* dminv = &m.Dminv[9 * static_cast<size_t>(e)];
    // element_frame (energy.cpp:163-175): Ds, Ds_rest (3 x 3, col c = edge c).
    double ds[9], dd[9];
    for (int c = 0; c < 3; ++c)
        for (int a = 0; a < 3; ++a) {
            const double xs = positions[3 * t[c + 1] + a] - positions[3 * t[0] + a];
            const double xr = m.X[3 * t[c + 1] + a] - m.X[3 * t[0] + a];
            ds[a * 3 + c] = xs;
            dd[a * 3 + c] = xs - xr;
        }
    double F[9], A[9];
    matmul3(dd, dminv, A);  // A = (ds - ds_rest) Dm^-1   (:172)
    matmul3(ds, dminv, F);  // F = ds Dm^-1               (:173)

    // snh_core (energy.cpp:199-221), de = 3, a = 3/4.
    const double de = 3.0, acoef = de / (de + 1.0);
    const double trA = A[0] + A[4] + A[8];
    double sqA = 0.0;
    for (int i = 0; i < 9; ++i) sqA += A[i] * A[i];
    const double i_minus = 2.0 * trA + sqA;  // (:207)
    // j_minus_one (:178-185)
    const double m2 = A[0] * A[4] - A[1] * A[3] + A[0] * A[8] - A[2] * A[6] + A[4] * A[8] - A[5] * A[7];
    const double jm1 = trA + m2 + det3(A);
    const double I = de + i_minus;
    const double psi = 0.5 * mu * i_minus - 0.5 * mu * std::log1p(i_minus / (de + 1.0)) +
                       0.5 * lambda * jm1 * jm1 - acoef * mu * jm1;
    const double u = I + 1.0;
    const double psiI = 0.5 * mu * (1.0 - 1.0 / u);
    const double psiII = 0.5 * mu / (u * u);
    const double psiJ = lambda * jm1 - acoef * mu;
    const double psiJJ = lambda;
    // vec() is column-major: index a + 3 b  (energy.cpp:23-25)
    double gI[9], gJ[9];
    double f[3][3];  // f[b] = column b of F
    for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) {
            f[b][a] = F[a * 3 + b];
            gI[a + 3 * b] = 2.0 * F[a * 3 + b];
        }
    // j_ops_det3 (:67-78): cof columns f1 x f2, f2 x f0, f0 x f1.
    auto cross = [](const double* x, const double* y, double* o) {
        o[0] = x[1] * y[2] - x[2] * y[1];
        o[1] = x[2] * y[0] - x[0] * y[2];
        o[2] = x[0] * y[1] - x[1] * y[0];
    };
    cross(f[1], f[2], &gJ[0]);
    cross(f[2], f[0], &gJ[3]);
    cross(f[0], f[1], &gJ[6]);

    const double vol = m.vol[e];
    out.energy = vol * psi;
    double gradF[9];
    for (int i = 0; i < 9; ++i) gradF[i] = psiI * gI[i] + psiJ * gJ[i];

    // element_shape_matrix (:257-271): B(a+3b, (c+1)*3+a) += Dminv(c,b); B(a+3b, a) -= Dminv(c,b).
    double B[9 * 12];
    for (int i = 0; i < 108; ++i) B[i] = 0.0;
    for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) {
            const int fidx = a + 3 * b;
            for (int c = 0; c < 3; ++c) {
                B[fidx * 12 + (c + 1) * 3 + a] += dminv[c * 3 + b];
                B[fidx * 12 + a] -= dminv[c * 3 + b];
            }
        }
    for (int j = 0; j < 12; ++j) {
        double s = 0.0;
        for (int i = 0; i < 9; ++i) s += B[i * 12 + j] * gradF[i];
        out.grad[j] = vol * s;
    }
    if (want_hessian) {
        // hf = psiII gI gI^T + psiJJ gJ gJ^T + 2 psiI Id + psiJ KJ   (:293-294)
        double KJ[81];
        for (int i = 0; i < 81; ++i) KJ[i] = 0.0;
        skew(f[2], -1.0, KJ, 9, 0, 3);  // kj_det3 (:55-65)
        skew(f[1], 1.0, KJ, 9, 0, 6);
        skew(f[2], 1.0, KJ, 9, 3, 0);
        skew(f[0], -1.0, KJ, 9, 3, 6);
        skew(f[1], -1.0, KJ, 9, 6, 0);
        skew(f[0], 1.0, KJ, 9, 6, 3);
        double hf[81];
        for (int i = 0; i < 9; ++i)
            for (int j = 0; j < 9; ++j)
                hf[i * 9 + j] = psiII * gI[i] * gI[j] + psiJJ * gJ[i] * gJ[j] +
                                (i == j ? 2.0 * psiI : 0.0) + psiJ * KJ[i * 9 + j];
        double hB[9 * 12];  // hf * B
        for (int i = 0; i < 9; ++i)
            for (int j = 0; j < 12; ++j) {
                double s = 0.0;
                for (int k = 0; k < 9; ++k) s += hf[i * 9 + k] * B[k * 12 + j];
                hB[i * 12 + j] = s;
            }
        for (int i = 0; i < 12; ++i)
            for (int j = 0; j < 12; ++j) {
                double s = 0.0;
                for (int k = 0; k < 9; ++k) s += B[k * 12 + i] * hB[k * 12 + j];
                out.hess[i * 12 + j] = vol * s;
            }
    }
}

Assembled assemble(const Mesh& m, const Material& mat, const std::vector<double>& q,
                   const std::vector<double>& pin_positions, const std::vector<int>* subset_ids,
                   const std::vector<double>* subset_w) {
    // energy.cpp:404-437 (elastic branch).
    if (static_cast<int>(q.size()) != m.num_dofs())
        throw std::invalid_argument("assemble: q has wrong length");
    const std::vector<double> X = dof_unpack(m, q, pin_positions);
    Assembled out;
    out.gradient.assign(m.num_dofs(), 0.0);
    const int count = subset_ids ? static_cast<int>(subset_ids->size()) : m.E;
    ElementDerivatives ed;
    for (int k = 0; k < count; ++k) {
        const int e = subset_ids ? (*subset_ids)[k] : k;
        const double w = subset_w ? (*subset_w)[k] : 1.0;
        element_snh(m, mat.mu[e], mat.lambda[e], e, X.data(), false, ed);
        out.value += w * ed.energy;
        for (int v = 0; v < 4; ++v) {  // scatter_gradient (:384-388) via element_dof_map (:273-278)
            const int f = m.free_index[m.T[4 * e + v]];
            if (f < 0) continue;
            for (int c = 0; c < 3; ++c) out.gradient[3 * f + c] += w * ed.grad[3 * v + c];
        }
    }
    return out;
}

void elastic_hessian_apply(const Mesh& m, const Material& mat, const std::vector<double>& positions,
                           const std::vector<double>& in, int k, std::vector<double>& out,
                           const std::vector<int>* ids, const std::vector<double>* w) {
    // energy.cpp:481-493 over an ElementSubset (ids, weights; null = full unit-weight set).
    ElementDerivatives ed;
    std::vector<double> loc_in(12 * static_cast<size_t>(k)), loc_out(12 * static_cast<size_t>(k));
    const int count = ids ? static_cast<int>(ids->size()) : m.E;
    for (int kk = 0; kk < count; ++kk) {
        const int e = ids ? (*ids)[kk] : kk;
        const double we = ids ? (*w)[kk] : 1.0;
        element_snh(m, mat.mu[e], mat.lambda[e], e, positions.data(), true, ed);
        if (ids)
            for (double& v : ed.hess) v *= we;
        int map[12];
        for (int v = 0; v < 4; ++v) {
            const int f = m.free_index[m.T[4 * e + v]];
            for (int c = 0; c < 3; ++c) map[3 * v + c] = f < 0 ? -1 : 3 * f + c;
        }
        for (int i = 0; i < 12; ++i)  // gather_local (:223-231 pattern)
            for (int j = 0; j < k; ++j) loc_in[i * k + j] = map[i] >= 0 ? in[static_cast<size_t>(map[i]) * k + j] : 0.0;
        for (int i = 0; i < 12; ++i)
            for (int j = 0; j < k; ++j) {
                double s = 0.0;
                for (int l = 0; l < 12; ++l) s += ed.hess[i * 12 + l] * loc_in[l * k + j];
                loc_out[i * k + j] = s;
            }
        for (int i = 0; i < 12; ++i)  // scatter_local
            if (map[i] >= 0)
                for (int j = 0; j < k; ++j) out[static_cast<size_t>(map[i]) * k + j] += loc_out[i * k + j];
    }
}

// ---------------------------------------------------------------- net.cpp
double activation_eval(int a, double x, int order) {
    // net.cpp:34-64
    switch (a) {
        case Identity:
            if (order < 0 || order > 3) break;
            return order == 0 ? x : (order == 1 ? 1.0 : 0.0);
        case Silu: {
            const double s = 1.0 / (1.0 + std::exp(-x));
            const double s1 = s * (1.0 - s);
            const double s2 = s1 * (1.0 - 2.0 * s);
            const double s3 = s2 * (1.0 - 2.0 * s) - 2.0 * s1 * s1;
            switch (order) {
                case 0: return x * s;
                case 1: return s + x * s1;
                case 2: return 2.0 * s1 + x * s2;
                case 3: return 3.0 * s2 + x * s3;
            }
            break;
        }
        case Tanh: {
            const double t = std::tanh(x);
            const double t1 = 1.0 - t * t;
            switch (order) {
                case 0: return t;
                case 1: return t1;
                case 2: return -2.0 * t * t1;
                case 3: return -2.0 * t1 * t1 + 4.0 * t * t * t1;
            }
            break;
        }
        case Elu: {
            // [EXT] ELU (alpha = 1).  The x <= 0 branch owns x == 0 at every
            // order, so phi'(0) = phi''(0) = phi'''(0) = 1.
            if (order < 0 || order > 3) break;
            if (x > 0.0) return order == 0 ? x : (order == 1 ? 1.0 : 0.0);
            return order == 0 ? std::expm1(x) : std::exp(x);
        }
    }
    throw std::invalid_argument("activation: derivative order must be 0..3");
}

Model make_bar_decoder(const Mesh& m, int r, int hidden_layers, int width, int act,
                       std::uint64_t seed, double out_scale) {
    Rng rng = substream(seed, 0);
    auto xavier = [&rng](int rows, int cols) {
        std::vector<double> W(static_cast<size_t>(rows) * cols);
        const double s = std::sqrt(2.0 / static_cast<double>(rows + cols));
        for (int j = 0; j < cols; ++j)  // column-major fill (net.cpp:99-100)
            for (int i = 0; i < rows; ++i) W[static_cast<size_t>(i) * cols + j] = s * randn(rng);
        return W;
    };
    Model model;
    model.r = r;
    model.n = m.num_dofs();
    int prev = r;
    for (int l = 0; l < hidden_layers; ++l) {
        Layer L;
        L.rows = width;
        L.cols = prev;
        L.W = xavier(width, prev);
        L.b.assign(width, 0.0);
        L.act = act;
        model.dec.push_back(std::move(L));
        prev = width;
    }
    const int full_rows = 3 * m.V;
    const std::vector<double> Wfull = xavier(full_rows, prev);
    Layer out;
    out.rows = model.n;
    out.cols = prev;
    out.W.resize(static_cast<size_t>(model.n) * prev);
    for (int v = 0; v < m.V; ++v) {
        const int f = m.free_index[v];
        if (f < 0) continue;
        for (int c = 0; c < 3; ++c)
            std::copy(&Wfull[static_cast<size_t>(3 * v + c) * prev], &Wfull[static_cast<size_t>(3 * v + c + 1) * prev],
                      &out.W[static_cast<size_t>(3 * f + c) * prev]);
    }
    out.b.assign(model.n, 0.0);
    out.act = Identity;
    model.dec.push_back(std::move(out));
    model.shift = dof_pack(m, m.X);
    model.scale.assign(model.n, out_scale);
    return model;
}

namespace {
std::vector<double> matvec(const Layer& l, const std::vector<double>& y) {
    std::vector<double> a(l.rows);
    for (int i = 0; i < l.rows; ++i) {
        double s = 0.0;
        const double* w = &l.W[static_cast<size_t>(i) * l.cols];
        for (int j = 0; j < l.cols; ++j) s += w[j] * y[j];
        a[i] = s;
    }
    return a;
}
}  // namespace

std::vector<double> decode(const Model& model, const std::vector<double>& z) {
    // mlp_forward + decode (net.cpp:134-150)
    if (static_cast<int>(z.size()) != model.r) throw std::invalid_argument("decode: z has wrong length");
    std::vector<double> y = z;
    for (const Layer& l : model.dec) {
        std::vector<double> a = matvec(l, y);
        for (int i = 0; i < l.rows; ++i) a[i] = activation_eval(l.act, a[i] + l.b[i], 0);
        y = std::move(a);
    }
    std::vector<double> q(model.n);
    for (int i = 0; i < model.n; ++i) q[i] = model.scale[i] * y[i] + model.shift[i];
    return q;
}

std::vector<double> decode_jacobian(const Model& model, const std::vector<double>& z) {
    // net.cpp:159-190: forward-mode G through the hidden layers, then J_i = (W_L,i G) phi'(a_i) s_i.
    const size_t L = model.dec.size();
    const int r = model.r;
    std::vector<double> y = z;
    std::vector<double> G(static_cast<size_t>(r) * r, 0.0);  // rows(width) x r
    for (int i = 0; i < r; ++i) G[static_cast<size_t>(i) * r + i] = 1.0;
    int width = r;
    for (size_t l = 0; l + 1 < L; ++l) {
        const Layer& ly = model.dec[l];
        std::vector<double> a = matvec(ly, y);
        std::vector<double> A(static_cast<size_t>(ly.rows) * r, 0.0);
        for (int i = 0; i < ly.rows; ++i)
            for (int k = 0; k < ly.cols; ++k) {
                const double w = ly.W[static_cast<size_t>(i) * ly.cols + k];
                for (int c = 0; c < r; ++c) A[static_cast<size_t>(i) * r + c] += w * G[static_cast<size_t>(k) * r + c];
            }
        for (int i = 0; i < ly.rows; ++i) {
            const double ai = a[i] + ly.b[i];
            const double d1 = activation_eval(ly.act, ai, 1);
            for (int c = 0; c < r; ++c) A[static_cast<size_t>(i) * r + c] *= d1;
            a[i] = activation_eval(ly.act, ai, 0);
        }
        y = std::move(a);
        G = std::move(A);
        width = ly.rows;
    }
    const Layer& last = model.dec[L - 1];
    std::vector<double> J(static_cast<size_t>(model.n) * r);
    std::vector<double> row(r);
    for (int i = 0; i < model.n; ++i) {
        const double* w = &last.W[static_cast<size_t>(i) * last.cols];
        double a = 0.0;
        for (int k = 0; k < width; ++k) a += w[k] * y[k];
        a += last.b[i];
        std::fill(row.begin(), row.end(), 0.0);
        for (int k = 0; k < width; ++k)
            for (int c = 0; c < r; ++c) row[c] += w[k] * G[static_cast<size_t>(k) * r + c];
        const double f = activation_eval(last.act, a, 1) * model.scale[i];
        for (int c = 0; c < r; ++c) J[static_cast<size_t>(i) * r + c] = row[c] * f;
    }
    return J;
}

std::vector<double> decode_second_directional(const Model& model, const std::vector<double>& z,
                                              const std::vector<double>& u,
                                              const std::vector<double>& v) {
    // net.cpp:192-240
    const size_t L = model.dec.size();
    std::vector<double> y = z, p = u, t = v, s(model.r, 0.0);
    for (size_t l = 0; l + 1 < L; ++l) {
        const Layer& ly = model.dec[l];
        std::vector<double> a = matvec(ly, y), ap = matvec(ly, p), at = matvec(ly, t), as = matvec(ly, s);
        std::vector<double> ny(ly.rows), np(ly.rows), nt(ly.rows), ns(ly.rows);
        for (int i = 0; i < ly.rows; ++i) {
            const double ai = a[i] + ly.b[i];
            const double d0 = activation_eval(ly.act, ai, 0);
            const double d1 = activation_eval(ly.act, ai, 1);
            const double d2 = activation_eval(ly.act, ai, 2);
            ny[i] = d0;
            np[i] = d1 * ap[i];
            nt[i] = d1 * at[i];
            ns[i] = d2 * (ap[i] * at[i]) + d1 * as[i];
        }
        y = std::move(ny);
        p = std::move(np);
        t = std::move(nt);
        s = std::move(ns);
    }
    const Layer& last = model.dec[L - 1];
    std::vector<double> out(model.n);
    for (int i = 0; i < model.n; ++i) {
        const double* w = &last.W[static_cast<size_t>(i) * last.cols];
        double a = 0.0, ap = 0.0, at = 0.0, as = 0.0;
        for (int k = 0; k < last.cols; ++k) {
            a += w[k] * y[k];
            ap += w[k] * p[k];
            at += w[k] * t[k];
            as += w[k] * s[k];
        }
        a += last.b[i];
        const double d1 = activation_eval(last.act, a, 1);
        const double d2 = activation_eval(last.act, a, 2);
        out[i] = model.scale[i] * (d2 * (ap * at) + d1 * as);
    }
    return out;
}

// ---------------------------------------------------------------- reduced_solver.cpp
namespace {
constexpr double kArmijoC = 1e-4;  // reduced_solver.cpp:36
double dot(const std::vector<double>& a, const std::vector<double>& b) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}
double norm(const std::vector<double>& a) { return std::sqrt(dot(a, a)); }
double inf_norm(const std::vector<double>& a) {
    double m = 0.0;
    for (double v : a) m = std::max(m, std::abs(v));
    return m;
}
void validate(const SolverConfig& cfg) {  // reduced_solver.cpp:14-20
    if (!(cfg.epsilon > 0.0)) throw std::invalid_argument("solver: epsilon must be > 0");
    if (cfg.max_iters < 1 || cfg.max_linesearch < 1)
        throw std::invalid_argument("solver: iteration caps must be >= 1");
    if (!(cfg.dt > 0.0)) throw std::invalid_argument("solver: dt must be > 0");
    if (cfg.lbfgs_history < 1) throw std::invalid_argument("solver: lbfgs history must be >= 1");
}
}  // namespace

ExitReport lbfgs_minimize(const Objective& objective, std::vector<double>& x, const SolverConfig& cfg) {
    // reduced_solver.cpp:58-131 with armijo (:43-54)
    validate(cfg);
    const auto t0 = std::chrono::steady_clock::now();
    ExitReport report;
    auto finish = [&](ExitReport r) {
        r.wall_time_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        return r;
    };
    const size_t n = x.size();
    std::vector<double> g(n);
    double f = objective(x, &g);
    report.evals++;
    std::deque<std::pair<std::vector<double>, std::vector<double>>> history;
    for (int iter = 0; iter < cfg.max_iters; ++iter) {
        report.iterations = iter;
        report.final_grad_inf_norm = inf_norm(g);
        if (report.final_grad_inf_norm < cfg.epsilon) {
            report.code = 1;
            return finish(report);
        }
        std::vector<double> d(n);
        for (size_t i = 0; i < n; ++i) d[i] = -g[i];
        std::vector<double> alpha(history.size());
        for (long i = static_cast<long>(history.size()) - 1; i >= 0; --i) {
            const auto& s = history[i].first;
            const auto& y = history[i].second;
            alpha[i] = dot(s, d) / dot(y, s);
            for (size_t k = 0; k < n; ++k) d[k] -= alpha[i] * y[k];
        }
        if (!history.empty()) {
            const auto& s = history.back().first;
            const auto& y = history.back().second;
            const double gamma = dot(s, y) / dot(y, y);
            for (size_t k = 0; k < n; ++k) d[k] *= gamma;
        }
        for (size_t i = 0; i < history.size(); ++i) {
            const auto& s = history[i].first;
            const auto& y = history[i].second;
            const double beta = dot(y, d) / dot(y, s);
            for (size_t k = 0; k < n; ++k) d[k] += (alpha[i] - beta) * s[k];
        }
        const double gtd = dot(g, d);
        if (!(gtd < 0.0)) {
            report.code = 2;
            return finish(report);
        }
        // armijo (:43-54)
        std::vector<double> trial(n);
        bool ok = false;
        double a = 1.0;
        for (int ls = 0; ls < cfg.max_linesearch; ++ls) {
            for (size_t k = 0; k < n; ++k) trial[k] = x[k] + a * d[k];
            const double ft = objective(trial, nullptr);
            report.value_evals++;
            if (std::isfinite(ft) && ft <= f + kArmijoC * a * gtd) {
                ok = true;
                break;
            }
            a *= 0.5;
        }
        if (!ok) {
            report.code = 3;
            return finish(report);
        }
        std::vector<double> g_new(n);
        const double f_new = objective(trial, &g_new);
        report.evals++;
        std::vector<double> s(n), y(n);
        for (size_t k = 0; k < n; ++k) {
            s[k] = trial[k] - x[k];
            y[k] = g_new[k] - g[k];
        }
        if (dot(s, y) > 1e-12 * norm(s) * norm(y)) {
            history.emplace_back(std::move(s), std::move(y));
            if (static_cast<int>(history.size()) > cfg.lbfgs_history) history.pop_front();
        }
        x = trial;
        f = f_new;
        g = std::move(g_new);
    }
    report.iterations = cfg.max_iters;
    report.final_grad_inf_norm = inf_norm(g);
    report.code = report.final_grad_inf_norm < cfg.epsilon ? 1 : 4;
    return finish(report);
}

// ---- project_spd (energy.cpp:370-380) and projective Newton (reduced_solver.cpp:133-182) ----
namespace {
// cyclic Jacobi: A (n x n, symmetric, row-major) -> eigenvalues w, eigenvectors V (columns)
void jacobi_eigh(std::vector<double> A, int n, std::vector<double>& w, std::vector<double>& V) {
    V.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) off += A[(size_t)p * n + q] * A[(size_t)p * n + q];
        if (off < 1e-30) break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = A[(size_t)p * n + q];
                if (std::fabs(apq) < 1e-300) continue;
                const double app = A[(size_t)p * n + p], aqq = A[(size_t)q * n + q];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
                for (int k = 0; k < n; ++k) {  // A <- A G (columns p, q)
                    const double akp = A[(size_t)k * n + p], akq = A[(size_t)k * n + q];
                    A[(size_t)k * n + p] = cs * akp - sn * akq;
                    A[(size_t)k * n + q] = sn * akp + cs * akq;
                }
                for (int k = 0; k < n; ++k) {  // A <- G^T A (rows p, q)
                    const double apk = A[(size_t)p * n + k], aqk = A[(size_t)q * n + k];
                    A[(size_t)p * n + k] = cs * apk - sn * aqk;
                    A[(size_t)q * n + k] = sn * apk + cs * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    const double vkp = V[(size_t)k * n + p], vkq = V[(size_t)k * n + q];
                    V[(size_t)k * n + p] = cs * vkp - sn * vkq;
                    V[(size_t)k * n + q] = sn * vkp + cs * vkq;
                }
            }
    }
    w.resize(n);
    for (int i = 0; i < n; ++i) w[i] = A[(size_t)i * n + i];
}

// LDL^T (no pivoting: the input is SPD after projection) solve of H d = rhs; false on a
// non-positive pivot
bool ldlt_solve(const std::vector<double>& H, int n, const std::vector<double>& rhs, std::vector<double>& x) {
    std::vector<double> L((size_t)n * n, 0.0), D(n);
    for (int j = 0; j < n; ++j) {
        double dj = H[(size_t)j * n + j];
        for (int k = 0; k < j; ++k) dj -= L[(size_t)j * n + k] * L[(size_t)j * n + k] * D[k];
        if (!(dj > 0.0)) return false;
        D[j] = dj;
        L[(size_t)j * n + j] = 1.0;
        for (int i = j + 1; i < n; ++i) {
            double s = H[(size_t)i * n + j];
            for (int k = 0; k < j; ++k) s -= L[(size_t)i * n + k] * L[(size_t)j * n + k] * D[k];
            L[(size_t)i * n + j] = s / dj;
        }
    }
    x = rhs;
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < i; ++k) x[i] -= L[(size_t)i * n + k] * x[k];
    for (int i = 0; i < n; ++i) x[i] /= D[i];
    for (int i = n - 1; i >= 0; --i)
        for (int k = i + 1; k < n; ++k) x[i] -= L[(size_t)k * n + i] * x[k];
    return true;
}
}  // namespace

std::vector<double> project_spd(const std::vector<double>& H, int n) {
    std::vector<double> w, V;
    jacobi_eigh(H, n, w, V);
    double wmin = w[0], wmax = w[0];
    for (double v : w) {
        wmin = std::min(wmin, v);
        wmax = std::max(wmax, v);
    }
    if (wmin >= 0.0) return H;  // energy.cpp:375
    const double floor = 1e-10 * std::max(wmax, 0.0);
    for (double& v : w)
        if (v < 0.0) v = floor;
    std::vector<double> P((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int k = 0; k < n; ++k) s += V[(size_t)i * n + k] * w[k] * V[(size_t)j * n + k];
            P[(size_t)i * n + j] = s;
        }
    return P;
}

ExitReport projective_newton_minimize(const Objective& objective, const HessianFn& hessian, std::vector<double>& x,
                                      const SolverConfig& cfg) {
    validate(cfg);
    const auto t0 = std::chrono::steady_clock::now();
    auto finish = [&](ExitReport r) {
        r.wall_time_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        return r;
    };
    const int n = (int)x.size();
    std::vector<double> g(n);
    double f = objective(x, &g);
    ExitReport report;
    report.evals++;
    for (int iter = 0; iter < cfg.max_iters; ++iter) {
        report.iterations = iter;
        report.final_grad_inf_norm = inf_norm(g);
        if (report.final_grad_inf_norm < cfg.epsilon) {
            report.code = 1;
            return finish(report);
        }
        const std::vector<double> H = project_spd(hessian(x), n);
        std::vector<double> mg(n), d;
        for (int k = 0; k < n; ++k) mg[k] = -g[k];
        if (!ldlt_solve(H, n, mg, d)) throw std::runtime_error("projective newton: factorization failed");
        for (double v : d)
            if (!std::isfinite(v)) throw std::runtime_error("projective newton: singular system");
        const double gtd = dot(g, d);
        if (!(gtd < 0.0)) {
            report.code = 2;
            return finish(report);
        }
        std::vector<double> trial(n);
        bool ok = false;
        double a = 1.0;
        for (int ls = 0; ls < cfg.max_linesearch; ++ls) {
            for (int k = 0; k < n; ++k) trial[k] = x[k] + a * d[k];
            const double ft = objective(trial, nullptr);
            report.value_evals++;
            if (std::isfinite(ft) && ft <= f + kArmijoC * a * gtd) {
                ok = true;
                break;
            }
            a *= 0.5;
        }
        if (!ok) {
            report.code = 3;
            return finish(report);
        }
        x = trial;
        f = objective(x, &g);
        report.evals++;
    }
    report.iterations = cfg.max_iters;
    report.final_grad_inf_norm = inf_norm(g);
    report.code = report.final_grad_inf_norm < cfg.epsilon ? 1 : 4;
    return finish(report);
}

double ReducedObjective::eval(const std::vector<double>& z, std::vector<double>* grad) const {
    // reduced_solver.cpp:184-202: the gradient goes through a materialised J (:200).
    const std::vector<double> q = decode(*model, z);
    const Assembled ap = assemble(*mesh, *mat, q, pin_positions, cub_ids, cub_w);
    double value = ap.value;
    std::vector<double> full_grad = ap.gradient;
    if (has_qbar) {
        const double inv_dt2 = 1.0 / (dt * dt);
        double s = 0.0;
        for (int i = 0; i < model->n; ++i) {
            const double diff = q[i] - qbar[i];
            s += mass[i] * diff * diff;
        }
        value += 0.5 * inv_dt2 * s;
        for (int i = 0; i < model->n; ++i) full_grad[i] += inv_dt2 * (mass[i] * (q[i] - qbar[i]));
    }
    if (!std::isfinite(value)) throw std::runtime_error("reduced objective: non-finite energy");
    if (grad) {
        const std::vector<double> J = decode_jacobian(*model, z);
        const int r = model->r;
        grad->assign(r, 0.0);
        for (int i = 0; i < model->n; ++i)
            for (int c = 0; c < r; ++c) (*grad)[c] += J[static_cast<size_t>(i) * r + c] * full_grad[i];
    }
    return value;
}

std::vector<double> ReducedObjective::hessian(const std::vector<double>& z) const {
    // reduced_solver.cpp:204-229
    const int r = model->r, n = model->n;
    const std::vector<double> q = decode(*model, z);
    const Assembled ap = assemble(*mesh, *mat, q, pin_positions, cub_ids, cub_w);
    const std::vector<double> J = decode_jacobian(*model, z);
    std::vector<double> residual = ap.gradient;
    std::vector<double> HJ(static_cast<size_t>(n) * r, 0.0);
    elastic_hessian_apply(*mesh, *mat, dof_unpack(*mesh, q, pin_positions), J, r, HJ, cub_ids, cub_w);
    if (has_qbar) {
        const double inv_dt2 = 1.0 / (dt * dt);
        for (int i = 0; i < n; ++i) {
            residual[i] += inv_dt2 * (mass[i] * (q[i] - qbar[i]));
            for (int c = 0; c < r; ++c) HJ[static_cast<size_t>(i) * r + c] += inv_dt2 * mass[i] * J[static_cast<size_t>(i) * r + c];
        }
    }
    std::vector<double> H(static_cast<size_t>(r) * r, 0.0);
    for (int i = 0; i < n; ++i)
        for (int a = 0; a < r; ++a)
            for (int b = 0; b < r; ++b) H[a * r + b] += J[static_cast<size_t>(i) * r + a] * HJ[static_cast<size_t>(i) * r + b];
    std::vector<double> ea(r, 0.0), eb(r, 0.0);
    for (int a = 0; a < r; ++a)
        for (int b = a; b < r; ++b) {
            std::fill(ea.begin(), ea.end(), 0.0);
            std::fill(eb.begin(), eb.end(), 0.0);
            ea[a] = 1.0;
            eb[b] = 1.0;
            const double v = dot(residual, decode_second_directional(*model, z, ea, eb));
            H[a * r + b] += v;
            if (a != b) H[b * r + a] += v;
        }
    return H;
}

ExitReport reduced_step(SimState& state, const std::vector<double>& pin_positions,
                        const std::vector<double>& external_force, const Model& model,
                        const Mesh& mesh, const Material& mat, const std::vector<double>& mass,
                        const SolverConfig& cfg, bool quasi_static, const std::vector<int>* cub_ids,
                        const std::vector<double>* cub_w) {
    // reduced_solver.cpp:235-277 (L-BFGS method); cfg.runtime_cubature (:246) as cub_ids / cub_w
    ReducedObjective obj;
    obj.cub_ids = cub_ids;
    obj.cub_w = cub_w;
    obj.model = &model;
    obj.mesh = &mesh;
    obj.mat = &mat;
    obj.pin_positions = pin_positions;
    obj.mass = mass;
    obj.dt = cfg.dt;
    const std::vector<double> q_prev = dof_pack(mesh, state.positions);
    if (!quasi_static) {
        const std::vector<double> v_prev = dof_pack(mesh, state.velocities);
        obj.has_qbar = true;
        obj.qbar.resize(q_prev.size());
        for (size_t i = 0; i < q_prev.size(); ++i)
            obj.qbar[i] = q_prev[i] + cfg.dt * v_prev[i] + (cfg.dt * cfg.dt) * (external_force[i] / mass[i]);
    }
    std::vector<double> z = state.z;
    const ExitReport report = lbfgs_minimize(
        [&obj](const std::vector<double>& zz, std::vector<double>* g) { return obj.eval(zz, g); }, z, cfg);
    const std::vector<double> q_new = decode(model, z);
    const std::vector<double> pos_new = dof_unpack(mesh, q_new, pin_positions);
    if (quasi_static) {
        std::fill(state.velocities.begin(), state.velocities.end(), 0.0);
    } else {
        for (size_t i = 0; i < pos_new.size(); ++i) state.velocities[i] = (pos_new[i] - state.positions[i]) / cfg.dt;
    }
    state.positions = pos_new;
    state.z = z;
    state.t += cfg.dt;
    return report;
}

std::vector<double> gravity_force(const Mesh& mesh, const std::vector<double>& mass, const double g[3]) {
    // scenario.cpp:193-199
    std::vector<double> f(mesh.num_dofs());
    for (int v = 0; v < mesh.V; ++v) {
        const int fi = mesh.free_index[v];
        if (fi < 0) continue;
        for (int c = 0; c < 3; ++c) f[3 * fi + c] = mass[3 * fi + c] * g[c];
    }
    return f;
}

// ---------------------------------------------------------------- losses.cpp
std::vector<double> reduced_potential_hessian(const Model& model, const Mesh& mesh, const Material& mat,
                                              const std::vector<double>& pin_positions,
                                              const std::vector<double>& z) {
    // losses.cpp:301-316: H = J^T (hess P J) + sum_{a<=b} g . d2f/dz_a dz_b
    ReducedObjective obj;
    obj.model = &model;
    obj.mesh = &mesh;
    obj.mat = &mat;
    obj.pin_positions = pin_positions;
    obj.has_qbar = false;
    return obj.hessian(z);
}

double lipschitz_loss2(const Model& model, const Mesh& mesh, const Material& mat,
                       const std::vector<double>& pin_positions, int P, const double* Z1,
                       const double* Z2, int nthreads) {
    // build_lipschitz_loss (losses.cpp:196-213), order 2, value only.
    if (P <= 0) throw std::invalid_argument("lipschitz loss: no pairs");
    const int r = model.r;
    for (int p = 0; p < P; ++p) {
        double dz2 = 0.0;
        for (int c = 0; c < r; ++c) dz2 += (Z1[p * r + c] - Z2[p * r + c]) * (Z1[p * r + c] - Z2[p * r + c]);
        if (dz2 <= 0.0) throw std::invalid_argument("lipschitz loss: coincident pair");
    }
    std::vector<double> terms(P, 0.0);
    auto work = [&](int p0, int p1) {
        for (int p = p0; p < p1; ++p) {
            const std::vector<double> z1(Z1 + p * r, Z1 + (p + 1) * r), z2(Z2 + p * r, Z2 + (p + 1) * r);
            const auto H1 = reduced_potential_hessian(model, mesh, mat, pin_positions, z1);
            const auto H2 = reduced_potential_hessian(model, mesh, mat, pin_positions, z2);
            double d2 = 0.0, dz2 = 0.0;
            for (size_t k = 0; k < H1.size(); ++k) d2 += (H1[k] - H2[k]) * (H1[k] - H2[k]);
            for (int c = 0; c < r; ++c) dz2 += (z1[c] - z2[c]) * (z1[c] - z2[c]);
            terms[p] = d2 / dz2;
        }
    };
    nthreads = std::max(1, std::min(nthreads, P));
    if (nthreads == 1) {
        work(0, P);
    } else {
        std::vector<std::thread> th;
        for (int k = 0; k < nthreads; ++k) th.emplace_back(work, (P * k) / nthreads, (P * (k + 1)) / nthreads);
        for (auto& t : th) t.join();
    }
    double total = 0.0;
    for (int p = 0; p < P; ++p) total += terms[p];  // sum in pair order (losses.cpp:212)
    return total / static_cast<double>(P);
}


// ---------------------------------------------------------------- third derivatives (energy.cpp)
namespace {

// kj_det3 (energy.cpp:55-65) for a matrix given by its columns x[0..2]: the 9 x 9 block
// matrix of skew(column) blocks (vec index a + 3 b).
void kj_det3_cols(const double x[3][3], double* KJ) {
    for (int i = 0; i < 81; ++i) KJ[i] = 0.0;
    skew(x[2], -1.0, KJ, 9, 0, 3);
    skew(x[1], 1.0, KJ, 9, 0, 6);
    skew(x[2], 1.0, KJ, 9, 3, 0);
    skew(x[0], -1.0, KJ, 9, 3, 6);
    skew(x[1], -1.0, KJ, 9, 6, 0);
    skew(x[0], 1.0, KJ, 9, 6, 3);
}

// The element quantities of element_snh (energy.cpp:280-298) plus psiIII (snh_core :216).
struct SnhFrame {
    double gI[9], gJ[9], KJ[81], B[108];
    double psiI, psiII, psiIII, psiJ, psiJJ, vol;
};

void snh_frame(const Mesh& m, double mu, double lambda, int e, const double* positions, SnhFrame& o) {
    const int* t = &m.T[4 * e];
    const double* dminv = &m.Dminv[9 * static_cast<size_t>(e)];
    double ds[9], dd[9];
    for (int c = 0; c < 3; ++c)
        for (int a = 0; a < 3; ++a) {
            const double xs = positions[3 * t[c + 1] + a] - positions[3 * t[0] + a];
            const double xr = m.X[3 * t[c + 1] + a] - m.X[3 * t[0] + a];
            ds[a * 3 + c] = xs;
            dd[a * 3 + c] = xs - xr;
        }
    double F[9], A[9];
    matmul3(dd, dminv, A);
    matmul3(ds, dminv, F);
    const double de = 3.0, acoef = de / (de + 1.0);
    const double trA = A[0] + A[4] + A[8];
    double sqA = 0.0;
    for (int i = 0; i < 9; ++i) sqA += A[i] * A[i];
    const double i_minus = 2.0 * trA + sqA;
    const double m2 = A[0] * A[4] - A[1] * A[3] + A[0] * A[8] - A[2] * A[6] + A[4] * A[8] - A[5] * A[7];
    const double jm1 = trA + m2 + det3(A);
    const double u = de + i_minus + 1.0;
    o.psiI = 0.5 * mu * (1.0 - 1.0 / u);
    o.psiII = 0.5 * mu / (u * u);
    o.psiIII = -mu / (u * u * u);
    o.psiJ = lambda * jm1 - acoef * mu;
    o.psiJJ = lambda;
    double f[3][3];
    for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) {
            f[b][a] = F[a * 3 + b];
            o.gI[a + 3 * b] = 2.0 * F[a * 3 + b];
        }
    auto cross = [](const double* x, const double* y, double* out) {
        out[0] = x[1] * y[2] - x[2] * y[1];
        out[1] = x[2] * y[0] - x[0] * y[2];
        out[2] = x[0] * y[1] - x[1] * y[0];
    };
    cross(f[1], f[2], &o.gJ[0]);
    cross(f[2], f[0], &o.gJ[3]);
    cross(f[0], f[1], &o.gJ[6]);
    kj_det3_cols(f, o.KJ);
    for (int i = 0; i < 108; ++i) o.B[i] = 0.0;
    for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) {
            const int fidx = a + 3 * b;
            for (int c = 0; c < 3; ++c) {
                o.B[fidx * 12 + (c + 1) * 3 + a] += dminv[c * 3 + b];
                o.B[fidx * 12 + a] -= dminv[c * 3 + b];
            }
        }
    o.vol = m.vol[e];
}

}  // namespace

void element_third_contraction(const Mesh& m, double mu, double lambda, int e, const double* positions,
                               const double* M_local, double* out12) {
    // snh_third_contraction (energy.cpp:303-320): grad_x <H_e(x), M>, M symmetric 12 x 12.
    SnhFrame c;
    snh_frame(m, mu, lambda, e, positions, c);
    double BM[9 * 12], MF[81];  // MF = B M B^T
    for (int i = 0; i < 9; ++i)
        for (int j = 0; j < 12; ++j) {
            double s = 0.0;
            for (int k = 0; k < 12; ++k) s += c.B[i * 12 + k] * M_local[k * 12 + j];
            BM[i * 12 + j] = s;
        }
    for (int i = 0; i < 9; ++i)
        for (int j = 0; j < 9; ++j) {
            double s = 0.0;
            for (int k = 0; k < 12; ++k) s += BM[i * 12 + k] * c.B[j * 12 + k];
            MF[i * 9 + j] = s;
        }
    double trM = 0.0, qII = 0.0, kJM = 0.0, MgI[9], MgJ[9];
    for (int i = 0; i < 9; ++i) {
        trM += MF[i * 9 + i];
        double s1 = 0.0, s2 = 0.0;
        for (int j = 0; j < 9; ++j) {
            s1 += MF[i * 9 + j] * c.gI[j];
            s2 += MF[i * 9 + j] * c.gJ[j];
            kJM += c.KJ[i * 9 + j] * MF[i * 9 + j];
        }
        MgI[i] = s1;
        MgJ[i] = s2;
    }
    for (int i = 0; i < 9; ++i) qII += c.gI[i] * MgI[i];
    // j_third (energy.cpp:120-131), 3D: g[i + 3 j] = <kj_det3(E_ij), MF>
    double j3[9];
    for (int j = 0; j < 3; ++j)
        for (int i = 0; i < 3; ++i) {
            double basis[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
            basis[j][i] = 1.0;  // column j, row i
            double K[81];
            kj_det3_cols(basis, K);
            double s = 0.0;
            for (int k = 0; k < 81; ++k) s += K[k] * MF[k];
            j3[i + 3 * j] = s;
        }
    double v[9];
    for (int i = 0; i < 9; ++i) {
        double kjmgj = 0.0;
        for (int j = 0; j < 9; ++j) kjmgj += c.KJ[i * 9 + j] * MgJ[j];
        v[i] = c.psiIII * qII * c.gI[i] + 4.0 * c.psiII * MgI[i] + 2.0 * c.psiJJ * kjmgj +
               2.0 * trM * c.psiII * c.gI[i] + c.psiJJ * kJM * c.gJ[i] + c.psiJ * j3[i];
    }
    for (int j = 0; j < 12; ++j) {
        double s = 0.0;
        for (int i = 0; i < 9; ++i) s += c.B[i * 12 + j] * v[i];
        out12[j] = c.vol * s;
    }
}

void elastic_third_contraction(const Mesh& m, const Material& mat, const std::vector<double>& positions,
                               const std::vector<double>& A, const std::vector<double>& B, int k,
                               std::vector<double>& qbar, const std::vector<int>* ids,
                               const std::vector<double>* w) {
    // energy.cpp:495-510: M_e = (A_e B_e^T + B_e A_e^T) / 2, qbar += w_e local.
    const int count = ids ? static_cast<int>(ids->size()) : m.E;
    std::vector<double> Ae(12 * static_cast<size_t>(k)), Be(12 * static_cast<size_t>(k));
    double M[144], local[12];
    for (int kk = 0; kk < count; ++kk) {
        const int e = ids ? (*ids)[kk] : kk;
        const double we = ids ? (*w)[kk] : 1.0;
        int map[12];
        for (int v = 0; v < 4; ++v) {
            const int f = m.free_index[m.T[4 * e + v]];
            for (int c = 0; c < 3; ++c) map[3 * v + c] = f < 0 ? -1 : 3 * f + c;
        }
        for (int i = 0; i < 12; ++i)
            for (int j = 0; j < k; ++j) {
                Ae[i * k + j] = map[i] >= 0 ? A[static_cast<size_t>(map[i]) * k + j] : 0.0;
                Be[i * k + j] = map[i] >= 0 ? B[static_cast<size_t>(map[i]) * k + j] : 0.0;
            }
        for (int i = 0; i < 12; ++i)
            for (int j = 0; j < 12; ++j) {
                double s = 0.0;
                for (int l = 0; l < k; ++l) s += Ae[i * k + l] * Be[j * k + l] + Be[i * k + l] * Ae[j * k + l];
                M[i * 12 + j] = 0.5 * s;
            }
        element_third_contraction(m, mat.mu[e], mat.lambda[e], e, positions.data(), M, local);
        for (int i = 0; i < 12; ++i)
            if (map[i] >= 0) qbar[map[i]] += we * local[i];
    }
}

// ---------------------------------------------------------------- theta gradient (losses.cpp, tape.cpp)
namespace {

// One point's forward trace: tape_decode with want_jacobian (losses.cpp:56-85) and every
// tape_second_directional (losses.cpp:105-118) for the pairs c <= d.
struct PointTrace {
    std::vector<std::vector<double>> y;     // y[l + 1] = layer l output; y[0] = z
    std::vector<std::vector<double>> a;     // pre-activations
    std::vector<std::vector<double>> G;     // G[l + 1] (rows x r); G[0] = I
    std::vector<std::vector<double>> ahat;  // W_l G[l]
    std::vector<std::vector<std::vector<double>>> S;  // S[l + 1][pair]; S[0] = 0
    std::vector<std::vector<double>> Ws;    // W_l S[l][pair] (per layer, pair-major rows x npair)
    std::vector<double> q, J;               // n, n x r
};

void trace_point(const Model& model, const std::vector<double>& z, PointTrace& t) {
    const int r = model.r, L = static_cast<int>(model.dec.size()), np = r * (r + 1) / 2;
    t.y.assign(1, z);
    t.G.assign(1, std::vector<double>(static_cast<size_t>(r) * r, 0.0));
    for (int i = 0; i < r; ++i) t.G[0][static_cast<size_t>(i) * r + i] = 1.0;
    t.S.assign(1, std::vector<std::vector<double>>(np, std::vector<double>(r, 0.0)));
    t.a.clear();
    t.ahat.clear();
    t.Ws.clear();
    for (int l = 0; l < L; ++l) {
        const Layer& ly = model.dec[l];
        const int R = ly.rows, K = ly.cols;
        std::vector<double> a = matvec(ly, t.y[l]), y(R), ah(static_cast<size_t>(R) * r, 0.0),
            G(static_cast<size_t>(R) * r), Ws(static_cast<size_t>(R) * np, 0.0);
        for (int i = 0; i < R; ++i) {
            a[i] += ly.b[i];
            y[i] = activation_eval(ly.act, a[i], 0);
            for (int k = 0; k < K; ++k) {
                const double w = ly.W[static_cast<size_t>(i) * K + k];
                for (int c = 0; c < r; ++c) ah[static_cast<size_t>(i) * r + c] += w * t.G[l][static_cast<size_t>(k) * r + c];
                for (int s = 0; s < np; ++s) Ws[static_cast<size_t>(i) * np + s] += w * t.S[l][s][k];
            }
            const double d1 = activation_eval(ly.act, a[i], 1);
            for (int c = 0; c < r; ++c) G[static_cast<size_t>(i) * r + c] = ah[static_cast<size_t>(i) * r + c] * d1;
        }
        std::vector<std::vector<double>> S(np, std::vector<double>(R));
        for (int i = 0; i < R; ++i) {
            const double d1 = activation_eval(ly.act, a[i], 1), d2 = activation_eval(ly.act, a[i], 2);
            int s = 0;
            for (int c = 0; c < r; ++c)
                for (int d = c; d < r; ++d, ++s)
                    S[s][i] = d2 * (ah[static_cast<size_t>(i) * r + c] * ah[static_cast<size_t>(i) * r + d]) +
                              d1 * Ws[static_cast<size_t>(i) * np + s];
        }
        t.a.push_back(std::move(a));
        t.y.push_back(std::move(y));
        t.ahat.push_back(std::move(ah));
        t.G.push_back(std::move(G));
        t.Ws.push_back(std::move(Ws));
        t.S.push_back(std::move(S));
    }
    const int n = model.n;
    t.q.resize(n);
    t.J.resize(static_cast<size_t>(n) * r);
    for (int i = 0; i < n; ++i) {
        t.q[i] = t.y[L][i] * model.scale[i] + model.shift[i];
        for (int c = 0; c < r; ++c) t.J[static_cast<size_t>(i) * r + c] = t.G[L][static_cast<size_t>(i) * r + c] * model.scale[i];
    }
}

// Per point: H (tape_reduced_derivative order 2, losses.cpp:136-146) and the state its
// backward needs.
struct PointState {
    PointTrace tr;
    std::vector<double> X, g, HJ, H;  // positions, grad P, K J, H (r x r)
};

void point_forward(const Model& model, const Mesh& mesh, const Material& mat, const std::vector<double>& pins,
                   const std::vector<double>& z, PointState& st) {
    const int r = model.r, n = model.n, L = static_cast<int>(model.dec.size());
    trace_point(model, z, st.tr);
    st.X = dof_unpack(mesh, st.tr.q, pins);
    st.g = assemble(mesh, mat, st.tr.q, pins).gradient;        // potential_gradient (tape.cpp:245-260)
    st.HJ.assign(static_cast<size_t>(n) * r, 0.0);            // potential_hessian_apply (tape.cpp:262-279)
    elastic_hessian_apply(mesh, mat, st.X, st.tr.J, r, st.HJ);
    st.H.assign(static_cast<size_t>(r) * r, 0.0);
    for (int i = 0; i < n; ++i)                               // matmul_tn(J, hj)
        for (int a = 0; a < r; ++a)
            for (int b = 0; b < r; ++b)
                st.H[a * r + b] += st.tr.J[static_cast<size_t>(i) * r + a] * st.HJ[static_cast<size_t>(i) * r + b];
    int s = 0;
    for (int a = 0; a < r; ++a)
        for (int b = a; b < r; ++b, ++s) {  // dot(g, s_ab), symmetric_from_entries
            double v = 0.0;
            for (int i = 0; i < n; ++i) v += st.g[i] * st.tr.S[L][s][i] * model.scale[i];
            st.H[a * r + b] += v;
            if (a != b) st.H[b * r + a] += v;
        }
}

// Reverse sweep of one point's H with adjoint Hbar (r x r), accumulating dL/dtheta.
void point_backward(const Model& model, const Mesh& mesh, const Material& mat, const PointState& st,
                    const std::vector<double>& Hbar, std::vector<std::vector<double>>& gW,
                    std::vector<std::vector<double>>& gb) {
    const int r = model.r, n = model.n, L = static_cast<int>(model.dec.size()), np = r * (r + 1) / 2;
    const PointTrace& tr = st.tr;
    // symmetric_from_entries backward (tape.cpp:212-222)
    std::vector<double> ebar(np);
    {
        int s = 0;
        for (int a = 0; a < r; ++a)
            for (int b = a; b < r; ++b, ++s) ebar[s] = Hbar[a * r + b] + (a != b ? Hbar[b * r + a] : 0.0);
    }
    // matmul_tn(J, hj) backward (tape.cpp:162-167): Jbar = hj Hbar^T, hjbar = J Hbar
    std::vector<double> Jbar(static_cast<size_t>(n) * r, 0.0), hjbar(static_cast<size_t>(n) * r, 0.0);
    for (int i = 0; i < n; ++i)
        for (int a = 0; a < r; ++a) {
            double s1 = 0.0, s2 = 0.0;
            for (int b = 0; b < r; ++b) {
                s1 += st.HJ[static_cast<size_t>(i) * r + b] * Hbar[a * r + b];
                s2 += tr.J[static_cast<size_t>(i) * r + b] * Hbar[b * r + a];
            }
            Jbar[static_cast<size_t>(i) * r + a] = s1;
            hjbar[static_cast<size_t>(i) * r + a] = s2;
        }
    // potential_hessian_apply backward (tape.cpp:271-277): Ybar += H hjbar; qbar += third(J, hjbar)
    elastic_hessian_apply(mesh, mat, st.X, hjbar, r, Jbar);
    std::vector<double> qbar(n, 0.0);
    elastic_third_contraction(mesh, mat, st.X, tr.J, hjbar, r, qbar);
    // dot(g, s_ab) backward: gbar = sum ebar s_ab; sbar_ab = ebar g
    std::vector<double> gbar(n, 0.0);
    for (int s = 0; s < np; ++s)
        for (int i = 0; i < n; ++i) gbar[i] += ebar[s] * tr.S[L][s][i] * model.scale[i];
    // potential_gradient backward (tape.cpp:254-259): qbar += H gbar
    elastic_hessian_apply(mesh, mat, st.X, gbar, 1, qbar);
    // decoder: q = y_L * scale + shift, J = G_L * scale, s_ab = S_L * scale
    std::vector<double> ybar(n), Gbar(static_cast<size_t>(n) * r);
    std::vector<std::vector<double>> Sbar(np, std::vector<double>(n));
    for (int i = 0; i < n; ++i) {
        ybar[i] = qbar[i] * model.scale[i];
        for (int c = 0; c < r; ++c) Gbar[static_cast<size_t>(i) * r + c] = Jbar[static_cast<size_t>(i) * r + c] * model.scale[i];
        for (int s = 0; s < np; ++s) Sbar[s][i] = ebar[s] * st.g[i] * model.scale[i];
    }
    for (int l = L - 1; l >= 0; --l) {
        const Layer& ly = model.dec[l];
        const int R = ly.rows, K = ly.cols;
        std::vector<double>& W = gW[l];
        std::vector<double>& bv = gb[l];
        std::vector<double> abar(R, 0.0), ahbar(static_cast<size_t>(R) * r, 0.0);
        std::vector<std::vector<double>> Sprev(np, std::vector<double>(K, 0.0));
        for (int i = 0; i < R; ++i) {
            const double ai = tr.a[l][i];
            const double d1 = activation_eval(ly.act, ai, 1), d2 = activation_eval(ly.act, ai, 2),
                         d3 = activation_eval(ly.act, ai, 3);
            // second directional recurrence (losses.cpp:111-116) backward, every pair
            int s = 0;
            for (int c = 0; c < r; ++c)
                for (int d = c; d < r; ++d, ++s) {
                    const double tb = Sbar[s][i];
                    if (tb == 0.0) continue;
                    const double pc = tr.ahat[l][static_cast<size_t>(i) * r + c], pd = tr.ahat[l][static_cast<size_t>(i) * r + d];
                    abar[i] += tb * pc * pd * d3 + tb * tr.Ws[l][static_cast<size_t>(i) * np + s] * d2;
                    ahbar[static_cast<size_t>(i) * r + c] += tb * d2 * pd;
                    ahbar[static_cast<size_t>(i) * r + d] += tb * d2 * pc;
                    const double u = tb * d1;  // carried = d1 * (W s_prev)
                    for (int k = 0; k < K; ++k) {
                        W[static_cast<size_t>(i) * K + k] += u * tr.S[l][s][k];
                        Sprev[s][k] += ly.W[static_cast<size_t>(i) * K + k] * u;
                    }
                }
            // G = ahat * d1 (losses.cpp:75-78)
            double gsum = 0.0;
            for (int c = 0; c < r; ++c) {
                const double gb_ = Gbar[static_cast<size_t>(i) * r + c];
                ahbar[static_cast<size_t>(i) * r + c] += gb_ * d1;
                gsum += gb_ * tr.ahat[l][static_cast<size_t>(i) * r + c];
            }
            abar[i] += gsum * d2 + ybar[i] * d1;  // d1 = act'(a); y = act(a)
        }
        // ahat = W G_prev; a = W y_prev + b
        std::vector<double> Gprev(static_cast<size_t>(K) * r, 0.0), yprev(K, 0.0);
        for (int i = 0; i < R; ++i) {
            bv[i] += abar[i];
            for (int k = 0; k < K; ++k) {
                double s = abar[i] * tr.y[l][k];
                for (int c = 0; c < r; ++c) s += ahbar[static_cast<size_t>(i) * r + c] * tr.G[l][static_cast<size_t>(k) * r + c];
                W[static_cast<size_t>(i) * K + k] += s;
                const double w = ly.W[static_cast<size_t>(i) * K + k];
                yprev[k] += w * abar[i];
                for (int c = 0; c < r; ++c) Gprev[static_cast<size_t>(k) * r + c] += w * ahbar[static_cast<size_t>(i) * r + c];
            }
        }
        ybar = std::move(yprev);
        Gbar = std::move(Gprev);
        Sbar = std::move(Sprev);
    }
}

}  // namespace

double lipschitz_loss2_grad(const Model& model, const Mesh& mesh, const Material& mat,
                            const std::vector<double>& pin_positions, int P, const double* Z1, const double* Z2,
                            std::vector<std::vector<double>>& gW, std::vector<std::vector<double>>& gb,
                            int nthreads) {
    // build_lipschitz_loss (losses.cpp:196-213) order 2 + Tape::backward (tape.cpp:46-59).
    if (P <= 0) throw std::invalid_argument("lipschitz loss: no pairs");
    const int r = model.r, L = static_cast<int>(model.dec.size());
    for (int p = 0; p < P; ++p) {
        double dz2 = 0.0;
        for (int c = 0; c < r; ++c) dz2 += (Z1[p * r + c] - Z2[p * r + c]) * (Z1[p * r + c] - Z2[p * r + c]);
        if (dz2 <= 0.0) throw std::invalid_argument("lipschitz loss: coincident pair");
    }
    nthreads = std::max(1, std::min(nthreads, P));
    std::vector<double> terms(P, 0.0);
    std::vector<std::vector<std::vector<double>>> tW(nthreads), tb(nthreads);
    for (int k = 0; k < nthreads; ++k)
        for (int l = 0; l < L; ++l) {
            tW[k].emplace_back(model.dec[l].W.size(), 0.0);
            tb[k].emplace_back(model.dec[l].b.size(), 0.0);
        }
    auto work = [&](int k, int p0, int p1) {
        PointState s1, s2;
        std::vector<double> Hbar(static_cast<size_t>(r) * r);
        for (int p = p0; p < p1; ++p) {
            const std::vector<double> z1(Z1 + p * r, Z1 + (p + 1) * r), z2(Z2 + p * r, Z2 + (p + 1) * r);
            point_forward(model, mesh, mat, pin_positions, z1, s1);
            point_forward(model, mesh, mat, pin_positions, z2, s2);
            double d2 = 0.0, dz2 = 0.0;
            for (size_t i = 0; i < s1.H.size(); ++i) d2 += (s1.H[i] - s2.H[i]) * (s1.H[i] - s2.H[i]);
            for (int c = 0; c < r; ++c) dz2 += (z1[c] - z2[c]) * (z1[c] - z2[c]);
            terms[p] = d2 / dz2;
            // scale(sum, 1/P) . scale(dot(diff, diff), 1/dz2) . sub(d1, d2) backward
            const double f = 2.0 / (dz2 * static_cast<double>(P));
            for (size_t i = 0; i < Hbar.size(); ++i) Hbar[i] = f * (s1.H[i] - s2.H[i]);
            point_backward(model, mesh, mat, s1, Hbar, tW[k], tb[k]);
            for (double& v : Hbar) v = -v;
            point_backward(model, mesh, mat, s2, Hbar, tW[k], tb[k]);
        }
    };
    if (nthreads == 1) {
        work(0, 0, P);
    } else {
        std::vector<std::thread> th;
        for (int k = 0; k < nthreads; ++k) th.emplace_back(work, k, (P * k) / nthreads, (P * (k + 1)) / nthreads);
        for (auto& t : th) t.join();
    }
    gW.assign(L, {});
    gb.assign(L, {});
    for (int l = 0; l < L; ++l) {
        gW[l].assign(model.dec[l].W.size(), 0.0);
        gb[l].assign(model.dec[l].b.size(), 0.0);
        for (int k = 0; k < nthreads; ++k) {
            for (size_t i = 0; i < gW[l].size(); ++i) gW[l][i] += tW[k][l][i];
            for (size_t i = 0; i < gb[l].size(); ++i) gb[l][i] += tb[k][l][i];
        }
    }
    double total = 0.0;
    for (int p = 0; p < P; ++p) total += terms[p];
    return total / static_cast<double>(P);
}

}  // namespace orc
