// Host-side setup (K0).  See lsb_setup.hpp.
#include "lsb_setup.hpp"

#include <algorithm>
#include <cmath>
#include <set>
#include <stdexcept>

namespace lsb {

double randu(Rng& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
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

namespace {
double det3(const double* m) {
    return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
           m[2] * (m[3] * m[7] - m[4] * m[6]);
}
void edge_matrix(const std::vector<double>& X, const int* t, double* dm) {
    for (int c = 0; c < 3; ++c)
        for (int a = 0; a < 3; ++a) dm[a * 3 + c] = X[3 * t[c + 1] + a] - X[3 * t[0] + a];
}
}  // namespace

void precompute(HostMesh& m) {
    if (static_cast<int>(m.X.size()) != 3 * m.V || static_cast<int>(m.T.size()) != 4 * m.E)
        throw std::invalid_argument("mesh: array sizes do not match V/E");
    for (int e = 0; e < m.E; ++e)
        for (int k = 0; k < 4; ++k) {
            const int v = m.T[4 * e + k];
            if (v < 0 || v >= m.V)
                throw std::runtime_error("mesh: element " + std::to_string(e) + " references vertex " +
                                         std::to_string(v) + " out of range [0," + std::to_string(m.V) + ")");
        }
    m.Dminv.resize(9 * static_cast<size_t>(m.E));
    m.vol.resize(m.E);
    for (int e = 0; e < m.E; ++e) {
        double dm[9];
        edge_matrix(m.X, &m.T[4 * e], dm);
        const double det = det3(dm);
        if (!(det > 1e-14))
            throw std::runtime_error("mesh: element " + std::to_string(e) +
                                     " has non-positive rest measure (det Dm = " + std::to_string(det) + ")");
        const double id = 1.0 / det;
        double* o = &m.Dminv[9 * static_cast<size_t>(e)];
        o[0] = (dm[4] * dm[8] - dm[5] * dm[7]) * id;
        o[1] = (dm[2] * dm[7] - dm[1] * dm[8]) * id;
        o[2] = (dm[1] * dm[5] - dm[2] * dm[4]) * id;
        o[3] = (dm[5] * dm[6] - dm[3] * dm[8]) * id;
        o[4] = (dm[0] * dm[8] - dm[2] * dm[6]) * id;
        o[5] = (dm[2] * dm[3] - dm[0] * dm[5]) * id;
        o[6] = (dm[3] * dm[7] - dm[4] * dm[6]) * id;
        o[7] = (dm[1] * dm[6] - dm[0] * dm[7]) * id;
        o[8] = (dm[0] * dm[4] - dm[1] * dm[3]) * id;
        m.vol[e] = det / 6.0;
    }
    std::set<int> pin_set(m.pinned.begin(), m.pinned.end());
    for (int v : pin_set)
        if (v < 0 || v >= m.V) throw std::runtime_error("mesh: pinned vertex " + std::to_string(v) + " out of range");
    m.pinned.assign(pin_set.begin(), pin_set.end());
    std::vector<char> is_pinned(m.V, 0);
    for (int v : m.pinned) is_pinned[v] = 1;
    m.free_index.assign(m.V, -1);
    m.free_vertex.clear();
    for (int v = 0; v < m.V; ++v)
        if (!is_pinned[v]) {
            m.free_index[v] = static_cast<int>(m.free_vertex.size());
            m.free_vertex.push_back(v);
        }
    m.n_free = static_cast<int>(m.free_vertex.size());
    // CSR over free vertices; entries appended in tet order, so each row is
    // ascending in tet id -- the scatter order of assemble (energy.cpp:421-432).
    std::vector<int> count(m.n_free + 1, 0);
    for (int e = 0; e < m.E; ++e)
        for (int k = 0; k < 4; ++k) {
            const int f = m.free_index[m.T[4 * e + k]];
            if (f >= 0) count[f + 1]++;
        }
    m.csr_ptr.assign(m.n_free + 1, 0);
    for (int f = 0; f < m.n_free; ++f) m.csr_ptr[f + 1] = m.csr_ptr[f] + count[f + 1];
    m.csr_ent.assign(m.csr_ptr[m.n_free], 0);
    std::vector<int> fill(m.csr_ptr.begin(), m.csr_ptr.end() - 1);
    for (int e = 0; e < m.E; ++e)
        for (int k = 0; k < 4; ++k) {
            const int f = m.free_index[m.T[4 * e + k]];
            if (f >= 0) m.csr_ent[fill[f]++] = 4 * e + k;
        }
}

HostMesh make_bar_mesh(int nx, int ny, int nz, double w, double h, double d, double jitter_frac,
                       std::uint64_t seed, bool pin_left) {
    if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("bar: grid sizes must be >= 1");
    HostMesh m;
    const int vx = nx + 1, vy = ny + 1, vz = nz + 1;
    auto vid = [&](int i, int j, int k) { return (i * vy + j) * vz + k; };
    m.V = vx * vy * vz;
    m.X.resize(3 * static_cast<size_t>(m.V));
    for (int i = 0; i < vx; ++i)
        for (int j = 0; j < vy; ++j)
            for (int k = 0; k < vz; ++k) {
                double* x = &m.X[3 * static_cast<size_t>(vid(i, j, k))];
                x[0] = w * i / nx;
                x[1] = h * j / ny;
                x[2] = d * k / nz;
            }
    if (jitter_frac > 0.0) {
        Rng rng = substream(seed, 1);
        const double cell[3] = {w / nx, h / ny, d / nz};
        for (int v = 0; v < m.V; ++v)
            for (int c = 0; c < 3; ++c) m.X[3 * static_cast<size_t>(v) + c] += jitter_frac * cell[c] * randn(rng);
    }
    // Kuhn split: tet p of a cube follows axis permutation p from v000 to v111.
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    m.E = 6 * nx * ny * nz;
    m.T.resize(4 * static_cast<size_t>(m.E));
    int e = 0;
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j)
            for (int k = 0; k < nz; ++k)
                for (int p = 0; p < 6; ++p, ++e) {
                    int* t = &m.T[4 * static_cast<size_t>(e)];
                    int o[3] = {0, 0, 0};
                    t[0] = vid(i, j, k);
                    o[perms[p][0]] = 1;
                    t[1] = vid(i + o[0], j + o[1], k + o[2]);
                    o[perms[p][1]] = 1;
                    t[2] = vid(i + o[0], j + o[1], k + o[2]);
                    t[3] = vid(i + 1, j + 1, k + 1);
                }
    for (int t = 0; t < m.E; ++t) {
        double dm[9];
        int* tt = &m.T[4 * static_cast<size_t>(t)];
        edge_matrix(m.X, tt, dm);
        if (det3(dm) < 0) std::swap(tt[2], tt[3]);
    }
    if (pin_left)
        for (int j = 0; j < vy; ++j)
            for (int k = 0; k < vz; ++k) m.pinned.push_back(vid(0, j, k));
    precompute(m);
    return m;
}

std::vector<double> lump_mass(const HostMesh& m, double density, double* total) {
    if (!(density > 0.0)) throw std::invalid_argument("material: density must be > 0");
    std::vector<double> vm(m.V, 0.0);
    for (int e = 0; e < m.E; ++e) {
        const double mm = density * m.vol[e] * 0.25;
        for (int k = 0; k < 4; ++k) vm[m.T[4 * static_cast<size_t>(e) + k]] += mm;
    }
    double tot = 0.0;
    for (double v : vm) tot += v;
    if (total) *total = tot;
    std::vector<double> diag(3 * static_cast<size_t>(m.n_free));
    for (int f = 0; f < m.n_free; ++f)
        for (int c = 0; c < 3; ++c) diag[3 * static_cast<size_t>(f) + c] = vm[m.free_vertex[f]];
    return diag;
}

HostDecoder make_bar_decoder(const HostMesh& m, int r, int hidden_layers, int width, int act,
                             std::uint64_t seed, double out_scale) {
    if (r < 1 || hidden_layers < 0 || width < 1) throw std::invalid_argument("decoder: bad architecture");
    Rng rng = substream(seed, 0);
    auto xavier = [&rng](int rows, int cols) {
        std::vector<double> W(static_cast<size_t>(rows) * cols);
        const double s = std::sqrt(2.0 / static_cast<double>(rows + cols));
        for (int j = 0; j < cols; ++j)
            for (int i = 0; i < rows; ++i) W[static_cast<size_t>(i) * cols + j] = s * randn(rng);
        return W;
    };
    HostDecoder dec;
    dec.r = r;
    dec.n = 3 * m.n_free;
    int prev = r;
    for (int l = 0; l < hidden_layers; ++l) {
        HostLayer L;
        L.rows = width;
        L.cols = prev;
        L.act = act;
        L.W = xavier(width, prev);
        L.b.assign(width, 0.0);
        dec.layers.push_back(std::move(L));
        prev = width;
    }
    const std::vector<double> full = xavier(3 * m.V, prev);
    HostLayer out;
    out.rows = dec.n;
    out.cols = prev;
    out.act = 0;
    out.W.resize(static_cast<size_t>(dec.n) * prev);
    for (int f = 0; f < m.n_free; ++f) {
        const int v = m.free_vertex[f];
        for (int c = 0; c < 3; ++c)
            std::copy(&full[static_cast<size_t>(3 * v + c) * prev], &full[static_cast<size_t>(3 * v + c) * prev] + prev,
                      &out.W[static_cast<size_t>(3 * f + c) * prev]);
    }
    out.b.assign(dec.n, 0.0);
    dec.layers.push_back(std::move(out));
    dec.shift.resize(dec.n);
    for (int f = 0; f < m.n_free; ++f)
        for (int c = 0; c < 3; ++c) dec.shift[3 * static_cast<size_t>(f) + c] = m.X[3 * static_cast<size_t>(m.free_vertex[f]) + c];
    dec.scale.assign(dec.n, out_scale);
    return dec;
}

}  // namespace lsb
