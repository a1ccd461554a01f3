// Host-side d x d algebra of the projective-Newton reduced solver: SPD projection
// (project_spd, proj/src/energy.cpp:370-380) and the LDL^T solve of the projected
// Newton system (reduced_solver.cpp:156-159).  d <= 64, so this is negligible next to
// the device evaluations and Hessians it consumes.
#pragma once

#include <algorithm>
#include <cmath>
#include <vector>

namespace lsb {
namespace newton {

// cyclic Jacobi eigendecomposition of a symmetric n x n (row-major) matrix
inline void eigh(std::vector<double> A, int n, std::vector<double>& w, std::vector<double>& V) {
    V.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0;
    auto at = [&](int i, int j) -> double& { return A[(size_t)i * n + j]; };
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) off += at(p, q) * at(p, q);
        if (off < 1e-30) break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = at(p, q);
                if (std::fabs(apq) < 1e-300) continue;
                const double theta = (at(q, q) - at(p, p)) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < n; ++k) {
                    const double akp = at(k, p), akq = at(k, q);
                    at(k, p) = c * akp - s * akq;
                    at(k, q) = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {
                    const double apk = at(p, k), aqk = at(q, k);
                    at(p, k) = c * apk - s * aqk;
                    at(q, k) = s * apk + c * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    const double vkp = V[(size_t)k * n + p], vkq = V[(size_t)k * n + q];
                    V[(size_t)k * n + p] = c * vkp - s * vkq;
                    V[(size_t)k * n + q] = s * vkp + c * vkq;
                }
            }
    }
    w.resize(n);
    for (int i = 0; i < n; ++i) w[i] = at(i, i);
}

// project_spd: unchanged if the smallest eigenvalue is >= 0, else negative eigenvalues
// clamp to 1e-10 * max(lambda_max, 0)
inline std::vector<double> project_spd(const std::vector<double>& H, int n) {
    std::vector<double> w, V;
    eigh(H, n, w, V);
    const double wmin = *std::min_element(w.begin(), w.end()), wmax = *std::max_element(w.begin(), w.end());
    if (wmin >= 0.0) return H;
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

// LDL^T solve H x = b (H SPD after projection); false on a non-positive pivot
inline bool ldlt_solve(const std::vector<double>& H, int n, const std::vector<double>& b, std::vector<double>& x) {
    std::vector<double> L((size_t)n * n, 0.0), D(n);
    for (int j = 0; j < n; ++j) {
        double dj = H[(size_t)j * n + j];
        for (int k = 0; k < j; ++k) dj -= L[(size_t)j * n + k] * L[(size_t)j * n + k] * D[k];
        if (!(dj > 0.0)) return false;
        D[j] = dj;
        for (int i = j + 1; i < n; ++i) {
            double s = H[(size_t)i * n + j];
            for (int k = 0; k < j; ++k) s -= L[(size_t)i * n + k] * L[(size_t)j * n + k] * D[k];
            L[(size_t)i * n + j] = s / dj;
        }
    }
    x = b;
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < i; ++k) x[i] -= L[(size_t)i * n + k] * x[k];
    for (int i = 0; i < n; ++i) x[i] /= D[i];
    for (int i = n - 1; i >= 0; --i)
        for (int k = i + 1; k < n; ++k) x[i] -= L[(size_t)k * n + i] * x[k];
    return true;
}

}  // namespace newton
}  // namespace lsb
