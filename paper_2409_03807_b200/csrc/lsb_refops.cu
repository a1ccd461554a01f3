// The reference's secondary hot-path primitives as device operations on a context's resident
// mesh, material and decoder (SURVEY §8(b) "Other ★ entry points"):
//
//   refops_assemble              <- assemble, elastic branch        (energy.hpp:99-101, energy.cpp:404-437)
//   refops_element_snh           <- element_snh (+ local Hessian)    (energy.hpp:71-72, energy.cpp:280-298)
//   refops_elastic_hessian_apply <- elastic_hessian_apply            (energy.hpp:109-112, energy.cpp:481-493)
//   refops_decode_jacobian       <- decode_jacobian                  (net.hpp:52-53, net.cpp:159-190)
//   refops_decode_second_dir     <- decode_second_directional        (net.hpp:57-59, net.cpp:192-240)
//
// They reuse the product's element records (storage precision), CSR force slots and the
// deterministic per-vertex gather, so a call is a handful of small kernels on the context
// stream; fp64 arithmetic throughout.  Element sums are fixed-order (block partials in block
// order), forces are summed per vertex in ascending tet order (energy.cpp:384-388): repeated
// calls are bitwise identical.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "lsb_context.hpp"
#include "lsb_refops.hpp"

namespace lsb {

namespace {

constexpr int kRefGrid = 296;  // 2 x 148 SMs: element passes (fixed grid => fixed summation order)

struct RefBuffers final : BatchedBase {
    double* xfree = nullptr;  // n: rest coordinates of the free DOFs
    double* xrest = nullptr;  // V x 3
    double* dU = nullptr;     // V x 4: direction / displacement scratch
    double* part = nullptr;   // kRefGrid energy partials
    double* scal = nullptr;   // 1 result scalar
    double* vec = nullptr;    // generic n-vector scratch (inputs / outputs)
    double* vec2 = nullptr;   // second n-vector scratch
    double* hid = nullptr;    // hidden-layer scratch: 2 x (kMaxHidden x (kMaxLatent + 1)) + a
    int n = 0, V = 0;
};

RefBuffers& bufs(Context& c) {
    if (!c.refops) {
        auto* b = new RefBuffers();
        c.refops.reset(b);
        const HostMesh& m = c.mesh;
        b->n = c.n;
        b->V = m.V;
        std::vector<double> xf(c.n);
        for (int f = 0; f < m.n_free; ++f)
            for (int k = 0; k < 3; ++k) xf[3 * (size_t)f + k] = m.X[3 * (size_t)m.free_vertex[f] + k];
        b->xfree = static_cast<double*>(c.dmalloc(8 * (size_t)c.n));
        c.copy(b->xfree, xf.data(), 8 * xf.size(), cudaMemcpyHostToDevice, "refops xfree");
        b->xrest = static_cast<double*>(c.dmalloc(8 * 3 * (size_t)m.V));
        c.copy(b->xrest, m.X.data(), 8 * 3 * (size_t)m.V, cudaMemcpyHostToDevice, "refops xrest");
        b->dU = static_cast<double*>(c.dmalloc(8 * 4 * (size_t)m.V));
        b->part = static_cast<double*>(c.dmalloc(8 * kRefGrid));
        b->scal = static_cast<double*>(c.dmalloc(8));
        b->vec = static_cast<double*>(c.dmalloc(8 * (size_t)std::max(c.n, 3 * kMaxLatent)));
        b->vec2 = static_cast<double*>(c.dmalloc(8 * (size_t)std::max(c.n, 3 * kMaxLatent)));
        b->hid = static_cast<double*>(c.dmalloc(8 * (2 * (size_t)kMaxHidden * (kMaxLatent + 1) + kMaxHidden)));
    }
    return *static_cast<RefBuffers*>(c.refops.get());
}

// ---------------------------------------------------------------- kernels
// U rows of the free vertices from a free-DOF configuration q (dof_unpack, mesh.cpp:448-461);
// pinned rows keep the pin displacement (upload_pins).
__global__ void q_to_u_kernel(int n, const int* vfree, const double* q, const double* xfree, double* U) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int f = i / 3, c = i - 3 * f;
        U[4 * (size_t)vfree[f] + c] = q[i] - xfree[i];
    }
}

// Direction rows: free rows from column j of the n x k matrix `in` (dir_free_kernel), pinned rows 0.
__global__ void zero_u_kernel(int V, double* dU) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
        reinterpret_cast<double4*>(dU)[v] = make_double4(0.0, 0.0, 0.0, 0.0);
}
__global__ void dir_free_kernel(int n, const int* vfree, const double* in, int k, int j, double* dU) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int f = i / 3, c = i - 3 * f;
        dU[4 * (size_t)vfree[f] + c] = in[(size_t)i * k + j];
    }
}

// Full-space positions (V x 3) -> displacements (V x 4).
__global__ void pos_to_u_kernel(int V, const double* pos, const double* xrest, double* U) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
#pragma unroll
        for (int c = 0; c < 3; ++c) U[4 * (size_t)v + c] = pos[3 * (size_t)v + c] - xrest[3 * (size_t)v + c];
        U[4 * (size_t)v + 3] = 0.0;
    }
}

// Strain increment A = (Ds - Ds_rest) Dm^-1 of displacements u0..u3 (element_frame, energy.cpp:163-175).
__device__ __forceinline__ void strain_of(const double* u0, const double* u1, const double* u2, const double* u3,
                                          const double* rec, double* A) {
    double D[9];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        D[a * 3 + 0] = u1[a] - u0[a];
        D[a * 3 + 1] = u2[a] - u0[a];
        D[a * 3 + 2] = u3[a] - u0[a];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            A[a * 3 + b] = D[a * 3 + 0] * rec[0 * 3 + b] + D[a * 3 + 1] * rec[1 * 3 + b] + D[a * 3 + 2] * rec[2 * 3 + b];
}

// 12 local forces vol P Dm^-T from a stress-like 3x3 matrix P (energy.cpp:290-291).
__device__ __forceinline__ void forces_of(const double* P, const double* rec, double* f) {
    const double vol = rec[9];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double s0 = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double hv =
                vol * (P[a * 3 + 0] * rec[c * 3 + 0] + P[a * 3 + 1] * rec[c * 3 + 1] + P[a * 3 + 2] * rec[c * 3 + 2]);
            f[(c + 1) * 3 + a] = hv;
            s0 += hv;
        }
        f[a] = -s0;
    }
}

// Cofactor matrix of M (row-major): column b = m_{b+1} x m_{b+2} (m_b = column b).
__device__ __forceinline__ void cofactor(const double* M, double* C) {
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        const int b1 = (b + 1) % 3, b2 = (b + 2) % 3;
        C[0 * 3 + b] = M[1 * 3 + b1] * M[2 * 3 + b2] - M[2 * 3 + b1] * M[1 * 3 + b2];
        C[1 * 3 + b] = M[2 * 3 + b1] * M[0 * 3 + b2] - M[0 * 3 + b1] * M[2 * 3 + b2];
        C[2 * 3 + b] = M[0 * 3 + b1] * M[1 * 3 + b2] - M[1 * 3 + b1] * M[0 * 3 + b2];
    }
}

// Directional derivative of the SNH stress: dP = dP/dF [dF] at F = I + A, i.e. the element
// Hessian vol B^T [psi_II g_I g_I^T + psi_JJ g_J g_J^T + 2 psi_I I + psi_J K_J] B applied to a
// direction (energy.cpp:213-218, 293-295): g_I = 2F, g_J = cof F, psi_I = mu/2 (3+i)/(4+i),
// psi_II = mu/2 / (4+i)^2, psi_J = lambda (J-1) - 3/4 mu, psi_JJ = lambda, K_J dF = d cof F [dF].
__device__ __forceinline__ void snh_dP(const double* A, const double* dF, double mu, double lambda, double* dP) {
    double F[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) F[k] = A[k] + ((k % 4) == 0 ? 1.0 : 0.0);
    const double trA = A[0] + A[4] + A[8];
    double q = 0.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) q += A[k] * A[k];
    const double m2 = A[0] * A[4] - A[1] * A[3] + A[0] * A[8] - A[2] * A[6] + A[4] * A[8] - A[5] * A[7];
    double cA[9];
    cofactor(A, cA);
    const double detA = A[0] * cA[0] + A[3] * cA[3] + A[6] * cA[6];
    const double jm1 = trA + m2 + detA;
    const double i_m = 2.0 * trA + q;
    const double psiI = 0.5 * mu * (3.0 + i_m) / (4.0 + i_m);
    const double psiII = 0.5 * mu / ((4.0 + i_m) * (4.0 + i_m));
    const double psiJ = lambda * jm1 - 0.75 * mu;
    double cF[9];
    cofactor(F, cF);
    double di = 0.0, dJ = 0.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        di += 2.0 * F[k] * dF[k];
        dJ += cF[k] * dF[k];
    }
    // d cof F [dF]: column b = df_{b+1} x f_{b+2} + f_{b+1} x df_{b+2}
    double dC[9];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        const int b1 = (b + 1) % 3, b2 = (b + 2) % 3;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const int r1 = (r + 1) % 3, r2 = (r + 2) % 3;
            dC[r * 3 + b] = dF[r1 * 3 + b1] * F[r2 * 3 + b2] - dF[r2 * 3 + b1] * F[r1 * 3 + b2] +
                            F[r1 * 3 + b1] * dF[r2 * 3 + b2] - F[r2 * 3 + b1] * dF[r1 * 3 + b2];
        }
    }
#pragma unroll
    for (int k = 0; k < 9; ++k)
        dP[k] = 2.0 * psiI * dF[k] + 2.0 * psiII * di * F[k] + psiJ * dC[k] + lambda * dJ * cF[k];
}

// Element pass of assemble: energies (block partials) and forces at their CSR slots.
template <typename TS>
__global__ void __launch_bounds__(256) asm_elem_kernel(int E, const int4* tets, const TS* rec, const double* U,
                                                       const int4* fpos, double* forces, double* part, int want_grad) {
    __shared__ double red[32];
    double eacc = 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        const int4 t = __ldg(tets + e);
        double u[4][3], rc[12], f[12];
        load_u(U, t.x, u[0]);
        load_u(U, t.y, u[1]);
        load_u(U, t.z, u[2]);
        load_u(U, t.w, u[3]);
        load_rec<TS>(rec, (size_t)e, rc);
        eacc += tet_energy_forces(u[0], u[1], u[2], u[3], rc, f);
        if (want_grad) store_forces_csr_t<TS>(forces, __ldg(fpos + e), f);
    }
    const double tot = block_sum(eacc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// Element pass of the Hessian apply: H_e d at the configuration U, direction dU, into CSR slots.
template <typename TS>
__global__ void __launch_bounds__(256) hvp_elem_kernel(int E, const int4* tets, const TS* rec, const double* U,
                                                       const double* dU, const int4* fpos, double* forces) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        const int4 t = __ldg(tets + e);
        const int vs[4] = {t.x, t.y, t.z, t.w};
        double u[4][3], du[4][3], rc[12];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            load_u(U, vs[k], u[k]);
            load_u(dU, vs[k], du[k]);
        }
        load_rec<TS>(rec, (size_t)e, rc);
        double A[9], dF[9], dP[9], f[12];
        strain_of(u[0], u[1], u[2], u[3], rc, A);
        strain_of(du[0], du[1], du[2], du[3], rc, dF);
        snh_dP(A, dF, rc[10], rc[11], dP);
        forces_of(dP, rc, f);
        store_forces_csr_t<TS>(forces, __ldg(fpos + e), f);
    }
}

// Per free vertex: its CSR segment summed in ascending tet order (energy.cpp:384-388);
// out[3f + c * ...] (+)= sum (column j of an n x k row-major matrix).
template <typename TS>
__global__ void grad_gather_kernel(int n_free, const int* csr_ptr, const double* forces, double* out, int k, int j,
                                   int accumulate) {
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < n_free; f += gridDim.x * blockDim.x) {
        const int b = csr_ptr[f], e = csr_ptr[f + 1];
        double g[3] = {0.0, 0.0, 0.0};
        for (int s = b; s < e; ++s) {
            if constexpr (sizeof(TS) == 4) {
                const float4 v = __ldcg(reinterpret_cast<const float4*>(forces) + s);
                g[0] += (double)v.x;
                g[1] += (double)v.y;
                g[2] += (double)v.z;
            } else {
                g[0] += __ldcg(forces + 4 * (size_t)s + 0);
                g[1] += __ldcg(forces + 4 * (size_t)s + 1);
                g[2] += __ldcg(forces + 4 * (size_t)s + 2);
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double* o = out + (size_t)(3 * f + c) * k + j;
            *o = accumulate ? *o + g[c] : g[c];
        }
    }
}

__global__ void sum_partials_kernel(const double* part, int count, double* out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int b = threadIdx.x; b < count; b += blockDim.x) s += part[b];
    const double t = block_sum(s, red);
    if (threadIdx.x == 0) *out = t;
}

// element_snh for listed tets at displacements U: energy, local gradient (vertex-major k*3+a)
// and, optionally, the 12 x 12 local Hessian (columns = H applied to unit directions).
template <typename TS>
__global__ void element_snh_kernel(int count, const int* ids, const int4* tets, const TS* rec, const double* U,
                                   double* energy, double* grad, double* hess) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < count; q += gridDim.x * blockDim.x) {
        const int e = ids[q];
        const int4 t = tets[e];
        double u[4][3], rc[12], f[12];
        load_u(U, t.x, u[0]);
        load_u(U, t.y, u[1]);
        load_u(U, t.z, u[2]);
        load_u(U, t.w, u[3]);
        load_rec<TS>(rec, (size_t)e, rc);
        energy[q] = tet_energy_forces(u[0], u[1], u[2], u[3], rc, f);
#pragma unroll
        for (int k = 0; k < 12; ++k) grad[(size_t)q * 12 + k] = f[k];
        if (!hess) continue;
        double A[9];
        strain_of(u[0], u[1], u[2], u[3], rc, A);
        const double z3[3] = {0.0, 0.0, 0.0};
        for (int jcol = 0; jcol < 12; ++jcol) {
            double d[4][3];
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int a = 0; a < 3; ++a) d[k][a] = (k * 3 + a == jcol) ? 1.0 : z3[a];
            double dF[9], dP[9], h[12];
            strain_of(d[0], d[1], d[2], d[3], rc, dF);
            snh_dP(A, dF, rc[10], rc[11], dP);
            forces_of(dP, rc, h);
#pragma unroll
            for (int i = 0; i < 12; ++i) hess[(size_t)q * 144 + i * 12 + jcol] = h[i];
        }
    }
}

struct HidDesc {
    int nhid, r, nt, mode;
    int hoff[kMaxLayers], boff[kMaxLayers], hrows[kMaxLayers], hcols[kMaxLayers], hact[kMaxLayers];
};

// Hidden layers at z with nt tangent columns (one CTA; net.cpp:159-240).  mode 0
// (decode_jacobian): T_0 = I (r x r), T' = phi'(a) (W T).  mode 1 (second directional):
// columns (p, t, s), T_0 = (u, v, 0), p' = phi'(a) Wp, t' = phi'(a) Wt,
// s' = phi''(a) (Wp)(Wt) + phi'(a) Ws.  Output: y (h) and T (h x nt) in `out`.
__global__ void __launch_bounds__(512) hidden_tangent_kernel(const HidDesc d, const double* Wh, const double* bh,
                                                             const double* z, const double* u, const double* v,
                                                             double* buf0, double* buf1) {
    const int nt = d.nt;
    const int ld = nt + 1;  // row layout: [y | T_0 .. T_{nt-1}]
    double* cur = buf0;
    double* nxt = buf1;
    for (int i = threadIdx.x; i < d.r; i += blockDim.x) {
        cur[(size_t)i * ld] = z[i];
        for (int k = 0; k < nt; ++k) {
            double t0;
            if (d.mode == 0) t0 = (i == k) ? 1.0 : 0.0;
            else t0 = k == 0 ? u[i] : (k == 1 ? v[i] : 0.0);
            cur[(size_t)i * ld + 1 + k] = t0;
        }
    }
    __syncthreads();
    for (int l = 0; l < d.nhid; ++l) {
        const int R = d.hrows[l], K = d.hcols[l], act = d.hact[l];
        const double* W = Wh + d.hoff[l];
        const double* b = bh + d.boff[l];
        for (int i = threadIdx.x; i < R; i += blockDim.x) {
            double acc[1 + kMaxLatent];
            for (int k = 0; k <= nt; ++k) acc[k] = 0.0;
            for (int jj = 0; jj < K; ++jj) {
                const double w = W[(size_t)i * K + jj];
                for (int k = 0; k <= nt; ++k) acc[k] += w * cur[(size_t)jj * ld + k];
            }
            const double a = acc[0] + b[i];
            const double p1 = act_eval(act, a, 1);
            nxt[(size_t)i * ld] = act_eval(act, a, 0);
            if (d.mode == 0) {
                for (int k = 0; k < nt; ++k) nxt[(size_t)i * ld + 1 + k] = p1 * acc[1 + k];
            } else {
                const double p2 = act_eval(act, a, 2);
                nxt[(size_t)i * ld + 1] = p1 * acc[1];
                nxt[(size_t)i * ld + 2] = p1 * acc[2];
                nxt[(size_t)i * ld + 3] = p2 * acc[1] * acc[2] + p1 * acc[3];
            }
        }
        __syncthreads();
        double* tmp = cur;
        cur = nxt;
        nxt = tmp;
    }
    // the caller reads the last layer from buf0 when nhid is even, else from buf1
}

// Output layer: one warp per row i.  a = W_i y + b_i; mode 0: J[i][k] = s_i phi'(a) (W_i T_k);
// mode 1: out_i = s_i [phi''(a) (W_i p)(W_i t) + phi'(a) (W_i s)].
template <typename TS>
__global__ void __launch_bounds__(256) output_tangent_kernel(int n, int hp, int h, int nt, int mode, int out_act,
                                                             const TS* Wout, const double* bout, const double* sout,
                                                             const double* hidT, double* out) {
    const int lane = threadIdx.x & 31;
    const int ld = nt + 1;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
        double acc[1 + kMaxLatent];
        for (int k = 0; k <= nt; ++k) acc[k] = 0.0;
        for (int jj = lane; jj < h; jj += 32) {
            const double w = (double)Wout[(size_t)i * hp + jj];
            for (int k = 0; k <= nt; ++k) acc[k] += w * hidT[(size_t)jj * ld + k];
        }
        for (int k = 0; k <= nt; ++k) acc[k] = warp_sum(acc[k]);
        if (lane == 0) {
            const double a = acc[0] + bout[i];
            const double s = sout[i];
            const double p1 = act_eval(out_act, a, 1);
            if (mode == 0) {
                for (int k = 0; k < nt; ++k) out[(size_t)i * nt + k] = s * p1 * acc[1 + k];
            } else {
                const double p2 = act_eval(out_act, a, 2);
                out[i] = s * (p2 * acc[1] * acc[2] + p1 * acc[3]);
            }
        }
    }
}

int grid_for(int count, int per = 256, int cap = 4 * 148) { return std::max(1, std::min((count + per - 1) / per, cap)); }

template <typename TS>
void assemble_t(Context& c, RefBuffers& b, const double* d_q, double* value, double* grad_host) {
    const HostMesh& m = c.mesh;
    q_to_u_kernel<<<grid_for(c.n), 256, 0, c.stream>>>(c.n, c.d_vfree, d_q, b.xfree, c.d_U);
    asm_elem_kernel<TS><<<kRefGrid, 256, 0, c.stream>>>(m.E, reinterpret_cast<const int4*>(c.d_tets),
                                                        static_cast<const TS*>(c.d_rec), c.d_U,
                                                        reinterpret_cast<const int4*>(c.d_fpos), c.d_forces, b.part,
                                                        grad_host ? 1 : 0);
    sum_partials_kernel<<<1, 256, 0, c.stream>>>(b.part, kRefGrid, b.scal);
    if (grad_host)
        grad_gather_kernel<TS><<<grid_for(m.n_free), 256, 0, c.stream>>>(m.n_free, c.d_csr_ptr, c.d_forces, b.vec2, 1,
                                                                         0, 0);
    cuda_check(cudaGetLastError(), "assemble launch");
    c.launches += grad_host ? 4 : 3;
    c.copy(value, b.scal, 8, cudaMemcpyDeviceToHost, "assemble value");
    if (grad_host) c.copy(grad_host, b.vec2, 8 * (size_t)c.n, cudaMemcpyDeviceToHost, "assemble grad");
}

template <typename TS>
void hessian_apply_t(Context& c, RefBuffers& b, const double* d_q, int k, const double* d_in, double* d_out) {
    const HostMesh& m = c.mesh;
    q_to_u_kernel<<<grid_for(c.n), 256, 0, c.stream>>>(c.n, c.d_vfree, d_q, b.xfree, c.d_U);
    zero_u_kernel<<<grid_for(m.V), 256, 0, c.stream>>>(m.V, b.dU);
    for (int j = 0; j < k; ++j) {
        dir_free_kernel<<<grid_for(c.n), 256, 0, c.stream>>>(c.n, c.d_vfree, d_in, k, j, b.dU);
        hvp_elem_kernel<TS><<<kRefGrid, 256, 0, c.stream>>>(m.E, reinterpret_cast<const int4*>(c.d_tets),
                                                            static_cast<const TS*>(c.d_rec), c.d_U, b.dU,
                                                            reinterpret_cast<const int4*>(c.d_fpos), c.d_forces);
        grad_gather_kernel<TS><<<grid_for(m.n_free), 256, 0, c.stream>>>(m.n_free, c.d_csr_ptr, c.d_forces, d_out, k,
                                                                         j, 1);
    }
    cuda_check(cudaGetLastError(), "hessian apply launch");
    c.launches += 2 + 3LL * k;
}

template <typename TS>
void element_snh_t(Context& c, RefBuffers& b, int count, const int* d_ids, double* d_e, double* d_g, double* d_h) {
    element_snh_kernel<TS><<<grid_for(count, 64), 64, 0, c.stream>>>(
        count, d_ids, reinterpret_cast<const int4*>(c.d_tets), static_cast<const TS*>(c.d_rec), b.dU, d_e, d_g, d_h);
    cuda_check(cudaGetLastError(), "element_snh launch");
    c.launches += 1;
}

template <typename TS>
void decode_tangent_t(Context& c, RefBuffers& b, int mode, const double* d_z, const double* d_u, const double* d_v,
                      double* d_out) {
    HidDesc d{};
    d.nhid = c.nhid;
    d.r = c.r;
    d.mode = mode;
    d.nt = mode == 0 ? c.r : 3;
    for (int l = 0; l < c.nhid; ++l) {
        d.hoff[l] = c.hoff[l];
        d.boff[l] = c.boff[l];
        d.hrows[l] = c.hrows[l];
        d.hcols[l] = c.hcols[l];
        d.hact[l] = c.hact[l];
    }
    const size_t half = (size_t)kMaxHidden * (kMaxLatent + 1);
    double* b0 = b.hid;
    double* b1 = b.hid + half;
    hidden_tangent_kernel<<<1, 512, 0, c.stream>>>(d, c.d_Wh, c.d_bh, d_z, d_u, d_v, b0, b1);
    const double* last = (c.nhid % 2 == 0) ? b0 : b1;
    const int h = c.nhid > 0 ? c.hrows[c.nhid - 1] : c.r;
    output_tangent_kernel<TS><<<std::min((c.n + 7) / 8, 8 * c.num_sms), 256, 0, c.stream>>>(
        c.n, c.hp, h, d.nt, mode, c.out_act, static_cast<const TS*>(c.d_Wout), c.d_bout, c.d_sout, last, d_out);
    cuda_check(cudaGetLastError(), "decode tangent launch");
    c.launches += 2;
}

}  // namespace

void refops_assemble(Context& c, const double* q, double* value, double* grad) {
    RefBuffers& b = bufs(c);
    c.copy(b.vec, q, 8 * (size_t)c.n, cudaMemcpyHostToDevice, "assemble q");
    if (c.precision == LSB_FP64) assemble_t<double>(c, b, b.vec, value, grad);
    else assemble_t<float>(c, b, b.vec, value, grad);
}

void refops_elastic_hessian_apply(Context& c, const double* q, int k, const double* in, double* out) {
    RefBuffers& b = bufs(c);
    const size_t bytes = 8 * (size_t)c.n * k;
    double* d_in = static_cast<double*>(c.dmalloc(bytes));
    double* d_out = static_cast<double*>(c.dmalloc(bytes));
    try {
        c.copy(b.vec, q, 8 * (size_t)c.n, cudaMemcpyHostToDevice, "hessian apply q");
        c.copy(d_in, in, bytes, cudaMemcpyHostToDevice, "hessian apply in");
        c.copy(d_out, out, bytes, cudaMemcpyHostToDevice, "hessian apply out");
        if (c.precision == LSB_FP64) hessian_apply_t<double>(c, b, b.vec, k, d_in, d_out);
        else hessian_apply_t<float>(c, b, b.vec, k, d_in, d_out);
        c.copy(out, d_out, bytes, cudaMemcpyDeviceToHost, "hessian apply result");
    } catch (...) {
        c.dfree(d_in);
        c.dfree(d_out);
        throw;
    }
    c.dfree(d_in);
    c.dfree(d_out);
}

void refops_element_snh(Context& c, int count, const int* ids, const double* positions, double* energy,
                        double* grad, double* hess) {
    RefBuffers& b = bufs(c);
    const HostMesh& m = c.mesh;
    double* d_pos = static_cast<double*>(c.dmalloc(8 * 3 * (size_t)m.V));
    int* d_ids = static_cast<int*>(c.dmalloc(4 * (size_t)count));
    double* d_e = static_cast<double*>(c.dmalloc(8 * (size_t)count));
    double* d_g = static_cast<double*>(c.dmalloc(8 * 12 * (size_t)count));
    double* d_h = hess ? static_cast<double*>(c.dmalloc(8 * 144 * (size_t)count)) : nullptr;
    auto release = [&] {
        c.dfree(d_pos);
        c.dfree(d_ids);
        c.dfree(d_e);
        c.dfree(d_g);
        if (d_h) c.dfree(d_h);
    };
    try {
        c.copy(d_pos, positions, 8 * 3 * (size_t)m.V, cudaMemcpyHostToDevice, "element_snh positions");
        c.copy(d_ids, ids, 4 * (size_t)count, cudaMemcpyHostToDevice, "element_snh ids");
        pos_to_u_kernel<<<grid_for(m.V), 256, 0, c.stream>>>(m.V, d_pos, b.xrest, b.dU);
        if (c.precision == LSB_FP64) element_snh_t<double>(c, b, count, d_ids, d_e, d_g, d_h);
        else element_snh_t<float>(c, b, count, d_ids, d_e, d_g, d_h);
        c.copy(energy, d_e, 8 * (size_t)count, cudaMemcpyDeviceToHost, "element_snh energy");
        c.copy(grad, d_g, 8 * 12 * (size_t)count, cudaMemcpyDeviceToHost, "element_snh grad");
        if (hess) c.copy(hess, d_h, 8 * 144 * (size_t)count, cudaMemcpyDeviceToHost, "element_snh hessian");
    } catch (...) {
        release();
        throw;
    }
    release();
}

void refops_decode_jacobian(Context& c, const double* z, double* J) {
    RefBuffers& b = bufs(c);
    double* d_J = static_cast<double*>(c.dmalloc(8 * (size_t)c.n * c.r));
    try {
        c.copy(b.vec, z, 8 * (size_t)c.r, cudaMemcpyHostToDevice, "jacobian z");
        if (c.precision == LSB_FP64) decode_tangent_t<double>(c, b, 0, b.vec, nullptr, nullptr, d_J);
        else decode_tangent_t<float>(c, b, 0, b.vec, nullptr, nullptr, d_J);
        c.copy(J, d_J, 8 * (size_t)c.n * c.r, cudaMemcpyDeviceToHost, "jacobian");
    } catch (...) {
        c.dfree(d_J);
        throw;
    }
    c.dfree(d_J);
}

void refops_decode_second_directional(Context& c, const double* z, const double* u, const double* v, double* out) {
    RefBuffers& b = bufs(c);
    std::vector<double> zuv(3 * (size_t)c.r);
    std::memcpy(zuv.data(), z, 8 * (size_t)c.r);
    std::memcpy(zuv.data() + c.r, u, 8 * (size_t)c.r);
    std::memcpy(zuv.data() + 2 * c.r, v, 8 * (size_t)c.r);
    c.copy(b.vec, zuv.data(), 8 * zuv.size(), cudaMemcpyHostToDevice, "second directional z u v");
    if (c.precision == LSB_FP64)
        decode_tangent_t<double>(c, b, 1, b.vec, b.vec + c.r, b.vec + 2 * c.r, b.vec2);
    else
        decode_tangent_t<float>(c, b, 1, b.vec, b.vec + c.r, b.vec + 2 * c.r, b.vec2);
    c.copy(out, b.vec2, 8 * (size_t)c.n, cudaMemcpyDeviceToHost, "second directional");
}

}  // namespace lsb
