// Training-side theta-gradient of the order-2 Lipschitz loss:
// the reverse sweep of build_lipschitz_loss (proj/src/losses.cpp:196-213) through
// tape_reduced_derivative order 2 (:136-146), tape_second_directional (:105-118),
// tape_decode (:56-85) and the potential couplings' backward (proj/src/tape.cpp:245-279),
// batched over PH latent points per chunk.  fp32 storage and arithmetic, fp64 gradient
// accumulation across chunks; every reduction has a fixed order (no atomics).
//
// Per point, with Hbar = dL/dH (symmetric) and ebar_ab = dL/d(g . s_ab):
//   W    = J Hbar                         (n x r)   -- hj-bar of matmul_tn(J, hj)
//   gbar = sum_ab ebar_ab s_ab            (n)       -- g-bar of dot(g, s_ab)
//   Jbar = 2 K W                          (n x r)   -- hj Hbar^T + K hj-bar
//   qbar = T[J, W] + K gbar               (n)       -- third contraction + grad-P VJP
// then the decoder's reverse sweep through [y | G | S] (value, first and second tangents).
#pragma once

#include "lsb_common.cuh"

namespace lsb {
namespace theta {

// ---------------------------------------------------------------- strided split-K SGEMM
// part[z][m][n] = sum_{k in chunk z} A[m*sam + k*sak] * B[k*sbk + n*sbn]  (128 x 128 tiles).
__global__ void __launch_bounds__(256) sgemm_strided_kernel(int M, int N, int K, int kchunk, const float* A,
                                                            long long sam, long long sak, const float* B,
                                                            long long sbk, long long sbn, float* part) {
    __shared__ float As[16][128 + 4];
    __shared__ float Bs[16][128 + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.y * 128, n0 = blockIdx.x * 128;
    const int kb0 = blockIdx.z * kchunk, kb1 = min(K, kb0 + kchunk);
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    for (int k0 = kb0; k0 < kb1; k0 += 16) {
        for (int t = threadIdx.x; t < 16 * 128; t += 256) {
            int kk, mm;
            if (sak == 1) {
                kk = t % 16;
                mm = t / 16;
            } else {
                kk = t / 128;
                mm = t % 128;
            }
            const int m = m0 + mm, k = k0 + kk;
            As[kk][mm] = (m < M && k < kb1) ? A[(long long)m * sam + (long long)k * sak] : 0.f;
            int kb, nn;
            if (sbn == 1) {
                kb = t / 128;
                nn = t % 128;
            } else {
                kb = t % 16;
                nn = t / 16;
            }
            const int n = n0 + nn, k2 = k0 + kb;
            Bs[kb][nn] = (n < N && k2 < kb1) ? B[(long long)k2 * sbk + (long long)n * sbn] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float a[8], b[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    float* out = part + (size_t)blockIdx.z * M * N;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
            if (m < M && n < N) out[(size_t)m * N + n] = acc[i][j];
        }
}

// out[i] = sum_z part[z][i] (fp64, z order); f32 store or f64 accumulate.
__global__ void splitk_out_kernel(long long MN, int nz, const float* part, float* out32, double* acc64) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < MN; i += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int z = 0; z < nz; ++z) s += part[(size_t)z * MN + i];
        if (out32) out32[i] = (float)s;
        if (acc64) acc64[i] += s;
    }
}

// acc[i] += sum_p src[i * ld + p * ps]  (bias gradients; fp64, p order)
__global__ void rowsum_acc_kernel(int rows, int P, long long ld, int ps, const float* src, double* acc) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int p = 0; p < P; ++p) s += src[(size_t)i * ld + (size_t)p * ps];
        acc[i] += s;
    }
}

__device__ __forceinline__ void pair_of(int s, int r, int& a, int& b) {
    a = 0;
    while (s >= r - a) {
        s -= r - a;
        ++a;
    }
    b = a + s;
}

// h-level operands of the backward, per (hidden row j, point p), from the top hidden
// block X_L = [y | G | S] (rows j, point-major column blocks of `cols`):
//   Bt2 [h][P*(r+1)]   : (G Hbar)_c, c < r, then sigma = sum_s ebar_s S_s
//   Bfwd[P*(r+2)][h]   : y, G_c, sigma   (right factor of dL/dW_out)
template <int R>
__global__ void theta_prep_kernel(int h, int P, int cols, const float* X, const float* Hbar, const float* ebar,
                                  float* Bt2, float* Bfwd) {
    constexpr int NP = R * (R + 1) / 2;
    const int total = h * P;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int j = idx / P, p = idx % P;
        const float* x = X + ((size_t)j * P + p) * cols;
        const float* Hb = Hbar + (size_t)p * R * R;
        float g[R];
#pragma unroll
        for (int d = 0; d < R; ++d) g[d] = x[1 + d];
        float* bt = Bt2 + (size_t)j * P * (R + 1) + (size_t)p * (R + 1);
#pragma unroll 4
        for (int c = 0; c < R; ++c) {
            float s = 0.f;
#pragma unroll
            for (int d = 0; d < R; ++d) s = fmaf(g[d], Hb[d * R + c], s);
            bt[c] = s;
        }
        const float* eb = ebar + (size_t)p * NP;
        float sg = 0.f;
        for (int s = 0; s < NP; ++s) sg = fmaf(eb[s], x[1 + R + s], sg);
        bt[R] = sg;
        const size_t r0 = (size_t)p * (R + 2);
        Bfwd[r0 * h + j] = x[0];
#pragma unroll
        for (int d = 0; d < R; ++d) Bfwd[(r0 + 1 + d) * h + j] = g[d];
        Bfwd[(r0 + 1 + R) * h + j] = sg;
    }
}

// C2 [n][P*(r+1)] = W_out Bt2 -> Wv[vc][P][r] = s (J Hbar), Gb[vc][P] = s (W_out sigma)
// (pinned vertex rows stay zero).
__global__ void theta_out_kernel(int n, int P, int r, const float* C2, const double* eprow, float* Wv, float* Gb) {
    const int w = r + 1;
    const int total = n * P;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int row = idx / P, p = idx % P;
        const double* e6 = eprow + (size_t)row * 6;
        const float* c = C2 + (size_t)row * P * w + (size_t)p * w;
        const int slot = (int)e6[4];
        const size_t vc = (size_t)(slot >> 2) * 3 + (slot & 3);
        const float s = (float)e6[1];
        float* wo = Wv + (vc * P + p) * r;
        if ((r & 3) == 0) {  // 16-byte stores (rows of r floats are 16-byte aligned)
            for (int a = 0; a < r; a += 4)
                *reinterpret_cast<float4*>(wo + a) = make_float4(s * c[a], s * c[a + 1], s * c[a + 2], s * c[a + 3]);
        } else {
            for (int a = 0; a < r; ++a) wo[a] = s * c[a];
        }
        Gb[vc * P + p] = s * c[r];
    }
}

// column c of the bilinear cofactor: out[:, c] = x_{c+1} x y_{c+2} + y_{c+1} x x_{c+2}
// (row-major 3x3).  bilin_cof(F, X) = dcof(F)[X] = KJ X; bilin_cof(X, Y) = D^3 det[X, Y, .].
__device__ __forceinline__ void bilin_cof(const float* x, const float* y, float* o) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int ci = (c + 1) % 3, cj = (c + 2) % 3;
        const float a1[3] = {x[ci], x[3 + ci], x[6 + ci]}, a2[3] = {x[cj], x[3 + cj], x[6 + cj]};
        const float d1[3] = {y[ci], y[3 + ci], y[6 + ci]}, d2[3] = {y[cj], y[3 + cj], y[6 + cj]};
        o[0 * 3 + c] = d1[1] * a2[2] - d1[2] * a2[1] + a1[1] * d2[2] - a1[2] * d2[1];
        o[1 * 3 + c] = d1[2] * a2[0] - d1[0] * a2[2] + a1[2] * d2[0] - a1[0] * d2[2];
        o[2 * 3 + c] = d1[0] * a2[1] - d1[1] * a2[0] + a1[0] * d2[1] - a1[1] * d2[0];
    }
}

// X (3x3 row-major) = [u1 - u0, u2 - u0, u3 - u0] Dm^-1 from 4 corners x 3 components.
__device__ __forceinline__ void grad_of(const float* u /*[corner*3 + comp]*/, const float* rc, float* X) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c2 = 0; c2 < 3; ++c2)
            X[a * 3 + c2] = (u[3 + a] - u[a]) * rc[c2] + (u[6 + a] - u[a]) * rc[3 + c2] + (u[9 + a] - u[a]) * rc[6 + c2];
}

__device__ __forceinline__ float ddot9(const float* a, const float* b) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 9; ++k) s = fmaf(a[k], b[k], s);
    return s;
}

// Element pass of the backward.  CTA = (block of tets, GP = 128 / R points); thread
// (point pl, direction c).  Tets go in batches of R: first thread (pl, t) forms, once per
// (tet, point), F, cof(F), the SNH derivatives and the gbar HVP's local forces
// (potential_gradient backward) into shared memory; then, per tet of the batch, lane c
// forms dF of J_c and W_c and
//   * the HVP of W_c -> local forces, accumulated as Jbar (x 2) in the block's slot
//     accumulators (column c owned by this thread: race-free, tet order);
//   * its share V_c of the third-contraction vector (snh_third_contraction,
//     energy.cpp:303-320, is linear in M = sym(A B^T) / 2, so it splits over columns);
//     V = sum_c V_c by an xor butterfly over the point's lanes (identical on every lane),
//     and lanes own local dofs d = c, c + R, ... (< 12) of vol B^T V + the gbar forces.
template <int R>
__global__ void __launch_bounds__(128) elem_theta_kernel(const int4* tets, const float* rec, const int* blk_tet0,
                                                        const int* blk_vptr, const short* tet_loc,
                                                        const int* blk_aptr, const int* blk_avert,
                                                        const short* tet_aloc, const float* U, const float* Jv,
                                                        const float* Wv, const float* Gb, int P, float* partJ,
                                                        float* partq) {
    constexpr int GP = 128 / R;
    constexpr int TBMAX = 48;
    constexpr int NB = 34;  // per (tet, point) batch record: F 9, cof 9, psiI, psiII, psiIII, psiJ, gbar forces 12
    __shared__ __align__(16) float sh_rec[TBMAX][12];
    __shared__ short sh_loc[TBMAX][8];
    __shared__ int4 sh_tq[TBMAX];  // the block's vertex ids (the one-tet-ahead J / W prefetch)
    __shared__ float sh_b[R][GP][NB];
    extern __shared__ __align__(16) float dyn[];
    const int tid = threadIdx.x;
    const int pl = tid / R, c = tid % R;
    const int p0 = blockIdx.y * GP;
    const int blk = blockIdx.x;
    const int e0 = blk_tet0[blk], e1 = blk_tet0[blk + 1];
    const int v0 = blk_vptr[blk], nv = blk_vptr[blk + 1] - v0;
    const int a0 = blk_aptr[blk], nva = blk_aptr[blk + 1] - a0;
    float* Us = dyn;                                  // [nva][3][GP]
    float* accJ = Us + (size_t)nva * 3 * GP;          // [nv*3][GP][R]
    float* accq = accJ + (size_t)nv * 3 * GP * R;     // [nv*3][GP]
    for (int i = tid; i < nva * 3 * (GP / 4); i += 128) {
        const int vcl = i / (GP / 4), k4 = i % (GP / 4);
        const int va = __ldg(blk_avert + a0 + vcl / 3), cc = vcl % 3;
        cp_async16(Us + (size_t)vcl * GP + 4 * k4, U + ((size_t)va * 3 + cc) * P + p0 + 4 * k4);
    }
    for (int i = tid; i < nv * 3 * GP * R; i += 128) accJ[i] = 0.f;
    for (int i = tid; i < nv * 3 * GP; i += 128) accq[i] = 0.f;
    for (int i = tid; i < (e1 - e0) * 12; i += 128) sh_rec[i / 12][i % 12] = rec[(size_t)e0 * 12 + i];
    for (int i = tid; i < (e1 - e0) * 4; i += 128) {
        sh_loc[i >> 2][i & 3] = tet_loc[(size_t)e0 * 4 + i];
        sh_loc[i >> 2][4 + (i & 3)] = tet_aloc[(size_t)e0 * 4 + i];
    }
    for (int i = tid; i < e1 - e0; i += 128) sh_tq[i] = __ldg(tets + e0 + i);
    cp_async_wait_all();
    __syncthreads();
    __syncthreads();
    const bool live = p0 + pl < P;
    const float* Jp = Jv + (size_t)(p0 + pl) * R + c;
    const float* Wp = Wv + (size_t)(p0 + pl) * R + c;
    const size_t jstride = (size_t)P * R;
    float jn[12], wn[12];
    if (live && e0 < e1) {
        const int4 t = __ldg(tets + e0);
        const int vv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const size_t row = (size_t)vv[k] * 3 + a;
                jn[k * 3 + a] = __ldg(Jp + row * jstride);
                wn[k * 3 + a] = __ldg(Wp + row * jstride);
            }
    }
    for (int eb = e0; eb < e1; eb += R) {
        // ---- batch phase: thread (pl, t = c) handles tet eb + c for point pl
        {
            const int e = eb + c;
            if (live && e < e1) {
                float rc[12], uu[12], gu[12];
#pragma unroll
                for (int qq = 0; qq < 12; ++qq) rc[qq] = sh_rec[e - e0][qq];
                const int4 tt = __ldg(tets + e);
                const int vv[4] = {tt.x, tt.y, tt.z, tt.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int la = sh_loc[e - e0][4 + k];
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        uu[k * 3 + a] = Us[(la * 3 + a) * GP + pl];
                        gu[k * 3 + a] = __ldg(Gb + ((size_t)vv[k] * 3 + a) * P + p0 + pl);
                    }
                }
                // F, cof(F), SNH derivatives (snh_core, energy.cpp:199-221)
                float A[9], F[9], cof[9];
                grad_of(uu, rc, A);
#pragma unroll
                for (int k = 0; k < 9; ++k) F[k] = A[k] + ((k % 4) == 0 ? 1.f : 0.f);
                bilin_cof(F, F, cof);
#pragma unroll
                for (int k = 0; k < 9; ++k) cof[k] *= 0.5f;
                const float vol = rc[9], mu = rc[10], lam = rc[11];
                const float trA = A[0] + A[4] + A[8];
                float qA = 0.f;
#pragma unroll
                for (int k = 0; k < 9; ++k) qA = fmaf(A[k], A[k], qA);
                const float m2 = A[0] * A[4] - A[1] * A[3] + A[0] * A[8] - A[2] * A[6] + A[4] * A[8] - A[5] * A[7];
                const float detA = A[0] * (A[4] * A[8] - A[7] * A[5]) - A[3] * (A[1] * A[8] - A[7] * A[2]) +
                                   A[6] * (A[1] * A[5] - A[4] * A[2]);
                const float jm1 = trA + m2 + detA;
                const float uI = 4.f + 2.f * trA + qA;
                const float iu = 1.f / uI;
                const float psiI = 0.5f * mu * (1.f - iu);
                const float psiII = 0.5f * mu * iu * iu;
                const float psiIII = -mu * iu * iu * iu;
                const float psiJ = lam * jm1 - 0.75f * mu;
                // gbar HVP -> local forces vol B^T (H gbar)
                float dG[9], dcG[9], Mg[9];
                grad_of(gu, rc, dG);
                bilin_cof(F, dG, dcG);
                const float t1 = 2.f * ddot9(F, dG), t2 = ddot9(cof, dG);
#pragma unroll
                for (int k = 0; k < 9; ++k)
                    Mg[k] = vol * (2.f * psiI * dG[k] + psiII * t1 * 2.f * F[k] + lam * t2 * cof[k] + psiJ * dcG[k]);
                float* o = sh_b[c][pl];
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    o[k] = F[k];
                    o[9 + k] = cof[k];
                }
                o[18] = psiI;
                o[19] = psiII;
                o[20] = psiIII;
                o[21] = psiJ;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    float h0 = 0.f;
#pragma unroll
                    for (int k = 1; k < 4; ++k) {
                        const float hk = Mg[a * 3] * rc[(k - 1) * 3] + Mg[a * 3 + 1] * rc[(k - 1) * 3 + 1] +
                                         Mg[a * 3 + 2] * rc[(k - 1) * 3 + 2];
                        h0 -= hk;
                        o[22 + k * 3 + a] = hk;
                    }
                    o[22 + a] = h0;
                }
            }
        }
        __syncthreads();
        const int nb = min(R, e1 - eb);
        for (int tb = 0; tb < nb; ++tb) {
            const int e = eb + tb;
            float V[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) V[k] = 0.f;
            float rc[12];
#pragma unroll
            for (int qq = 0; qq < 12; ++qq) rc[qq] = sh_rec[e - e0][qq];
            const float* bq = sh_b[tb][pl];
            if (live) {
                float ju[12], wu[12];
#pragma unroll
                for (int q = 0; q < 12; ++q) {
                    ju[q] = jn[q];
                    wu[q] = wn[q];
                }
                if (e + 1 < e1) {
                    const int4 t = sh_tq[e + 1 - e0];
                    const int vv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            const size_t row = (size_t)vv[k] * 3 + a;
                            jn[k * 3 + a] = __ldg(Jp + row * jstride);
                            wn[k * 3 + a] = __ldg(Wp + row * jstride);
                        }
                }
                float F[9], cof[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    F[k] = bq[k];
                    cof[k] = bq[9 + k];
                }
                const float psiI = bq[18], psiII = bq[19], psiIII = bq[20], psiJ = bq[21];
                const float vol = rc[9], lam = rc[11];
                // ---- HVP of W_c:  M = 2 psiI dW + psiII (gI.dW) gI + lam (gJ.dW) gJ + psiJ KJ dW
                float dW[9], dcW[9];
                grad_of(wu, rc, dW);
                bilin_cof(F, dW, dcW);
                const float s1 = 2.f * ddot9(F, dW), s2 = ddot9(cof, dW);
                {
                    float M[9];
#pragma unroll
                    for (int k = 0; k < 9; ++k)
                        M[k] = vol * (2.f * psiI * dW[k] + psiII * s1 * 2.f * F[k] + lam * s2 * cof[k] + psiJ * dcW[k]);
                    // local forces B^T M, x 2 (Jbar = hj Hbar^T + K hj-bar = 2 K W)
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        float h0 = 0.f;
#pragma unroll
                        for (int k = 1; k < 4; ++k) {
                            const float hk = 2.f * (M[a * 3] * rc[(k - 1) * 3] + M[a * 3 + 1] * rc[(k - 1) * 3 + 1] +
                                                    M[a * 3 + 2] * rc[(k - 1) * 3 + 2]);
                            h0 -= hk;
                            const int lv = sh_loc[e - e0][k];
                            if (lv >= 0) accJ[((size_t)(lv * 3 + a) * GP + pl) * R + c] += hk;
                        }
                        const int lv0 = sh_loc[e - e0][0];
                        if (lv0 >= 0) accJ[((size_t)(lv0 * 3 + a) * GP + pl) * R + c] += h0;
                    }
                }
                // ---- third contraction share of column c (A = J_c, B = W_c)
                float dA[9], tmp[9], x[9];
                grad_of(ju, rc, dA);
                const float aI = 2.f * ddot9(F, dA), aJ = ddot9(cof, dA);
                const float trM = ddot9(dA, dW), kJM = ddot9(dA, dcW), qII = aI * s1;
                const float cI = 2.f * (psiIII * qII + 2.f * psiII * trM);  // coefficient of F (gI = 2F)
                // lam s2 KJ dA + psiJ j_third(dA, dW) = bilin_cof(dA, lam s2 F + psiJ dW)
#pragma unroll
                for (int k = 0; k < 9; ++k) x[k] = lam * s2 * F[k] + psiJ * dW[k];
                bilin_cof(dA, x, tmp);
#pragma unroll
                for (int k = 0; k < 9; ++k)
                    V[k] = cI * F[k] + 2.f * psiII * (dA[k] * s1 + dW[k] * aI) + lam * (dcW[k] * aJ + kJM * cof[k]) +
                           tmp[k];
            }
            // V = sum over the point's R lanes (xor butterfly: identical on every lane)
#pragma unroll
            for (int off = R / 2; off >= 1; off >>= 1)
#pragma unroll
                for (int k = 0; k < 9; ++k) V[k] += __shfl_xor_sync(0xffffffffu, V[k], off);
            if (live) {
                // local dofs d = c, c + R, ... (< 12) = (corner d / 3, component d % 3) of vol B^T V
#pragma unroll
                for (int d0 = 0; d0 < 12; d0 += R) {
                    const int d = d0 + c;
                    if (d < 12) {
                        float hv = 0.f;
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            float h0 = 0.f;
#pragma unroll
                            for (int k = 1; k < 4; ++k) {
                                const float hk = V[a * 3] * rc[(k - 1) * 3] + V[a * 3 + 1] * rc[(k - 1) * 3 + 1] +
                                                 V[a * 3 + 2] * rc[(k - 1) * 3 + 2];
                                h0 -= hk;
                                if (d == k * 3 + a) hv = hk;
                            }
                            if (d == a) hv = h0;
                        }
                        const int lv = sh_loc[e - e0][d / 3];
                        if (lv >= 0) accq[(lv * 3 + d % 3) * GP + pl] += rc[9] * hv + bq[22 + d];
                    }
                }
            }
            __syncwarp();  // accq slots are revisited by other lanes of this point at the next tet
        }
        __syncthreads();  // sh_b is rewritten by the next batch
    }
    for (int i = tid; i < nv * 3 * GP * R; i += 128) {
        const int cc = i % R, pp = (i / R) % GP, row = i / (R * GP);
        if (p0 + pp < P) partJ[(((size_t)(v0 * 3) + row) * P + p0 + pp) * R + cc] = accJ[i];
    }
    for (int i = tid; i < nv * 3 * GP; i += 128) {
        const int pp = i % GP;
        if (p0 + pp < P) partq[((size_t)(v0 * 3) + i / GP) * P + p0 + pp] = accq[i];
    }
}

// Abar[row][p*(r+2) + {0, 1+c, r+1}] = s * {qbar, Jbar_c, g}: qbar, Jbar summed over the
// free vertex's block partials in block order (fp64); g column = T (= s * g) as given.
__global__ void theta_combine_kernel(int n, int P, int r, const int* vslot_ptr, const int* vslot,
                                     const float* partJ, const float* partq, const double* eprow, const float* Th,
                                     float* Abar) {
    const int w = r + 2;
    const size_t total = (size_t)n * P;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const int row = (int)(idx / P), p = (int)(idx % P);
        const int f = row / 3, cc = row - 3 * f;
        const float s = (float)eprow[(size_t)row * 6 + 1];
        float* o = Abar + (size_t)row * P * w + (size_t)p * w;
        const int kb = __ldg(vslot_ptr + f), ke = __ldg(vslot_ptr + f + 1);
        double q = 0.0;
        for (int k = kb; k < ke; ++k) q += partq[((size_t)__ldg(vslot + k) * 3 + cc) * P + p];
        o[0] = s * (float)q;
        if (r == 16) {
            // the 16 direction entries of one (slot, row, point) are 64 contiguous bytes: four
            // 16-byte loads per slot; per-direction sums keep the slot order
            double jb[16];
#pragma unroll
            for (int a = 0; a < 16; ++a) jb[a] = 0.0;
            for (int k = kb; k < ke; ++k) {
                const float4* src = reinterpret_cast<const float4*>(partJ + (((size_t)__ldg(vslot + k) * 3 + cc) * P + p) * 16);
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const float4 x = __ldg(src + v);
                    jb[4 * v] += x.x;
                    jb[4 * v + 1] += x.y;
                    jb[4 * v + 2] += x.z;
                    jb[4 * v + 3] += x.w;
                }
            }
#pragma unroll
            for (int a = 0; a < 16; ++a) o[1 + a] = s * (float)jb[a];
        } else {
            for (int a = 0; a < r; ++a) {
                double jb = 0.0;
                for (int k = kb; k < ke; ++k) jb += partJ[(((size_t)vslot[k] * 3 + cc) * P + p) * r + a];
                o[1 + a] = s * (float)jb;
            }
        }
        o[1 + r] = Th[(size_t)row * P + p];
    }
}

// Adjoint of the top hidden block [y | G | S] (h x P x cols) from Xb = W_out^T Abar
// ([h][P*(r+2)]: ybar, Gbar_c, rho = W_out^T (s g)) and S-bar_s = ebar_s rho.
template <int R>
__global__ void theta_top_kernel(int h, int P, int cols, const float* Xb, const float* ebar, float* Xbar) {
    constexpr int NP = R * (R + 1) / 2;
    const size_t total = (size_t)h * P * cols;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx % cols);
        const size_t ip = idx / cols;
        const int i = (int)(ip / P), p = (int)(ip % P);
        const float* x = Xb + (size_t)i * P * (R + 2) + (size_t)p * (R + 2);
        Xbar[idx] = j <= R ? x[j] : ebar[(size_t)p * NP + (j - 1 - R)] * x[R + 1];
    }
}

// Reverse of tangent_act_kernel (losses.cpp:66-79 and :111-116) for one hidden layer: from
// the pre-activation block Q = W X ([q | adot_c | ahat_s], a = q + b) and the output
// adjoint Xbar = [ybar | Gbar_c | Sbar_s], the pre-activation adjoint
//   abar   = phi' ybar + phi'' sum_c adot_c Gbar_c + sum_s Sbar_s (phi''' adot_a adot_b + phi'' ahat_s)
//   adbar_c = phi' Gbar_c + phi'' sum_{s = (a,b)} Sbar_s (d_ac adot_b + d_bc adot_a)
//   ahbar_s = phi' Sbar_s
template <int R>
__global__ void tangent_act_bwd_kernel(int rows, int P, int cols, const float* Q, const double* bias, int act,
                                       const float* Xbar, float* Abar) {
    const int total = rows * P;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int i = idx / P;
        const float* q = Q + (size_t)idx * cols;
        const float* xb = Xbar + (size_t)idx * cols;
        float* ab = Abar + (size_t)idx * cols;
        const double a = (double)q[0] + bias[i];
        const float d1 = (float)act_eval(act, a, 1), d2 = (float)act_eval(act, a, 2), d3 = (float)act_eval(act, a, 3);
        float ad[R], adb[R];
        float abar = d1 * xb[0];
#pragma unroll
        for (int cc = 0; cc < R; ++cc) {
            ad[cc] = q[1 + cc];
            adb[cc] = d1 * xb[1 + cc];
            abar = fmaf(d2 * ad[cc], xb[1 + cc], abar);
        }
        int s = 0;
#pragma unroll 1
        for (int ca = 0; ca < R; ++ca)
#pragma unroll 1
            for (int cb = ca; cb < R; ++cb, ++s) {
                const float sb = xb[1 + R + s];
                abar = fmaf(sb, d3 * ad[ca] * ad[cb] + d2 * q[1 + R + s], abar);
                ab[1 + R + s] = d1 * sb;
                adb[ca] = fmaf(d2 * sb, ad[cb], adb[ca]);
                adb[cb] = fmaf(d2 * sb, ad[ca], adb[cb]);
            }
        ab[0] = abar;
#pragma unroll
        for (int cc = 0; cc < R; ++cc) ab[1 + cc] = adb[cc];
    }
}

}  // namespace theta
}  // namespace lsb
