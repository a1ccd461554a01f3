// Persistent "solve" kernel: one cooperative launch (grid of thread-block
// clusters) runs a whole objective evaluation, L-BFGS solve or implicit-Euler
// step, with grid barriers between phases instead of kernel boundaries.
//
//   cluster 0 (the control cluster) keeps the hidden-layer weight slices and the
//   solver state in shared memory for the lifetime of the launch;
//   every CTA owns a TMA ring (producer warp 8) used by the two W_out streams;
//   the Armijo / need-gradient decision is evaluated redundantly by every CTA
//   from the same partials (identical fixed-order sums), so it costs no barrier.
//
// Per evaluation:  out_fwd | grid | elem | grid | [gather | grid | vjp | grid] | ctrl | grid
#pragma once

#include "lsb_stream.cuh"

namespace lsb {

// Launch-wide scalars the non-control CTAs need (written by the control CTA).
struct SolveShared {
    int mode, phase, want_grad, done;
    double f, armijo_slope;  // f + 1e-4 alpha gtd threshold pieces
    int status;
};

struct SolveParams {
    int task;         // 0 = eval (ctrl start + one evaluation), 1 = minimize, 2 = step
    int quasi;        // step: quasi-static
    int want_grad;    // eval: gradient wanted
    int nst;          // ring stages (8 or 16: a multiple of the 8 consumer warps)
    // dynamics
    const double* u_state;
    const double* v_state;
    const double* a_ext;
    double* z_state;
    double* u_state_w;
    double* v_state_w;
    const char* vpinned;
    const double* pin_disp;
    SolveShared* sh;
    long long* launch_acc;
    unsigned long long* trace;  // optional phase timestamps (CTA 0), nullptr = off
};


// ---- control-cluster helpers (weights resident in smem) -------------------------------------------
struct CtrlSmem {
    double* wsl;      // staged W row slices
    double* ybuf;     // kMaxHidden
    double* slice[2]; // 64 each
    double* part[2];  // kMaxHidden each
    double* bsl;      // kMaxLayers * 64
    double* asl;      // kMaxLayers * 64
    DevState* sst;
    int woff[kMaxLayers];
};

template <typename TS, int CS>
__device__ void ctrl_stage(const EvalParams<TS>& p, CtrlSmem& cs, int c, bool with_state) {
    const int tid = threadIdx.x;
    int off = 0;
    for (int l = 0; l < p.nhid; ++l) {
        const int R = p.hrows[l], C = p.hcols[l];
        const int i0 = part_lo(R, CS, c), i1 = part_lo(R, CS, c + 1);
        cs.woff[l] = off;
        stage_doubles(cs.wsl + off, p.Wh + p.hoff[l] + (size_t)i0 * C, (i1 - i0) * C);
        stage_doubles(cs.bsl + l * 64, p.bh + p.boff[l] + i0, i1 - i0);
        off += ((i1 - i0) * C + 1) & ~1;
    }
    if (with_state && c == 0)
        stage_doubles(reinterpret_cast<double*>(cs.sst), reinterpret_cast<const double*>(p.st),
                      (int)(sizeof(DevState) / sizeof(double)));
    cp_async_wait_all();
    (void)tid;
    __syncthreads();
}

// Backward through the hidden layers; ybar of the last hidden layer is the
// fixed-order sum of the per-CTA partials (G x hp).  Result -> sst->gz (CTA 0).
template <typename TS, int CS>
__device__ void ctrl_backward(const EvalParams<TS>& p, CtrlSmem& cs, cg::cluster_group& cluster, int c, int G,
                              const double* ypart) {
    const int tid = threadIdx.x;
    if (p.nhid == 0) {
        if (c == 0)
            for (int j = tid; j < p.r; j += blockDim.x) {
                double s = 0.0;
                for (int b = 0; b < G; ++b) s += __ldcg(ypart + (size_t)b * p.hp + j);
                cs.sst->gz[j] = s;
            }
        __syncthreads();
        return;
    }
    const int Rl = p.hrows[p.nhid - 1];
    {
        // own columns j0..j1 of ybar: threads split (column, partial chunk), fixed combine order
        const int j0 = part_lo(Rl, CS, c), j1 = part_lo(Rl, CS, c + 1);
        const int ncol = j1 - j0;
        const int per = ncol > 0 ? max(1, (int)blockDim.x / ncol) : 1;  // threads per column
        const int chunk = (G + per - 1) / per;
        double* tmp = cs.part[0];  // ncol x per partial sums (<= blockDim.x)
        const int col = tid / per, q = tid % per;
        if (col < ncol) {
            double s = 0.0;
            const int b0 = q * chunk, b1 = min(G, b0 + chunk);
#pragma unroll 4
            for (int b = b0; b < b1; ++b) s += __ldcg(ypart + (size_t)b * p.hp + j0 + col);
            tmp[col * per + q] = s;
        }
        __syncthreads();
        for (int j = tid; j < ncol; j += blockDim.x) {
            double s = 0.0;
            for (int k = 0; k < per; ++k) s += tmp[j * per + k];
            cs.slice[0][j] = s;
        }
    }
    __syncthreads();
    for (int l = p.nhid - 1; l >= 0; --l) {
        const int R = p.hrows[l], C = p.hcols[l];
        const int i0 = part_lo(R, CS, c), i1 = part_lo(R, CS, c + 1);
        double* pt = cs.part[l & 1];
        for (int i = tid; i < i1 - i0; i += blockDim.x)
            cs.slice[0][i] *= act_eval(p.hact[l], cs.asl[l * 64 + i], 1);
        __syncthreads();
        const double* Ws = cs.wsl + cs.woff[l];
        for (int j = tid; j < C; j += blockDim.x) {
            double s = 0.0;
            for (int i = 0; i < i1 - i0; ++i) s = fma(Ws[i * C + j], cs.slice[0][i], s);
            pt[j] = s;
        }
        cluster.sync();
        if (l > 0) {
            const int Rp = p.hrows[l - 1];
            const int k0 = part_lo(Rp, CS, c), k1 = part_lo(Rp, CS, c + 1);
            for (int j = k0 + tid; j < k1; j += blockDim.x) {
                double vals[CS];
#pragma unroll
                for (int q = 0; q < CS; ++q) vals[q] = cluster.map_shared_rank(pt, q)[j];
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < CS; ++q) s += vals[q];
                cs.slice[0][j - k0] = s;
            }
        } else if (c == 0) {
            for (int j = tid; j < C; j += blockDim.x) {
                double vals[CS];
#pragma unroll
                for (int q = 0; q < CS; ++q) vals[q] = cluster.map_shared_rank(pt, q)[j];
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < CS; ++q) s += vals[q];
                cs.sst->gz[j] = s;
            }
        }
        __syncthreads();
    }
}

// Hidden forward at zt (broadcast from CTA 0's state through DSMEM); keeps
// own-row pre-activations in smem (asl) for the next backward; CTA 0 writes y_last.
template <typename TS, int CS>
__device__ void ctrl_forward(const EvalParams<TS>& p, CtrlSmem& cs, cg::cluster_group& cluster, int c) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nw = blockDim.x >> 5;
    const double* zsrc = cluster.map_shared_rank(cs.sst->zt, 0);
    for (int j = tid; j < p.r; j += blockDim.x) cs.ybuf[j] = zsrc[j];
    __syncthreads();
    // layer inputs: ybuf (layer 0) or the previous layer's slices in every CTA (DSMEM)
    for (int l = 0; l < p.nhid; ++l) {
        const int R = p.hrows[l], C = p.hcols[l];
        const int i0 = part_lo(R, CS, c), i1 = part_lo(R, CS, c + 1);
        double* out = cs.slice[l & 1];
        const double* in_prev = cs.slice[(l & 1) ^ 1];
        const double* Ws = cs.wsl + cs.woff[l];
        // operand fetch: lane j's inputs y[j], y[j+32], ... from their owners
        double yin[kMaxHidden / 32];
#pragma unroll
        for (int k = 0; k < kMaxHidden / 32; ++k) {
            const int j = lane + 32 * k;
            double v = 0.0;
            if (j < C) {
                if (l == 0) {
                    v = cs.ybuf[j];
                } else {
                    const int Rp = p.hrows[l - 1];
                    int q = (int)(((long long)j * CS) / Rp);
                    while (q + 1 < CS && part_lo(Rp, CS, q + 1) <= j) ++q;
                    while (part_lo(Rp, CS, q) > j) --q;
                    v = cluster.map_shared_rank(in_prev, q)[j - part_lo(Rp, CS, q)];
                }
            }
            yin[k] = v;
        }
        for (int i = warp; i < i1 - i0; i += nw) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < kMaxHidden / 32; ++k) {
                const int j = lane + 32 * k;
                if (j < C) s = fma(Ws[i * C + j], yin[k], s);
            }
            s = warp_sum(s);
            if (lane == 0) {
                const double a = s + cs.bsl[l * 64 + i];
                cs.asl[l * 64 + i] = a;
                out[i] = act_eval(p.hact[l], a, 0);
            }
        }
        cluster.sync();
    }
    if (p.nhid > 0) {  // gather the last layer for y_last (CTA 0)
        const int l = p.nhid - 1, R = p.hrows[l];
        const double* lastv = cs.slice[l & 1];
        if (c == 0)
            for (int j = tid; j < p.hp; j += blockDim.x) {
                double v = 0.0;
                if (j < R) {
                    int q = (int)(((long long)j * CS) / R);
                    while (q + 1 < CS && part_lo(R, CS, q + 1) <= j) ++q;
                    while (part_lo(R, CS, q) > j) --q;
                    v = cluster.map_shared_rank(lastv, q)[j - part_lo(R, CS, q)];
                }
                p.y_last[j] = v;
            }
    } else if (c == 0) {
        for (int j = tid; j < p.hp; j += blockDim.x) p.y_last[j] = j < p.r ? cs.ybuf[j] : 0.0;
    }
}

// ---- the persistent kernel ---------------------------------------------------------------------------
template <typename TS, int HP, int CS>
__global__ void __launch_bounds__(kStreamThreads, 1) solve_kernel(const EvalParams<TS> p, const SolveParams sp) {
    using C = StreamCfg<TS, HP>;
    extern __shared__ __align__(128) unsigned char smem[];
    cg::grid_group grid = cg::this_grid();
    cg::cluster_group cluster = cg::this_cluster();
    const int G = gridDim.x, cta = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool is_ctrl = cta < CS;  // cluster 0 (clusters are contiguous block ranges)
    const int crank = (int)cluster.block_rank();
    // ---- shared memory carve-up
    unsigned char* ring = smem;
    const int NS = sp.nst;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * C::STAGEB);
    uint64_t* empty = full + NS;
    double* cbase = reinterpret_cast<double*>(empty + NS);
    CtrlSmem cs;
    cs.wsl = cbase;
    cs.ybuf = cbase + p.ctrl_smem_w;
    cs.slice[0] = cs.ybuf + kMaxHidden;
    cs.slice[1] = cs.ybuf + kMaxHidden + 64;
    cs.part[0] = cs.ybuf + kMaxHidden + 128;
    cs.part[1] = cs.ybuf + 2 * kMaxHidden + 128;
    cs.bsl = cs.ybuf + 3 * kMaxHidden + 128;
    cs.asl = cs.bsl + kMaxLayers * 64;
    cs.sst = reinterpret_cast<DevState*>(cs.asl + kMaxLayers * 64);
    __shared__ double red[32];
    __shared__ int s_flag;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_fence_init();
    }
    __syncthreads();
    int ring_i = 0;  // tiles passed through this CTA's ring (producer and consumers agree)
    const int ntiles = (p.n + C::TR - 1) / C::TR;
    const int t0 = (int)(((long long)ntiles * cta) / G);
    const int t1 = (int)(((long long)ntiles * (cta + 1)) / G);
    DevState* st = p.st;
    SolveShared* sh = sp.sh;
    int tr = 0;
    auto stamp = [&](int tag) {
        if (sp.trace && cta == 0 && tid == 0 && tr < 255) {
            sp.trace[1 + 2 * tr] = (unsigned long long)tag;
            sp.trace[2 + 2 * tr] = globaltimer();
            sp.trace[0] = (unsigned long long)(++tr);
        }
    };
    stamp(0);

    // ---- control cluster: stage weights (+ state) once
    if (is_ctrl) ctrl_stage<TS, CS>(p, cs, crank, true);
    stamp(1);

    // ---- step prologue: qbar - X and warm start (all CTAs), reference reduced_step :249-256
    if (sp.task == 2) {
        const double dt = is_ctrl && crank == 0 ? cs.sst->dt : __ldcg(&st->dt);
        for (int i = cta * blockDim.x + tid; i < p.n; i += G * blockDim.x) {
            const int f = i / 3, c = i - 3 * f;
            const size_t vi = (size_t)p.vfree[f] * 3 + c;
            const double ut = sp.quasi ? 0.0 : sp.u_state[vi] + dt * sp.v_state[vi] + (dt * dt) * sp.a_ext[i];
            p.eprow[6 * (size_t)i + 5] = ut;
        }
        if (is_ctrl && crank == 0) {
            for (int i = tid; i < p.r; i += blockDim.x) cs.sst->zt[i] = sp.z_state[i];
            if (tid == 0) {
                cs.sst->has_inertia = sp.quasi ? 0 : 1;
                cs.sst->inv_dt2 = 1.0 / (dt * dt);
                cs.sst->quasi_static = sp.quasi;
            }
        }
    }
    // ---- start: reset solver state, hidden forward at zt
    if (is_ctrl) {
        if (crank == 0 && tid == 0) {
            DevState* s = cs.sst;
            s->mode = sp.task == 0 ? kModeEval : kModeLbfgs;
            s->want_grad = sp.task == 0 ? sp.want_grad : 1;
            s->status = kStOk;
            s->phase = kPhaseInit;
            s->done = 0;
            s->code = 4;
            s->iter = 0;
            s->ls = 0;
            s->hist_n = 0;
            s->hist_head = 0;
            s->value_evals = 0;
            s->grad_evals = 0;
            s->need_grad = 0;
            s->accept = 0;
            s->gnorm = 0.0;
            s->loop_iters = 0;
            s->t_start = globaltimer();
            sh->mode = s->mode;
            sh->phase = s->phase;
            sh->want_grad = s->want_grad;
            sh->done = 0;
            sh->status = kStOk;
            sh->f = 0.0;
            sh->armijo_slope = 0.0;
            st->has_inertia = s->has_inertia;
            st->inv_dt2 = s->inv_dt2;
        }
        cluster.sync();
        ctrl_forward<TS, CS>(p, cs, cluster, crank);
    }
    stamp(2);
    grid.sync();
    stamp(3);

    double inv_dt2 = __ldcg(&st->inv_dt2);
    int has_inertia = __ldcg(&st->has_inertia);
    for (;;) {
        // ================= out_fwd (TMA ring)
        {
            double eacc = 0.0;
            if (warp == 8) {
                if (lane == 0) {
                    const uint64_t pol = l2_policy(p.w_resident), keep = l2_policy(1);
                    for (int t = t0, i = ring_i; t < t1; ++t, ++i) {
                        const int s = i % NS, k = i / NS;
                        if (k > 0) mbar_wait(&empty[s], (k - 1) & 1);
                        const int r0 = t * C::TR, rows = min(C::TR, p.n - r0);
                        unsigned char* stg = ring + (size_t)s * C::STAGEB;
                        mbar_expect_tx(&full[s], rows * C::ROWB + rows * 48);
                        tma_load_1d(stg, p.Wout + (size_t)r0 * HP, rows * C::ROWB, &full[s], pol);
                        tma_load_1d(stg + C::TILEB, p.eprow + (size_t)r0 * 6, rows * 48, &full[s], keep);
                    }
                }
            } else {
                double y[C::NCH][C::V4];
#pragma unroll
                for (int c = 0; c < C::NCH; ++c)
#pragma unroll
                    for (int q = 0; q < C::V4; ++q) y[c][q] = __ldcg(p.y_last + (c * 32 + lane) * C::V4 + q);
                const bool ident = p.out_act == kIdentity;
                for (int t = t0 + warp, i = ring_i + warp; t < t1; t += 8, i += 8) {
                    const int s = i % NS, k = i / NS;
                    mbar_wait(&full[s], k & 1);
                    eacc += fwd_tile<TS, HP>(p, ring + (size_t)s * C::STAGEB, t, y, has_inertia, inv_dt2, ident);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
                }
            }
            __syncwarp();
            ring_i += t1 - t0;
            const double tot = block_sum(eacc, red);
            if (tid == 0) p.e_part_out[cta] = 0.5 * inv_dt2 * tot;
        }
        stamp(10);
        grid.sync();
        stamp(11);
        // ================= element pass
        {
            double eacc = 0.0;
            const int stride = G * blockDim.x;
            for (int e = cta * blockDim.x + tid; e < p.E; e += stride) {
                const int4 t = __ldg(p.tets + e);
                double rc[12];
                load_rec<TS>(p.rec, (size_t)e, rc);
                double u0[3], u1[3], u2[3], u3[3];
                load_u(p.U, t.x, u0);
                load_u(p.U, t.y, u1);
                load_u(p.U, t.z, u2);
                load_u(p.U, t.w, u3);
                double f[12];
                eacc += tet_energy_forces(u0, u1, u2, u3, rc, f);
                store_forces_csr(p.forces, __ldg(p.fpos + e), f);
            }
            const double tot = block_sum(eacc, red);
            if (tid == 0) p.e_part_elem[cta] = tot;
        }
        stamp(20);
        grid.sync();
        stamp(21);
        // ================= energy + decision (every CTA, identical fixed-order sums)
        int need = 0;
        double E = 0.0;
        {
            double s = 0.0;
            for (int b = tid; b < G; b += blockDim.x) s += __ldcg(p.e_part_elem + b);
            const double e_el = block_sum(s, red);
            s = 0.0;
            for (int b = tid; b < G; b += blockDim.x) s += __ldcg(p.e_part_out + b);
            const double e_in = block_sum(s, red);
            E = e_el + (has_inertia ? e_in : 0.0);
            const int phase = __ldcg(&sh->phase), mode = __ldcg(&sh->mode);
            if (phase == kPhaseFinalDecode || !isfinite(E)) need = 0;
            else if (mode == kModeEval) need = __ldcg(&sh->want_grad);
            else if (phase == kPhaseInit) need = 1;
            else need = E <= __ldcg(&sh->f) + __ldcg(&sh->armijo_slope);
        }
        if (need) {
            // ================= gather (4 lanes per vertex, contiguous CSR segments)
            {
                const bool ident = p.out_act == kIdentity;
                const int nthr = G * blockDim.x;
                for (int wb = (cta * blockDim.x + tid) & ~31; wb < 4 * p.n_free; wb += nthr)
                    gather_vertex4(p, (wb + lane) >> 2, has_inertia, ident);
            }
            stamp(30);
            grid.sync();
            stamp(31);
            // ================= vjp (TMA ring)
            {
                double acc[C::NCH][C::V4];
#pragma unroll
                for (int c = 0; c < C::NCH; ++c)
#pragma unroll
                    for (int q = 0; q < C::V4; ++q) acc[c][q] = 0.0;
                if (warp == 8) {
                    if (lane == 0) {
                        const uint64_t pol = l2_policy(p.w_resident), keep = l2_policy(1);
                        for (int t = t0, i = ring_i; t < t1; ++t, ++i) {
                            const int s = i % NS, k = i / NS;
                            if (k > 0) mbar_wait(&empty[s], (k - 1) & 1);
                            const int r0 = t * C::TR, rows = min(C::TR, p.n - r0);
                            const unsigned ub = ((unsigned)rows * 8 + 15) & ~15u;
                            unsigned char* stg = ring + (size_t)s * C::STAGEB;
                            mbar_expect_tx(&full[s], rows * C::ROWB + ub);
                            tma_load_1d(stg, p.Wout + (size_t)r0 * HP, rows * C::ROWB, &full[s], pol);
                            tma_load_1d(stg + C::TILEB, p.tv + r0, ub, &full[s], keep);
                        }
                    }
                } else {
                    for (int t = t0 + warp, i = ring_i + warp; t < t1; t += 8, i += 8) {
                        const int s = i % NS, k = i / NS;
                        mbar_wait(&full[s], k & 1);
                        vjp_tile<TS, HP>(p, ring + (size_t)s * C::STAGEB, t, acc);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[s]);
                    }
                }
                ring_i += t1 - t0;
                // per-warp partials -> this CTA's ybar partial (fixed warp order); the
                // ring is idle now (every issued tile has been consumed)
                __syncwarp();
                double* wred = reinterpret_cast<double*>(ring);  // 8 x HP doubles <= ring bytes
                __syncthreads();
                if (warp < 8) {
#pragma unroll
                    for (int c = 0; c < C::NCH; ++c)
#pragma unroll
                        for (int q = 0; q < C::V4; ++q) wred[warp * HP + (c * 32 + lane) * C::V4 + q] = acc[c][q];
                }
                __syncthreads();
                for (int j = tid; j < HP; j += blockDim.x) {
                    double s = 0.0;
#pragma unroll
                    for (int w = 0; w < 8; ++w) s += wred[w * HP + j];
                    p.ybar_part[(size_t)cta * HP + j] = s;
                }
            }
            stamp(40);
            grid.sync();
            stamp(41);
        }
        // ================= control cluster: gradient, L-BFGS, next hidden forward
        if (is_ctrl) {
            DevState* s = cs.sst;
            if (crank == 0 && tid == 0) {
                s->f_eval = E;
                s->need_grad = need;
                const bool skip = s->phase == kPhaseFinalDecode;
                if (!skip) s->value_evals++;
                if (!skip && !isfinite(E)) s->status = kStNonFinite;
                if (s->mode == kModeLbfgs && s->phase == kPhaseLineSearch && !skip) s->accept = need;
                if (need) s->grad_evals++;
            }
            // pre-activations of the point just evaluated are in asl (own rows)
            cluster.sync();
            if (need) ctrl_backward<TS, CS>(p, cs, cluster, crank, G, p.ybar_part);
            if (crank == 0) {
                if (warp == 0) {
                    int m = 0;
                    if (s->mode == kModeLbfgs) m = lbfgs_control(s, p.r);
                    else if (lane == 0) s->done = 1;
                    if (lane == 0) {
                        s->loop_iters++;
                        if (!m) {
                            s->phase = kPhaseDone;
                            s->t_end = globaltimer();
                        }
                        s_flag = m;
                        sh->done = m ? 0 : 1;
                        sh->phase = s->phase;
                        sh->f = s->f;
                        sh->armijo_slope = 1e-4 * s->alpha * s->gtd;
                        sh->status = s->status;
                    }
                }
                __syncthreads();
            }
            cluster.sync();
            const int more = *cluster.map_shared_rank(&s_flag, 0);
            if (more) ctrl_forward<TS, CS>(p, cs, cluster, crank);
        }
        stamp(50);
        grid.sync();
        stamp(51);
        if (__ldcg(&sh->done)) break;
    }
    // ---- epilogue: publish state; step finalize (reference reduced_step :266-276)
    if (is_ctrl && crank == 0) {
        __syncthreads();
        const int nwords = sizeof(DevState) / 4;
        int* dst = reinterpret_cast<int*>(st);
        const int* src = reinterpret_cast<const int*>(cs.sst);
        for (int k = tid; k < nwords; k += blockDim.x) dst[k] = src[k];
    }
    if (sp.task == 2) {
        grid.sync();
        const double dt = __ldcg(&st->dt);
        for (int v = cta * blockDim.x + tid; v < p.V; v += G * blockDim.x)
            for (int c = 0; c < 3; ++c) {
                const size_t k = (size_t)v * 3 + c;
                const double un = sp.vpinned[v] ? sp.pin_disp[k] : __ldcg(p.U + (size_t)v * 4 + c);
                sp.v_state_w[k] = sp.quasi ? 0.0 : (un - sp.u_state[k]) / dt;
                sp.u_state_w[k] = un;
            }
        if (cta == 0) {
            const int idx = st->step_idx;
            for (int i = tid; i < p.r; i += blockDim.x) {
                sp.z_state[i] = st->x[i];
                if (st->z_traj) st->z_traj[(size_t)idx * p.r + i] = st->x[i];
            }
            if (tid == 0) {
                struct Rep {
                    int code, iterations;
                    double gnorm, ms;
                    int ve, ge;
                };
                Rep* reps = static_cast<Rep*>(st->reports);
                Rep rr;
                rr.code = st->status != kStOk ? -st->status : st->code;
                rr.iterations = st->iter;
                rr.gnorm = st->gnorm;
                rr.ms = (double)(st->t_end - st->t_start) * 1e-6;
                rr.ve = st->value_evals;
                rr.ge = st->grad_evals;
                if (reps) reps[idx] = rr;
                st->step_idx = idx + 1;
                st->t += dt;
            }
        }
    }
    if (cta == 0 && tid == 0 && sp.launch_acc) sp.launch_acc[0] += 0;  // single launch
    cluster.sync();  // keep DSMEM alive until every remote read is done
}

}  // namespace lsb
