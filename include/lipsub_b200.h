/*
 * lipsub_b200 — C ABI of the B200-native reduced-objective hot path
 * (arXiv 2409.03807 reduced-order solver; reference: /root/reference/proj).
 *
 * Plain pointers and sizes only; no CUDA, Eigen or torch types.  Every entry
 * point returns an lsb_status; on failure lsb_last_error() (thread-local)
 * holds the message.  The C++ mirror of the reference interface
 * (include/lipsub_b200/lipsub.hpp) re-throws these as the reference's
 * exception types (std::invalid_argument / std::runtime_error).
 *
 * Replaced reference interfaces (paths relative to /root/reference/):
 *   lsb_create            <- PotentialContext + MassMatrix + SubspaceModel construction
 *                            (proj/include/lipsub/energy.hpp:46-60, mesh.hpp:85-92, net.hpp:27-37)
 *   lsb_set_inertia       <- ReducedObjective::qbar / ::dt          (proj/include/lipsub/reduced_solver.hpp:61-68)
 *   lsb_set_pin_positions <- PotentialContext::pin_positions         (proj/include/lipsub/energy.hpp:49)
 *   lsb_eval              <- ReducedObjective::eval, the Objective plug-in
 *                            `double(const VectorXd&, VectorXd* grad)` with a nullable grad
 *                                                                     (proj/include/lipsub/reduced_solver.hpp:51,70; proj/src/reduced_solver.cpp:184-202)
 *   lsb_decode            <- decode                                   (proj/include/lipsub/net.hpp:47; proj/src/net.cpp:146-150)
 *   lsb_lbfgs             <- lbfgs_minimize(ReducedObjective::as_objective(), z, cfg)
 *                                                                     (proj/include/lipsub/reduced_solver.hpp:55; proj/src/reduced_solver.cpp:58-131)
 *   lsb_step              <- reduced_step (L-BFGS method)             (proj/include/lipsub/reduced_solver.hpp:82-84; proj/src/reduced_solver.cpp:235-277)
 *   lsb_simulate          <- the cmd_simulate step loop               (proj/tools/lipsub_cli.cpp:280-297)
 *   lsb_eval_batched      <- a loop of ReducedObjective::eval over z  (no reference batched API)
 *   lsb_hessian_batched   <- reduced_potential_hessian                (proj/include/lipsub/losses.hpp:131-133; proj/src/losses.cpp:301-316)
 *   lsb_set_cubature      <- SolverConfig::runtime_cubature / ReducedObjective::runtime_cubature
 *                            (proj/include/lipsub/reduced_solver.hpp:23,67; ElementSubset energy.hpp:25-36)
 *   lsb_objective_hessian <- ReducedObjective::hessian                (proj/include/lipsub/reduced_solver.hpp:71; proj/src/reduced_solver.cpp:204-229)
 *   lsb_projective_newton <- projective_newton_minimize(obj, hessian) (proj/include/lipsub/reduced_solver.hpp:56-57; proj/src/reduced_solver.cpp:133-182)
 *   lsb_lipschitz_loss    <- lipschitz_loss(model, pairs, 2, pot)     (proj/include/lipsub/losses.hpp:120-122; proj/src/losses.cpp:237-244)
 *   lsb_make_bar_mesh     <- make_bar_3d (6-tet variant)              (proj/include/lipsub/mesh.hpp:76-77; proj/src/mesh.cpp:357-397)
 *   lsb_make_bar_decoder  <- make_mlp_model (Xavier-normal variant)   (proj/include/lipsub/net.hpp:39-41; proj/src/net.cpp:90-123)
 */
#ifndef LIPSUB_B200_H
#define LIPSUB_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LSB_OK = 0,
    LSB_EINVAL = 1,      /* bad shapes / config: reference std::invalid_argument */
    LSB_ENONFINITE = 2,  /* non-finite energy: reference std::runtime_error (reduced_solver.cpp:198-199) */
    LSB_ECUDA = 3,       /* CUDA runtime error or no device */
    LSB_EMESH = 4,       /* degenerate / out-of-range mesh: reference std::runtime_error (mesh.cpp:113-125) */
    LSB_ESTATE = 5       /* call order violated (e.g. step before state) */
} lsb_status;

typedef enum { LSB_FP64 = 0, LSB_FP32 = 1 } lsb_precision;

/* Activation tags (reference net.hpp:13 + ELU). */
typedef enum { LSB_ACT_IDENTITY = 0, LSB_ACT_SILU = 1, LSB_ACT_TANH = 2, LSB_ACT_ELU = 3 } lsb_activation;

/* Exit taxonomy (reference reduced_solver.hpp:28-39). */
typedef enum { LSB_CONVERGED = 1, LSB_SADDLE = 2, LSB_LINESEARCH_CAP = 3, LSB_ITERATION_CAP = 4 } lsb_exit_code;

typedef struct lsb_context lsb_context;

typedef struct {
    int num_vertices;            /* V */
    const double* rest_positions;/* V*3 row-major */
    int num_tets;                /* E */
    const int32_t* tets;         /* E*4 vertex ids, positive orientation */
    int num_pinned;
    const int32_t* pinned;       /* vertex ids (any order, duplicates ignored) */
    const double* mu;            /* E per-tet Lame mu  (reference MaterialParams::mu, per tet) */
    const double* lambda;        /* E per-tet Lame lambda */
    double density;              /* kg/m^3 (lumped mass, mesh.cpp:417-434) */
} lsb_mesh_desc;

typedef struct {
    int latent_dim;              /* r */
    int num_layers;              /* L: hidden layers + output layer */
    const int* rows;             /* L: rows[l] (rows[L-1] == n == 3 * free vertices) */
    const int* cols;             /* L: cols[0] == r, cols[l] == rows[l-1] */
    const int* activations;      /* L: lsb_activation per layer */
    const double* const* weights;/* L: row-major rows x cols */
    const double* const* biases; /* L: rows */
    const double* norm_shift;    /* n */
    const double* norm_scale;    /* n, > 0 */
} lsb_decoder_desc;

typedef struct {                 /* reference SolverConfig (reduced_solver.hpp:16-26) */
    double epsilon;              /* |g|_inf threshold, default 1e-5 */
    int max_iters;               /* default 1024 */
    int max_linesearch;          /* default 128 */
    int lbfgs_history;           /* default 8 */
    double dt;                   /* default 0.05 */
} lsb_solver_config;

typedef struct {                 /* reference ExitReport (reduced_solver.hpp:33-39) + counters */
    int code;                    /* lsb_exit_code */
    int iterations;
    double final_grad_inf_norm;
    double wall_time_ms;         /* device clock (globaltimer) from solve start to exit */
    int value_evals;             /* objective evaluations (energy), incl. line-search trials */
    int grad_evals;              /* of which also produced the gradient */
} lsb_exit_report;

/* ---- errors -------------------------------------------------------------------------- */
const char* lsb_last_error(void);
const char* lsb_version(void);

/* ---- setup helpers (kernel K0, host fp64) ----------------------------------------------- */
/* Sizes of a Kuhn bar mesh; pass NULL arrays to lsb_make_bar_mesh first to query. */
lsb_status lsb_bar_mesh_size(int nx, int ny, int nz, int pin_left, int* V, int* E, int* num_pinned);
lsb_status lsb_make_bar_mesh(int nx, int ny, int nz, double width, double height, double depth,
                             double jitter_frac, uint64_t seed, int pin_left,
                             double* rest_positions, int32_t* tets, int32_t* pinned);
/* Xavier-normal decoder for a mesh: hidden_layers x width (activation act) + linear output
 * of size n = 3 * free vertices.  Weights are written packed: layer l row-major, layers
 * concatenated; biases are zero.  shift = rest free DOFs, scale = out_scale. */
lsb_status lsb_make_bar_decoder(int V, const double* rest_positions, int num_pinned, const int32_t* pinned,
                                int latent_dim, int hidden_layers, int width, int act, uint64_t seed,
                                double out_scale, double* weights_packed, double* norm_shift, double* norm_scale);
/* Per-tet Lame parameters from Young's modulus E in [E_lo, E_hi] (uniform per tet from
 * substream(seed, 2) when E_hi > E_lo, else constant) and Poisson ratio nu. */
lsb_status lsb_lame_from_young(int num_tets, double E_lo, double E_hi, double nu, uint64_t seed,
                               double* mu, double* lambda);

/* std * randn draws from substream(seed, tag) (reference rng.hpp:23-51), in order. */
lsb_status lsb_gaussian_stream(uint64_t seed, uint64_t tag, int count, double std_dev, double* out);

/* ---- context ------------------------------------------------------------------------------ */
lsb_status lsb_create(const lsb_mesh_desc* mesh, const lsb_decoder_desc* decoder, int precision,
                      int device, lsb_context** out);
void lsb_destroy(lsb_context* ctx);
/* n = free DOFs, r = latent dim, h = hidden width of the last hidden layer. */
lsb_status lsb_get_info(const lsb_context* ctx, int* n, int* r, int* V, int* E, int* h, int* precision);
/* Lumped mass per free DOF (n) and total mass over all vertices. */
lsb_status lsb_get_mass(const lsb_context* ctx, double* mass_diag, double* total_mass);

/* Prescribed pin positions (V*3; only pinned rows are read). Default: rest. */
lsb_status lsb_set_pin_positions(lsb_context* ctx, const double* pin_positions);
/* Inertia target qbar (n, absolute free-DOF positions) and dt; qbar == NULL drops the
 * inertia term (quasi-static objective). */
lsb_status lsb_set_inertia(lsb_context* ctx, const double* qbar, double dt);

/* E(z) and optionally grad (r) — ReducedObjective::eval. */
lsb_status lsb_eval(lsb_context* ctx, const double* z, double* value, double* grad /* nullable */);
/* q = decode(z) (n absolute free-DOF positions). */
lsb_status lsb_decode(lsb_context* ctx, const double* z, double* q);
/* Device-resident L-BFGS + Armijo on the current objective; z in/out. */
lsb_status lsb_lbfgs(lsb_context* ctx, double* z, const lsb_solver_config* cfg, lsb_exit_report* report);

/* ---- dynamics (device-resident state) ------------------------------------------------------ */
/* Simulation state: absolute positions and velocities (V*3) and z (r). */
lsb_status lsb_set_state(lsb_context* ctx, const double* positions, const double* velocities, const double* z);
lsb_status lsb_get_state(lsb_context* ctx, double* positions, double* velocities, double* z, double* t);
/* Per-frame external force on free DOFs (n); default zero. */
lsb_status lsb_set_external_force(lsb_context* ctx, const double* force);
/* One implicit-Euler (or quasi-static) reduced step — reduced_step. */
lsb_status lsb_step(lsb_context* ctx, const lsb_solver_config* cfg, int quasi_static, lsb_exit_report* report);
/* `steps` reduced steps launched back to back with no host synchronisation in
 * between; per-step reports (steps) and z after each step (steps*r, nullable). */
lsb_status lsb_simulate(lsb_context* ctx, int steps, const lsb_solver_config* cfg, int quasi_static,
                        lsb_exit_report* reports, double* z_traj);

/* ---- batched / second order ----------------------------------------------------------------- */
/* E and grad for B latent vectors (Z: B*r row-major) of the current objective. */
/* ---- the reference's secondary hot-path primitives, evaluated on the device over the context's
 * resident mesh, per-tet material (the active element set under lsb_set_cubature) and decoder.
 * q is a free-DOF configuration (n, the layout of decode), pinned vertices sit at the context's pin
 * positions (dof_unpack, proj/src/mesh.cpp:448-461).  fp64 arithmetic; element records in the
 * context's storage precision. */
/* assemble(ctx, q) elastic branch (proj/include/lipsub/energy.hpp:99-101; proj/src/energy.cpp:404-437):
 * value = sum_e E_e over all elements (pinned included), grad (nullable) = free-DOF gradient (n). */
lsb_status lsb_assemble(lsb_context* ctx, const double* q, double* value, double* grad /* nullable */);
/* element_snh (proj/include/lipsub/energy.hpp:71-72; proj/src/energy.cpp:280-298) for `count` element ids at
 * full-space positions (V x 3) with each element's own mu, lambda: energy[k], grad[12 k..] (local order
 * vertex-major, k*3+a), hess[144 k..] (12 x 12 row-major, nullable). */
lsb_status lsb_element_snh(lsb_context* ctx, int count, const int* ids, const double* positions, double* energy,
                           double* grad, double* hess /* nullable */);
/* elastic_hessian_apply (proj/include/lipsub/energy.hpp:109-112; proj/src/energy.cpp:481-493):
 * out += H(q) in, in / out n x k row-major. */
lsb_status lsb_elastic_hessian_apply(lsb_context* ctx, const double* q, int k, const double* in, double* out);
/* decode_jacobian (proj/include/lipsub/net.hpp:52-53; proj/src/net.cpp:159-190): J = d decode / dz, n x r row-major. */
lsb_status lsb_decode_jacobian(lsb_context* ctx, const double* z, double* J);
/* decode_second_directional (proj/include/lipsub/net.hpp:57-59; proj/src/net.cpp:192-240): d2 decode / dz2 (u, v). */
lsb_status lsb_decode_second_directional(lsb_context* ctx, const double* z, const double* u, const double* v,
                                         double* out);

lsb_status lsb_eval_batched(lsb_context* ctx, int B, const double* Z, double* E, double* G /* nullable */);
/* Reduced elastic-potential Hessians d2P/dz2 (B*r*r) — reduced_potential_hessian. */
lsb_status lsb_hessian_batched(lsb_context* ctx, int B, const double* Z, double* H);
/* Runtime cubature: the elastic term becomes sum_k weights[k] * E_{ids[k]} (ElementSubset).
 * count == 0 or ids == NULL restores the full element set.  Applies to every evaluation,
 * solve, step, batched and Hessian call of the context; the mass matrix is unchanged. */
lsb_status lsb_set_cubature(lsb_context* ctx, int count, const int* ids, const double* weights);
/* Objective Hessians d2E/dz2 (B*r*r) — ReducedObjective::hessian: the elastic part plus,
 * when lsb_set_inertia set qbar, the M/h^2 block and the inertia residual's decoder curvature. */
lsb_status lsb_objective_hessian(lsb_context* ctx, int B, const double* Z, double* H);
/* Projective-Newton minimisation of the current objective from z (in/out):
 * projective_newton_minimize with the SPD-projected objective Hessian and the
 * Armijo line search; exit codes as lsb_lbfgs (lbfgs_history unused). */
lsb_status lsb_projective_newton(lsb_context* ctx, double* z, const lsb_solver_config* cfg, lsb_exit_report* report);
/* Second-order Lipschitz loss mean_p |H(z1_p) - H(z2_p)|_F^2 / |z1_p - z2_p|^2. */
lsb_status lsb_lipschitz_loss(lsb_context* ctx, int P, const double* Z1, const double* Z2, double* loss);
/* The same loss and its gradient with respect to every decoder parameter: the
 * training-side backward of build_lipschitz_loss(..., order 2, pot) followed by
 * Tape::backward / param_gradient (proj/src/losses.cpp:196-213, proj/src/tape.cpp:46-79,
 * 245-279).  grad holds, per decoder layer in order (hidden layers, then the output
 * layer), W (rows x cols, row-major) then b (rows): sum over layers of rows*(cols+1)
 * doubles.  Requires an identity output layer and r in {8, 16, 32} (as the Hessian path);
 * fp32 device arithmetic, fp64 accumulation; LSB_EINVAL on a coincident pair. */
lsb_status lsb_lipschitz_loss_grad(lsb_context* ctx, int P, const double* Z1, const double* Z2, double* loss,
                                   double* grad);

/* Persistent solve kernel (one cooperative launch of thread-block clusters per
 * evaluation / solve / step).  lsb_get_solve_info reports its grid (0 = not
 * available for this problem, the multi-kernel CUDA-graph path is used) and whether
 * it is in use; lsb_set_solve_kernel(ctx, 0) forces the graph path. */
lsb_status lsb_get_solve_info(const lsb_context* ctx, int* solve_grid, int* in_use);
lsb_status lsb_set_solve_kernel(lsb_context* ctx, int enable);
/* Phase timestamps of the last solve-kernel launch (contexts created with LSB_TRACE=1):
 * pairs (tag, globaltimer ns), count pairs. */
lsb_status lsb_get_trace(const lsb_context* ctx, unsigned long long* out, int cap, int* count);
/* The raw 2048-word trace buffer: [0] pair count, [1..510] pairs; [512 + 256 k + b] for CTA
 * b < 256 (globaltimer ns): k = 0 entry, 1 first grid-barrier arrival, 2 / 3 / 4 end of the first
 * evaluation's output-layer / element / VJP phase. */
lsb_status lsb_get_trace_raw(const lsb_context* ctx, unsigned long long* out);
/* Developer hook (LSB_TRACE=1 at create): per ticket of the last sweep-pass launch
 * {cta << 32 | item code, t_start, t_dependencies_met, t_end} (globaltimer ns); *count = tickets. */
lsb_status lsb_get_sweep_trace(const lsb_context* ctx, unsigned long long* out, int cap, int* count);

/* ---- measurement hooks (bench.py) ------------------------------------------------------------ */
/* Number of kernels this library launched since creation (every launch, graph node
 * executions counted per execution as reported by the device counters). */
lsb_status lsb_get_launch_count(const lsb_context* ctx, long long* launches);
/* Developer switches this context was created with ("NAME=value ..."; empty when none): the
 * LSB_* environment variables are read once, at lsb_create, and never change results except
 * the timing-only LSB_SOLVE_EXP bits, which a production build rejects. */
lsb_status lsb_get_dev_flags(const lsb_context* ctx, char* buf, int cap);
/* Average device duration (ms) of the output-layer forward kernel over the last
 * lsb_profile_eval call, measured with CUDA events on the launching stream. */
lsb_status lsb_profile_eval(lsb_context* ctx, const double* z, int reps, double* ms_out_fwd,
                            double* ms_elem, double* ms_vjp, double* ms_total);

/* K evaluations of the current objective at Z (K*r), each preceded by an L2 flush
 * (write of flush_bytes) outside the timed interval; per evaluation: device time of
 * the whole evaluation and of the output-layer kernel (CUDA events on the context
 * stream), and the energy. */
lsb_status lsb_bench_evals(lsb_context* ctx, int K, const double* Z, size_t flush_bytes, double* eval_ms,
                           double* out_fwd_ms, double* E);
/* lsb_bench_evals with want_grad = 0: value-only evaluations (lsb_eval with grad == NULL). */
lsb_status lsb_bench_evals_ex(lsb_context* ctx, int K, const double* Z, size_t flush_bytes, int want_grad,
                              double* eval_ms, double* out_fwd_ms, double* E);
/* reps calls of lsb_eval_batched (kind 0: B latents Z1 -> E, G) or lsb_lipschitz_loss (kind 1: B pairs
 * Z1, Z2 -> loss), each preceded by an L2 flush and bracketed by CUDA events on the context stream
 * (the bracket includes the call's own small host<->device copies); ms[k] per call. */
lsb_status lsb_bench_batched(lsb_context* ctx, int kind, int B, const double* Z1, const double* Z2, int reps,
                             size_t flush_bytes, double* ms, double* E, double* G, double* loss);
/* K reduced steps from the current state (lsb_set_state), each preceded by an L2
 * flush; per step: device time (CUDA events) and exit report. */
lsb_status lsb_bench_steps(lsb_context* ctx, int K, const lsb_solver_config* cfg, int quasi_static,
                           size_t flush_bytes, double* step_ms, lsb_exit_report* reports);
/* End-to-end through the C ABI: K calls of lsb_eval(ctx, Z + k r, &E[k], G + k r) on host
 * buffers (host z in, host E and grad out, the copies inside every call), timed on the host
 * clock around the loop: *seconds. */
lsb_status lsb_bench_e2e(lsb_context* ctx, int K, const double* Z, double* E, double* G, double* seconds);

#ifdef __cplusplus
}
#endif
#endif /* LIPSUB_B200_H */
