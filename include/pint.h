/*
 * pint.h — C ABI of libpint: one alpha-circulant preconditioned Richardson iteration
 * ("Paralpha", arXiv 2103.12571) on the all-at-once Radau IIA collocation system,
 * computed by hand-written sm_100a CUDA kernels.
 *
 * Citations: "P:n" = PAPER.md line n (LaTeX source of arXiv 2103.12571).
 *
 * Problem statement: u_t = A u + b on [0, T], u(0) = u0, b == 0 (b != 0:
 * pint_set_forcing),
 * L equal steps dT = T/L, M right-included Gauss-Radau (Radau IIA) nodes.
 * The all-at-once system is C u = w with (block matrix P:115-135)
 *     C = I_L (x) (I_MN - dT Q (x) A) + E (x) (H_M (x) I_N),  E = -1 on the sub-diagonal,
 *     w = (u0 replicated over the M nodes, 0, ..., 0).
 * One iteration with parameter alpha (correction form, reading R1):
 *     u <- u + C_alpha^{-1} (w - C u),   C_alpha = C with -alpha in the (1, L) corner of E.
 * computed as (north star steps (i)-(v), Alg. 1):
 *   (i)   r = w - C u, scaled by alpha^{l/L}               (J^{-1})
 *   (ii)  L-point DFT along time                              (Lemma P:164-171)
 *   (iii) x1_k = S_k^{-1} x_k, Q G_k^{-1} = S_k D_k S_k^{-1}
 *   (iv)  (I - d_km dT A) x2 = x1 for every (k, m)
 *   (v)   y_k = G_k^{-1} S_k x2_k, inverse DFT, alpha^{-l/L}/L, u += c
 *
 * Spatial operators (periodic [0,1)^dim, x_j = j/nx, n = y*nx + x; 2-D sums the axes):
 *   PINT_OP_HEAT:       A = nu * Laplacian  ((u_{j-1} - 2u_j + u_{j+1}) nx^2 per axis)
 *   PINT_OP_ADVECTION:  A = -(cx d/dx + cy d/dy)  (-c n/2 (u_{j+1} - u_{j-1}) per axis)
 * and the paper's other discretisations (Tables 1-2; reading R14):
 *   PINT_OP_HEAT4/6:    nu * centred second differences of order 4 / 6 (5- / 7-point)
 *   PINT_OP_UPWIND1/3/5: -(cx d/dx + cy d/dy) by upwind-biased first differences of order 1/3/5
 *                        (offsets -(k+1)/2 .. (k-1)/2 for c > 0, mirrored per axis for c < 0)
 *   PINT_OP_UPWIND2/4:   the same with order 2 / 4 (Table 1), offsets -(k/2+1) .. k/2-1
 *                        (reading R16: one point more upwind than downwind)
 * 1-D solves (I - s A) by PCR on the tridiagonal factors of I - s A (the 3-point operators are
 * one factor; wider stencils are factored on the host per (alpha, k, m); pint_set_alpha_schedule
 * fails with PINT_ERR_NUMERIC if a factor cannot be formed).  2-D solves are diagonal in Fourier.
 *
 * Data layout: complex128, interleaved (re, im) doubles, u[l][m][n], n fastest (the real-data
 * mode of pint_set_hermitian stores u as real fp64 u[l][m][n] in the same buffer instead).
 *
 * Ownership: the caller owns all device memory (u_dev, work_dev); the context keeps
 * non-owning pointers and carves its small tables out of work_dev.  Host inputs are copied
 * at call time.  Outputs go to caller buffers.
 *
 * Concurrency: a context is not thread-safe.  All device work is stream-ordered on
 * pint_dist.stream.  pint_iterate only enqueues work (CUDA-graph capturable when
 * last_step_diff_inf == NULL); pint_residual_norm / pint_get_* synchronise the stream.
 *
 * Errors: every function returns pint_status (never throws across the ABI); the message of
 * the last non-OK status of the calling thread is pint_last_error().  After PINT_ERR_CUDA
 * the context is poisoned and every later call returns PINT_ERR_STATE.
 */
#ifndef PINT_H
#define PINT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PINT_ABI_VERSION 1
#define PINT_MAX_M 8            /* Radau IIA nodes supported */
#define PINT_MAX_SCHEDULE 64    /* alpha values per pint_set_alpha_schedule */

typedef struct pint_ctx pint_ctx;

typedef enum {
  PINT_OK = 0,
  PINT_ERR_INVALID = 1,             /* bad argument / unsupported size; nothing was changed   */
  PINT_ERR_SCHEDULE = 2,            /* alpha outside (0,1), schedule exhausted, m_k < 4 gamma */
  PINT_ERR_NOT_DIAGONALIZABLE = 3,  /* cond(S_k) > 1e8 or eigenvalue gap < 1e-8 rho(B_k)     */
  PINT_ERR_NUMERIC = 4,             /* non-finite u0, residual norm or last-step difference     */
  PINT_ERR_CUDA = 5,                /* CUDA runtime error (context poisoned)                   */
  PINT_ERR_NCCL = 6,                /* communication error, also an asynchronous one found while
                                       waiting on the stream (communicator aborted, context poisoned) */
  PINT_ERR_STATE = 7                /* context poisoned by an earlier CUDA/NCCL error          */
} pint_status;

typedef enum {
  PINT_OP_HEAT = 0,
  PINT_OP_ADVECTION = 1,
  PINT_OP_HEAT4 = 2,
  PINT_OP_HEAT6 = 3,
  PINT_OP_UPWIND1 = 4,
  PINT_OP_UPWIND3 = 5,
  PINT_OP_UPWIND5 = 6,
  PINT_OP_UPWIND2 = 7,
  PINT_OP_UPWIND4 = 8
} pint_op;

typedef struct {
  int32_t dim;     /* 1 or 2                                                                  */
  int32_t nx, ny;  /* grid, >= 4 per axis (ny == 1 if dim == 1): powers of two (every BASELINE
                      config; 1-D nx <= 2^20, 2-D <= 4096), or 7-smooth sizes 2^a 3^b 5^c 7^d <= 4096
                      (the paper's Table 1/2 grids) on the generic-grid path: one rank,
                      correction form, no Hermitian mode (generic.cu: mixed-radix FFT solves) */
  int32_t op;      /* pint_op                                                                 */
  double nu;       /* heat diffusivity                                                        */
  double cx, cy;   /* advection velocity (cy ignored in 1-D)                                  */
  double T;        /* interval length, dT = T / L                                             */
  int32_t L;       /* time steps, power of two, 1 <= L <= 1024                        */
  int32_t M;       /* Radau IIA nodes, 1 <= M <= PINT_MAX_M                                   */
} pint_problem;

/* Time sharding (north star "partitioned by time steps"): with nranks = P > 1 rank
 * g owns the global steps l = g + P j, j < L/P (cyclic distribution).  The time DFT becomes a
 * four-step FFT: local L/P-point FFT + twiddle, one all-to-all, P-point DFT across ranks (and the
 * same backwards); the H-term of the residual needs the last node of step l-1, i.e. a ring halo
 * from rank g-1.  Requires (L/P) % P == 0 and M*P <= 32. */
typedef struct {
  int32_t rank, nranks;          /* nranks in {1, 2, 4, 8}, 0 <= rank < nranks                  */
  const void *nccl_unique_id;    /* nranks > 1: 128-byte ncclUniqueId (pint_nccl_unique_id on rank
                                    0, broadcast by the caller) -> NCCL over NVLink; NULL -> a
                                    "virtual rank" of a single-process loopback group driven by
                                    pint_group_iterate (all ranks on one device; tests)          */
  int32_t device;                /* CUDA device ordinal                                        */
  void *stream;                  /* cudaStream_t on which all work is enqueued (NULL = legacy) */
} pint_dist;

/* Bytes of device scratch pint_create needs in work_dev for this problem (0 on invalid input;
 * then pint_last_error() says why).  Includes one or two L*M*N complex128 work vectors, the
 * per-alpha factor tables for up to PINT_MAX_SCHEDULE alphas and reduction scratch. */
size_t pint_workspace_bytes(const pint_problem *p, const pint_dist *d);

/* Creates a context.  u_dev: caller-owned device buffer of (L/nranks)*M*N complex128 (16-byte
 * aligned; local steps j hold global steps rank + nranks*j), set here to u^(0) = u0 replicated
 * over all (l, m).  work_dev/work_bytes: caller-owned
 * device scratch (256-byte aligned, >= pint_workspace_bytes).  u0_host: 2N doubles (re, im),
 * copied.  forcing_host must be NULL (b == 0 at creation; a forcing is attached with
 * pint_set_forcing).  This call and every later one that enqueues work first make dist->device
 * the calling thread's current CUDA device (cudaSetDevice), so one thread may drive contexts on
 * several devices.
 * Errors: PINT_ERR_INVALID (sizes, alignment, NULL), PINT_ERR_NUMERIC (u0 not finite),
 * PINT_ERR_CUDA / PINT_ERR_NCCL (nothing is leaked: the context and its communicator are freed). */
pint_status pint_create(const pint_problem *p, const pint_dist *d, void *u_dev, void *work_dev,
                        size_t work_bytes, const double *u0_host, const double *forcing_host,
                        pint_ctx **out);

/* Algorithm 2's a-priori alpha sequence: gamma = L (3 eps + tau) w_inf,
 * alpha_{k+1} = sqrt(gamma / m_k), m_{k+1} = 2 sqrt(m_k gamma), m_0 = m0.  Pure host function.
 * alpha_out: K doubles; m_out: K+1 doubles (nullable).  PINT_ERR_SCHEDULE if m_k < 4 gamma. */
pint_status pint_adaptive_schedule(int32_t L, double w_inf, double m0, double eps, double tau,
                                   int32_t K, double *alpha_out, double *m_out);

/* ||w||_inf of the assembled w (Alg. 2's gamma), for pint_adaptive_schedule: ||u0||_inf
 * when b == 0 (host copy, no device work); with a forcing attached (pint_set_forcing)
 * max(||u0 + v_0||_inf, max_l ||v_l||_inf) reduced on the device (and over ranks with NCCL;
 * synchronises the stream).  Errors: PINT_ERR_INVALID, PINT_ERR_NUMERIC (non-finite),
 * PINT_ERR_STATE (loopback ranks with a forcing), PINT_ERR_CUDA / PINT_ERR_NCCL. */
pint_status pint_w_inf(pint_ctx *c, double *w_inf);

/* Copies K alphas (each in (0,1)), builds their per-alpha factor tables on the host in long
 * double (d_k, r_k, S_k, S_k^{-1}, G_k^{-1} S_k, d_km, PCR level coefficients) and uploads them;
 * resets the iteration counter to 0.  Every entry is built and validated before anything is
 * uploaded: on PINT_ERR_SCHEDULE / _NOT_DIAGONALIZABLE / _NUMERIC / _INVALID the context keeps
 * its previous schedule untouched.  Errors: PINT_ERR_SCHEDULE, PINT_ERR_NOT_DIAGONALIZABLE,
 * PINT_ERR_NUMERIC (1-D factorisation), PINT_ERR_INVALID (K > PINT_MAX_SCHEDULE), PINT_ERR_CUDA
 * (then the context holds no schedule). */
pint_status pint_set_alpha_schedule(pint_ctx *c, const double *alpha, int32_t K);

/* Iteration form.  PINT_FORM_CORRECTION (default; north star, reading R1):
 * u <- u + C_a^{-1}(w - C u).  PINT_FORM_DIRECT (Alg. 1 as printed, eq. Riteration
 * P:159): u <- C_a^{-1}((C_a - C) u + w); (C_a - C) u + w = w - alpha e_1 (x) H u_L has a
 * single non-zero block r0 = u0 - alpha u_{L-1,M-1}, so the residual pass and the forward time
 * transform collapse to one N-vector.  nranks > 1: the rank holding global
 * step L - 1 forms r0 and broadcasts it (N complex values); every rank synthesizes its local
 * frequencies S^{-1} x_k = sig_k r0, solves, and the inverse cross-rank DFT + all-to-all return
 * the result (no halo, no forward all-to-all).  Errors: PINT_ERR_INVALID (unknown form, a forcing
 * attached, non-power-of-two grids). */
#define PINT_FORM_CORRECTION 0
#define PINT_FORM_DIRECT 1
pint_status pint_set_form(pint_ctx *c, int32_t form);

/* Real-data fast path.  For real A, w and alpha (every
 * config: real u0, b == 0) the alpha-scaled time spectrum is Hermitian, x_{L-k} = conj(x_k)
 * (P:164-171 with real J and V^{-1} = F* J^{-1}), and so is the solution of the frequency-block
 * systems (the blocks of L - k are the complex conjugates of those of k).  on = 1: only the
 * L/2 + 1 frequencies k <= L/2 are node-transformed and solved; y_{L-k} = conj(y_k) is written
 * by the solve.  Same result as on = 0 up to the roundoff imaginary part of the iterate (which
 * on = 1 projects out).  The time transforms run on complex series that pack two real points,
 * z_l(n') = r_l(n') + i r_l(n' + N/2), so they do half the work; the solves unpack X_k from the
 * slots of k and L - k and the backward pass repacks both slots from one read.  Storage: while
 * on, the iterate is REAL fp64 u[l][m][n] in the first L M N doubles of u_dev (half the bytes of
 * every iterate read and write); switching on converts the current iterate (dropping its
 * roundoff imaginary parts), switching off converts back to complex128.  pint_get_iterate and
 * pint_get_final_value still return (re, 0) pairs.  Requirements: nranks == 1, u0 real (imaginary
 * parts exactly 0; pint_set_initial_value then rejects non-real data), 2-D: grids of the register
 * FFT engine, 4 <= L <= 1024; 1-D: N >= 8 and L >= 2; not with pint_sequential.  Errors:
 * PINT_ERR_INVALID, PINT_ERR_CUDA (storage conversion). */
pint_status pint_set_hermitian(pint_ctx *c, int32_t on);

/* Forcing b != 0: w = (u0 + v_0, v_1, ..., v_{L-1}) with
 * v_l = dT (Q (x) I_N) b_l, b_l[m] = b(t_l + tau_m dT) (the collocation integral of the forcing,
 * P:105).  v_dev: caller-owned device buffer, complex128 [L/P][M][N] (the local
 * steps l = rank + P j of this rank), 16-byte aligned, read by every iteration's residual (never
 * written; the caller keeps it alive); NULL removes the forcing.  The residual norms include it.
 * Not combinable with the direct form, the Hermitian mode or pint_sequential (the direct form's
 * single non-zero block and the packed real data assume b == 0).  The Algorithm 2 driver takes
 * gamma = L (3 eps + tau) ||w||_inf of this w (pint_w_inf).  Errors: PINT_ERR_INVALID. */
pint_status pint_set_forcing(pint_ctx *c, const void *v_dev);

/* Algorithm 2 of the paper, the stopping driver: gamma = L (3 eps + tau) ||w||_inf;
 * while m_k > tol: m_{k+1} = 2 sqrt(m_k gamma), alpha_{k+1} = sqrt(gamma / m_k), one iteration
 * (pint_iterate, current form), stop as soon as ||u_{L-1}^{k+1} - u_{L-1}^{k}||_inf <= tol.  Also
 * stops at max_iter and when m_k < 4 gamma (alpha would exceed 1/2).  The whole alpha
 * schedule (a function of gamma / m0 only) is built up front (replaces the current schedule);
 * one 8-byte read-back per iteration.  Outputs: *iters = iterations done; diffs (nullable,
 * max_iter entries) = the consecutive-iterate norms; m_out (nullable, max_iter + 1 entries) =
 * m_0 .. m_iters; *stop_reason (nullable): 0 consecutive iterates <= tol, 1 m_k <= tol,
 * 2 max_iter, 3 m_k < 4 gamma.  Errors: PINT_ERR_INVALID (m0, tol <= 0, max_iter outside
 * [1, PINT_MAX_SCHEDULE]), those of pint_set_alpha_schedule and pint_iterate. */
/* Sequential Radau IIA baseline: overwrites u_dev with the
 * sequential collocation solution u* of C u = w, step by step: (I - dT Q (x) A) U_l = 1 (x)
 * u_{l-1,M-1} (u_{-1} = u0), solved per step through Q = V diag(lambda) V^{-1} and the FFT
 * diagonal spatial solves on the same kernels as the iteration (one spatial pipeline launch per
 * step).  The fixed point of the iteration; used as the honest single-GPU time-stepping baseline.
 * 1-D: the M shifted tridiagonal solves of each step by the PCR kernels of the iteration (the
 * direct-form solve path with the shifts dT lambda_m), then U_l = (V (x) I) z.  Synchronous.
 * Requirements: power-of-two grids (2-D: grids of the spatial pipeline), nranks == 1.  Errors:
 * PINT_ERR_INVALID, PINT_ERR_NOT_DIAGONALIZABLE, PINT_ERR_CUDA. */
pint_status pint_sequential(pint_ctx *c);

pint_status pint_solve(pint_ctx *c, double m0, double eps, double tau, double tol, int32_t max_iter,
                       int32_t *iters, double *diffs, double *m_out, int32_t *stop_reason);

/* CUDA-graph form of pint_iterate for launch-bound problems (configs 1-2: a few microseconds of
 * kernels per iteration).  pint_graph_create captures n_iter iterations k, k+1, ... (alpha_k from
 * the schedule; advances k by n_iter like pint_iterate) into one executable graph on the context
 * stream; every pint_graph_launch replays exactly those iterations on the current buffers (with
 * the alphas captured: a fixed-alpha schedule makes each replay n_iter further iterations).
 * No last-step difference is produced.  One rank only.  The caller owns the graph
 * (pint_graph_destroy).  Errors: PINT_ERR_INVALID, PINT_ERR_SCHEDULE, PINT_ERR_CUDA. */
pint_status pint_graph_create(pint_ctx *c, int32_t n_iter, void **graph_exec);
pint_status pint_graph_launch(pint_ctx *c, void *graph_exec);
pint_status pint_graph_destroy(void *graph_exec);

/* Enqueues n_iter iterations k, k+1, ... with alpha_k from the schedule.  last_step_diff_inf:
 * nullable; if given, n_iter doubles receive ||u_{L-1}^{k+1} - u_{L-1}^{k}||_inf (Alg. 2 line 7,
 * P:421) and the call synchronises the stream; a non-finite difference (diverged or NaN iterate:
 * the device max propagates NaN) returns PINT_ERR_NUMERIC after filling the array.
 * PINT_ERR_SCHEDULE if the schedule would run out. */
pint_status pint_iterate(pint_ctx *c, int32_t n_iter, double *last_step_diff_inf);

/* ||w - C u||_2 and ||w - C u||_inf of the current (global) iterate (synchronises; with NCCL ranks
 * it exchanges the halo and all-reduces).  PINT_ERR_NUMERIC if non-finite. */
pint_status pint_residual_norm(pint_ctx *c, double *l2, double *linf);

/* D2H of the whole local iterate (2*L*M*N doubles) — parity checks (synchronises). */
pint_status pint_get_iterate(pint_ctx *c, double *u_host);

/* D2H of the last node of the last LOCAL step (2N doubles); on rank nranks-1 (and with one rank)
 * that is u_{L-1, M-1, :}, the solution at T. */
pint_status pint_get_final_value(pint_ctx *c, double *u_host);

/* Replaces u0 (H2D copy of 2N doubles, changes w) and, if reset_iterate != 0, resets the iterate
 * to u0 replicated.  Used by the end-to-end benchmark. */
pint_status pint_set_initial_value(pint_ctx *c, const double *u0_host, int32_t reset_iterate);

/* Windowed time stepping: start the next window of L steps from the current
 * iterate's final value, u0 := u_{L-1,M-1} (device copy; the host copy used by pint_w_inf and the
 * Hermitian check is refreshed), reset the iterate to it replicated and the schedule counter to 0.
 * Covering W L steps with W windows of Paralpha reproduces the paper's windowed runs.
 * One rank only.  Errors: PINT_ERR_INVALID, PINT_ERR_CUDA. */
pint_status pint_next_window(pint_ctx *c);

/* nranks > 1: a fresh 128-byte NCCL unique id for pint_dist.nccl_unique_id (call on rank 0 and
 * broadcast).  PINT_ERR_NCCL on failure. */
pint_status pint_nccl_unique_id(void *out128);

/* The global steps the local iterate holds: first, first + stride, ..., count of them. */
pint_status pint_local_steps(pint_ctx *c, int32_t *first, int32_t *stride, int32_t *count);

/* Single-process loopback group: ctxs[r] is rank r of a P-rank group created with
 * nccl_unique_id == NULL on ONE device and ONE stream.  Runs n_iter iterations of the sharded
 * algorithm phase by phase, moving the halo / all-to-all chunks with device-to-device copies
 * (no kernel ever waits on another rank).  last_step_diff_inf as in pint_iterate (nullable). */
pint_status pint_group_iterate(pint_ctx *const *ctxs, int32_t P, int32_t n_iter, double *last_step_diff_inf);

/* Global residual norms of a loopback group. */
pint_status pint_group_residual_norm(pint_ctx *const *ctxs, int32_t P, double *l2, double *linf);

/* Frees context-owned host state and the NCCL communicator; never caller buffers. */
pint_status pint_destroy(pint_ctx *c);

/* Thread-local message of the last non-OK status. */
const char *pint_last_error(void);

int32_t pint_abi_version(void);

/* 1 if the library was built with -DPINT_EXPERIMENTS (A/B builds that read the PINT_* environment
 * switches of csrc/internal.h), 0 for the product library, which ignores the environment. */
int32_t pint_experiments_enabled(void);

/* ---- introspection (tests / benchmarks) ------------------------------------------------- */

/* Number of kernel launches one iteration enqueues, and the names of the kernels. */
int32_t pint_launches_per_iteration(pint_ctx *c);

/* Runs n_iter iterations like pint_iterate (same kernels, same launch configuration) and records a
 * CUDA event after every launch on the context stream; kernel_ms[i] (pint_launches_per_iteration
 * entries) receives the average duration of launch i of an iteration.  Synchronises every
 * iteration. */
pint_status pint_iterate_profiled(pint_ctx *c, int32_t n_iter, double *kernel_ms);

/* Per-phase device times of the last iteration of an NCCL rank (nranks > 1), for the
 * communication / computation split of the overlapped schedule.  With timing on,
 * pint_iterate records CUDA events around the phases; ms[7] receives: 0 halo (pack + ring),
 * 1 forward (residual + local time FFT), 2 all-to-all #1 on the comm stream (first band issued ->
 * last band received), 3 middle on the compute stream (bands' cross-rank DFTs + spatial solves),
 * 4 from the end of the middle to the end of the iteration (exposed all-to-all #2 + backward),
 * 5 forward start -> all-to-all #2 complete, 6 the whole iteration.  Synchronises on the
 * iteration's last event.  Errors: PINT_ERR_INVALID (one rank / loopback), PINT_ERR_STATE. */
pint_status pint_set_phase_timing(pint_ctx *c, int32_t on);
pint_status pint_phase_times(pint_ctx *c, double *ms);

/* Name of launch i of an iteration ("" if out of range). */
const char *pint_kernel_name(pint_ctx *c, int32_t i);

/* Host copies of the factor tables of schedule entry `a` for frequency k (natural order):
 * d_k (2 doubles), S_k, S_k^{-1} (2*M*M doubles each, row-major), d_km (2*M doubles).
 * Any output pointer may be NULL. */
pint_status pint_get_factors(pint_ctx *c, int32_t a, int32_t k, double *d_k, double *S,
                             double *Sinv, double *d_km);

/* Radau IIA nodes t (M doubles) and Q (M*M, row-major) as computed by the library (long double,
 * rounded). */
pint_status pint_tableau(int32_t M, double *t, double *Q);

/* Stage-level debug entry: runs only stage s of iteration with schedule entry a on the current
 * buffers: 0 = forward (residual, scale, time DFT, S^-1) u -> X; 1 = spatial solves X -> X';
 * 2 = backward (G^-1 S, inverse DFT, unscale, u += c).  X/X' can be read with
 * pint_debug_get_work (which = 0 forward output, 1 solve output), frequency index bit-reversed. */
pint_status pint_debug_stage(pint_ctx *c, int32_t a, int32_t s);
pint_status pint_debug_get_work(pint_ctx *c, int32_t which, double *host);

#ifdef __cplusplus
}
#endif
#endif /* PINT_H */
