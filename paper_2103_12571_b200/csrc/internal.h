// Internal (non-ABI) declarations shared by the host side (pint_abi.cpp) and the kernels
// (kernels.cu).  No torch types anywhere.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

namespace pint {

// A/B experiment switches read from the environment (PINT_LEGACY2D, PINT_LEGACY_PIPE, PINT_FWD_T,
// PINT_BWD_T, PINT_SP_SKIP, PINT_SP_CLAIM).  Compiled in only with -DPINT_EXPERIMENTS: the product
// library ignores the environment (pint_experiments_enabled() == 0; bench.py refuses otherwise).
inline const char *experiment_env(const char *name) {
#ifdef PINT_EXPERIMENTS
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// Per-alpha device tables (pointers into work_dev).  Frequency index p is BIT-REVERSED:
// slot p holds frequency k = bitrev_L(p) (the time FFT leaves its output in that order).
struct AlphaTables {
  const double *scale_fwd;    // [L]       alpha^{l/L}                        (J^{-1})
  const double *scale_bwd;    // [L]       alpha^{-l/L} / L                   (J and 1/L of V)
  const double2 *Sinv;        // [L][M][M] S_k^{-1}
  const double2 *SG;          // [L][M][M] G_k^{-1} S_k = (I - r_k H_M) S_k
  const double2 *shift;       // [L][M]    s_km = d_km dT
  const double2 *pcr;         // [L][M][nlev] (p_j, q_j) pairs: 2 double2 per level  (1-D only)
  const double2 *inv_e;       // [L][M]    1 / e_final of the row-sum-carrying PCR   (1-D only)
  const double2 *sig;         // [L][M]    row sums of S_k^{-1} (direct form: S^{-1} (1 (x) r0))
  double alpha;
};

struct Geometry {
  int dim, nx, ny, N, L, M, op;
  int logL, logN, lognx, logny;
  double dT;
  // stencil of A (the paper's discretisations P:751-799, readings R8, R14):
  //   (A u)_n = sum_{o=-hx0}^{hx1} wx[3+o] u[x+o, y] + sum_{o=-hy0}^{hy1} wy[3+o] u[x, y+o]
  // periodic; the centre weights of both axes are folded into wx[3] (wy[3] = 0); hw = widest halo
  int hx0, hx1, hy0, hy1, hw;
  double wx[7], wy[7];
  int nfac;                   // 1-D: tridiagonal factors of I - s A solved by PCR (1..3)
  int pow2;                   // 1: power-of-two grid; 0: 7-smooth grid on the generic path (log2 fields 0)
  double dTQ[8 * 8];          // dT * Q, row-major
};

struct StaticTables {
  const double2 *twL;         // [L]  e^{-2 pi i q / L}   (L = local step count L/P)
  const double2 *twx;         // [nx] e^{-2 pi i q / nx}
  const double2 *twy;         // [ny] e^{-2 pi i q / ny}
  const double2 *lamx;        // [nx] per-axis symbol, natural kx
  const double2 *lamy;        // [ny]
  const double2 *u0;          // [N]
  // H-term source of the residual: the last node of the previous global step of local step l is
  // prev_base[(l - prev_shift) * prev_stride + n]; l - prev_shift < 0 means global step 0 (w = u0).
  //   1 rank:  prev_base = u + (M-1) N, prev_stride = M N, prev_shift = 1
  //   P ranks: prev_base = received ring halo [L/P][N], prev_stride = N, prev_shift = (rank == 0)
  const double2 *prev_base;
  long long prev_stride;
  int prev_shift;
  // four-step time FFT across P ranks (P > 1 only, else null): twr[p] = e^{-2 pi i rank kappa / L},
  // kappa = bitrev_{L/P}(p); twP[q] = e^{-2 pi i q / P}
  const double2 *twr;
  const double2 *twP;
  int P, rank;
  // per-pass twiddle tables of the register FFT engine (fft_reg.cuh) for nx, ny
  const double2 *ptwx, *ptwy;
  const double2 *ptwx5, *ptwy5;   // nx / ny plans with radix-32 passes (pipelined plane stages)
  const double2 *ptwL;            // L plan with radix-32 passes (pipelined time transforms)
  // Frequency units of the 2-D spatial solves: unit q < nsolve solves slot slots[q].  Default:
  // every slot (slots[q] = q), X holds the planes.  Hermitian (packed) mode (real data,
  // pint_set_hermitian): two real spatial points n' and n' + N/2 share one complex time series
  // Z[l][m][n'] = r(n') + i r(n' + N/2) in the first half of X (N/2 points per plane), units are
  // the L/2 + 1 frequencies k <= L/2, unit q's full planes live at X + L M N/2 + q M N, and
  // unitof[p] = q (slot p holds k <= L/2) or -1 - q (slot p holds L - k of unit q).
  const int *slots, *unitof;
  int nsolve;
  int packed;
  // packed mode on the pipelined plane passes: the complex series pairs the points (y, x) and
  // (y, x + nx/2), packed column y nx/2 + x (x < nx/2), so the R pass unpacks X_k row by row;
  // 0: the pairs (y, x), (y + ny/2, x) (packed column = point index of the first half)
  int xpair;
  int sm_reserve;             // NCCL ranks: SMs the persistent kernels leave free (comm/compute overlap)
  const double2 *v;           // forcing part of w, [L][M][N] local steps (nullptr: b == 0)
};

struct Buffers {
  double2 *u;                 // [L][M][N] iterate (caller-owned)
  double2 *X;                 // [L][M][N] work 1
  double2 *Y;                 // [L][M][N] work 2 (1-D two-pass PCR only; else == X)
  double *red;                // reduction scratch (doubles)
  unsigned *sync;             // 2-D spatial pipeline: per-(stage, batch) completion counters
};

// packed (Hermitian) mode: start of the unit planes inside the work vector X
__host__ __device__ inline double2 *unit_planes(const Geometry &g, double2 *X) { return X + (size_t)g.L * g.M * (g.N / 2); }

// ---- launch wrappers (kernels.cu) -----------------------------------------------------------
// All return cudaGetLastError() after enqueueing on `st`.
struct LaunchCfg {
  int fwd_T;                  // spatial points per forward tile (all l x all m, 1-D; <= 64 KB, 3 CTAs/SM)
  int bwd_T;                  // spatial points per backward tile (<= 100 KB: 128-byte rows at 2 CTAs/SM)
  int tfft_T;                 // spatial points per 2-D time-FFT tile (all l x one m)
  int pcr_mode;               // 0: single-pass line PCR; 1: two-pass (classes + chunks)
  int pcr_R;                  // residue-class modulus of the two-pass scheme
  int pcr_T;                  // class columns per CTA
  int pcr_chunk;              // contiguous chunk length of the small-stride pass
};

LaunchCfg choose_launch(const Geometry &g);

// cuTensorMapEncodeTiled from the driver (a PFN_cuTensorMapEncodeTiled_v12000), or nullptr
void *tma_encode_fn();
bool fwd1d_tma_ok(const Geometry &g, const StaticTables &st, int T);
// 1-D pipelined PCR passes (pcr1d.cu): classes of 256 points, one tridiagonal factor
bool pcr1d_pipe_supported(const Geometry &g, int R);
bool pcr1d_path(const Geometry &g, const LaunchCfg &lc);
cudaError_t launch_pcr1d_pipe(const Geometry &g, const AlphaTables &at, double2 *X, double2 *Y, const int *slots,
                              int lines, int R, cudaStream_t s, int sm_reserve);

// 2-D spatial solves as one persistent L2-resident pipeline (spatial2d.cu)
struct SpatialPlan {
  int lines;                  // planes (p, m) to solve
  int B, nbatch;              // planes per batch, batches
  int YR, TC;                 // rows per R/I item, columns per C item (64 KB tiles)
  int nRI, nC;                // items per batch of the R/I stages and of the C stage
  int synth;                  // direct form: C synthesizes sig_q * r0hat, no R stage
  int nstage, rounds;         // 3 (R, C, I) or 2 (C, I); nbatch + nstage - 1
  int skip;                   // timing experiments only (PINT_SP_SKIP): bit s = stage s does no work
  int claim;                  // 1: items claimed from a device counter; 0: static t = cta (mod grid)
};
SpatialPlan make_spatial_plan(const Geometry &g, int lines, bool synth);
int spatial_maxb(const Geometry &g);   // largest radix (log2) of the spatial FFT plan in use
size_t spatial_sync_bytes(int lines);
// X (lines planes [ny][nx]) solved in place; spec != nullptr: direct form (C reads spec = r0hat)
cudaError_t launch_spatial2d(const Geometry &g, const StaticTables &st, const AlphaTables &at, double2 *X,
                             const double2 *spec, unsigned *sync, int lines, cudaStream_t s);
bool spatial2d_supported(const Geometry &g);
// Pipelined per-stage plane passes (spatial2d.cu): the default for the grids and
// modes they serve (2-D, 512..4096 per axis, M <= 4, complex storage)
// Pipelined 2-D time transforms (spatial2d.cu): forward X in place (residual output -> slot order),
// inverse x2 -> u (+= or overwrite) with the last-step difference; L = 128 .. 1024, complex storage
bool tfft_pipe_supported(const Geometry &g, const StaticTables &st);
cudaError_t launch_tfft_pipe(const Geometry &g, const StaticTables &st, const AlphaTables *at, double2 *X,
                             const double2 *x2, double2 *u, bool inverse, unsigned long long *diff_slot, int overwrite,
                             cudaStream_t s);
// Generic-grid path (generic.cu): 7-smooth, non-power-of-two nx / ny (Tables 1-2), one rank,
// correction form; the residual and the spatial solves (node transforms included)
bool grid_is_smooth(long long n);
int generic_launches(const Geometry &g);
const char *generic_kernel_name(const Geometry &g, int i);
cudaError_t launch_generic_residual(const Geometry &g, const StaticTables &st, const AlphaTables &at,
                                    const double2 *u, double2 *X, cudaStream_t s);
cudaError_t launch_generic_solve(const Geometry &g, const StaticTables &st, const AlphaTables &at, double2 *X,
                                 cudaStream_t s);
// Fused R/C/I persistent launch (1024^2 grids, one rank, complex storage): the default there
bool spatial_fused_supported(const Geometry &g, const StaticTables &st);
cudaError_t launch_spatial_fused(const Geometry &g, const StaticTables &st, const AlphaTables &at, double2 *X,
                                 double2 *Yb, unsigned *sync, cudaStream_t s);
bool spatial_pipe_geometry(const Geometry &g);                          // grid/M served (needs a 2nd vector)
bool hermitian_pipe_path(const Geometry &g);                            // packed mode runs on the plane passes
bool spatial_pipe_supported(const Geometry &g, const StaticTables &st);  // ... and the current mode
// X natural -> R -> Yb blocked -> C (in place) -> I -> X natural; Yb must be a distinct vector.
// spec != nullptr: direct form -- no R pass; spec (the plane spectrum of r0) is re-laid out blocked
// into the first plane of X, the C pass loads it and synthesizes sig_q r0hat into Yb, then I -> X
cudaError_t launch_spatial_pipe(const Geometry &g, const StaticTables &st, const AlphaTables &at, double2 *X,
                                double2 *Yb, cudaStream_t s, const double2 *spec = nullptr);
bool reg2d_path(const Geometry &g);
bool pipe2d_geometry(const Geometry &g);   // the 2-D path can run the pipelined passes (2 work vectors)   // the 2-D path runs spatial2d (else the generic row/column kernels)
size_t fwd_smem_bytes(const Geometry &g, int T);

cudaError_t launch_forward(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                           const AlphaTables &at, const Buffers &b, cudaStream_t s);
// spatial solves on the lines of `in` (which must be b.X): result in *out (b.X or b.Y).
// node = true applies S^{-1} / G^{-1}S inside the solve passes where the design puts them
// (2-D row passes); with P > 1 they live in launch_xdft instead.
cudaError_t launch_solve(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                         const AlphaTables &at, const Buffers &b, cudaStream_t s, double2 **out);
cudaError_t launch_backward(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                            const AlphaTables &at, const Buffers &b, const double2 *x2,
                            double *diff_slot, cudaStream_t s, int overwrite);
// Direct form (Alg. 1 as printed, 1 rank): r0 = u0 - alpha u_{L-1,M-1}; its time transform is
// constant over frequencies, so x1_{k,m} = sig_km r0.  front: r0 (+ 2-D: one-plane forward FFT
// and the synthesized column pass into b.X); solve: 1-D PCR reading sig*r0 / 2-D inverse row
// pass; then launch_backward(..., overwrite = 1).
cudaError_t launch_direct_front(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                                const AlphaTables &at, const Buffers &b, double2 *r0, cudaStream_t s);
// the two halves of launch_direct_front: r0 = u0 - alpha u_{L-1,M-1} (local last step), and (2-D)
// its plane spectrum (+ the synthesized column pass on the legacy path); P ranks: rank P - 1
// computes r0, every rank the spectrum of the broadcast r0
cudaError_t launch_direct_r0(const Geometry &g, const StaticTables &st, const AlphaTables &at, const Buffers &b,
                             double2 *r0, cudaStream_t s);
cudaError_t launch_direct_spectrum(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                                   const AlphaTables &at, const Buffers &b, double2 *r0, cudaStream_t s);
cudaError_t launch_direct_solve(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                                const AlphaTables &at, const Buffers &b, const double2 *r0, cudaStream_t s,
                                double2 **out);
int launches_per_iteration_direct(const Geometry &g, const LaunchCfg &lc, const StaticTables &st);
const char *kernel_name_direct(const Geometry &g, const LaunchCfg &lc, const StaticTables &st, int i);
// Sequential Radau IIA baseline (2-D, one step): the spectrum of r0 (in place), then the direct-form
// synthesized spatial pipeline with the Q-eigen tables `at` (sig, shift, SG = V) writing the M
// stage planes of the step at `out`.
cudaError_t launch_sequential_step(const Geometry &g, const StaticTables &st, const AlphaTables &at,
                                   const Buffers &b, double2 *r0, double2 *out, cudaStream_t s);
// 1-D step of the sequential baseline: the M shifted PCR solves of sig_m r0 (launch_direct_solve
// on one slot with the tables `at`), then U_m = sum_j V_mj y_j into `out` ([M][N])
cudaError_t launch_sequential_step_1d(const Geometry &g, const LaunchCfg &lc, const StaticTables &st,
                                      const AlphaTables &at, const Buffers &b, double2 *r0, double2 *out,
                                      cudaStream_t s);
cudaError_t launch_residual_norm(const Geometry &g, const StaticTables &st, const Buffers &b,
                                 double *out2, cudaStream_t s);
cudaError_t launch_init_iterate(const Geometry &g, const StaticTables &st, const Buffers &b,
                                cudaStream_t s);
// ||w||_inf of w = (u0 + v_0, v_1, ...) with the forcing st.v attached (one double at `out`)
cudaError_t launch_w_inf(const Geometry &g, const StaticTables &st, double *out, cudaStream_t s);
// Hermitian mode storage switch of the iterate u: complex128 <-> real fp64 (first L M N doubles)
cudaError_t launch_storage_convert(const Geometry &g, const Buffers &b, bool to_real, cudaStream_t s);
cudaError_t launch_square_first(const double *in, double *out, cudaStream_t s);
cudaError_t launch_sqrt_into(const double *in, double *out, cudaStream_t s);
// P > 1: pack the last-node planes u[l][M-1][:] of all local steps into hsend[l][:]
cudaError_t launch_halo_pack(const Geometry &g, const Buffers &b, double2 *hsend, cudaStream_t s);
// P > 1: cross-rank P-point DFT (+ S^{-1}) from the all-to-all receive buffer Yin[src][pl][m][n]
// into slot order Xout[q*(L/P^2... see kernels.cu)], and its inverse (G^{-1} S, inverse DFT) into
// send chunks by destination.
// pl0 / npl: the band of chunk slots pl0 .. pl0 + npl (npl < 0: to the end) of the overlapped
// schedule
cudaError_t launch_xdft(const Geometry &g, const StaticTables &st, const AlphaTables &at,
                        const double2 *in, double2 *out, bool inverse, cudaStream_t s, int pl0 = 0, int npl = -1);
int launches_per_iteration(const Geometry &g, const LaunchCfg &lc, const StaticTables &st);
const char *kernel_name(const Geometry &g, const LaunchCfg &lc, const StaticTables &st, int i);

// Optional per-launch event recorder (pint_iterate_profiled): when set, every launch wrapper
// records ev[n++] on the launch stream right after each kernel it enqueues.
struct Recorder {
  cudaEvent_t *ev;
  int n, cap;
};
void set_recorder(Recorder *r);
void record_launch(cudaStream_t s);   // records the recorder's next event (no-op when unset)

}  // namespace pint
