// C ABI of libpint (include/pint.h): validation, host factor tables (long double), workspace
// carving and the stream-ordered iteration driver.  Every step of the iteration runs in the
// kernels of kernels.cu; this file only builds tables and enqueues launches.
#include <cuda_runtime.h>
#include <nccl.h>
#include <thread>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: named ranges for nsys / ncu timelines

#include "../../include/pint.h"
#include "host_numerics.h"
#include "internal.h"

using namespace pint;

namespace {

thread_local std::string g_err;

pint_status fail(pint_status s, const std::string &msg) {
  g_err = msg;
  return s;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Layout {
  size_t vec_bytes;      // one local (L/P)*M*N complex128 vector
  size_t off_X, off_Y;
  size_t off_hsend, off_hrecv, halo_bytes;   // P > 1: ring halo buffers [L/P][N]
  size_t off_r0;                              // direct form: r0 / its 2-D spectrum [N]
  size_t off_static, static_bytes;
  size_t off_alpha, alpha_bytes_each;
  size_t off_red, red_bytes;
  size_t off_sync, sync_bytes;                // 2-D spatial pipeline completion counters
  size_t off_sym;                             // unit slot list and slot -> unit map [2][L] int
  size_t off_band;                            // P > 1: band slot lists of the overlapped schedule
  size_t off_seq;                             // sequential baseline: Q eigen tables (sig, shift, V)
  size_t total;
  bool two_vectors;
};

}  // namespace

struct pint_ctx {
  pint_problem prob;
  pint_dist dist;
  int P = 1, rank = 0;
  ncclComm_t comm = nullptr;       // P > 1 with an NCCL unique id
  bool loopback = false;           // P > 1 without an id: driven by pint_group_iterate
  Geometry g;
  LaunchCfg lc;
  Layout lay;
  cudaStream_t stream;
  char *work;
  double2 *u;
  StaticTables st;
  std::vector<AlphaTables> at;
  std::vector<double> alphas;
  int k = 0;
  int form = PINT_FORM_CORRECTION;
  bool hermitian = false;
  bool poisoned = false;
  // P > 1, overlapped schedule: the chunk slots pl < L/P^2 split into `bands`
  // bands; the all-to-alls of band b run on `comm` while the compute stream solves band b - 1
  int bands = 1;
  cudaStream_t commstream = nullptr;
  bool commstream_owned = false;
  std::vector<cudaEvent_t> ev;     // [0] forward done, then per band: a2a#1, mid, a2a#2
  bool phase_timing = false;       // pint_set_phase_timing: timed events around the phases
  cudaEvent_t tev[8] = {};         // start, halo, fwd, a2a#1 first, a2a#1 last, mid end, a2a#2 last, end
  std::vector<ld> t, Q;
  std::vector<double> u0;          // host copy (2N)
  // host copies of the factor tables (natural frequency order) for introspection
  std::vector<std::vector<cld>> h_S, h_Sinv, h_dkm;
  std::vector<std::vector<cld>> h_dk;
};

static pint_status validate(const pint_problem *p, const pint_dist *d) {
  if (!p) return fail(PINT_ERR_INVALID, "problem is NULL");
  if (p->dim != 1 && p->dim != 2) return fail(PINT_ERR_INVALID, "dim must be 1 or 2");
  // power-of-two grids (every BASELINE config), or 7-smooth sizes 2^a 3^b 5^c 7^d (Tables 1-2,
  // P:751-799) on the generic path: <= 4096 per axis, one rank
  if (!grid_is_smooth(p->nx) || p->nx < 4) return fail(PINT_ERR_INVALID, "nx must be a power of two or 7-smooth, >= 4");
  if (p->dim == 1 && p->ny != 1) return fail(PINT_ERR_INVALID, "ny must be 1 in 1-D");
  if (p->dim == 2 && (!grid_is_smooth(p->ny) || p->ny < 4))
    return fail(PINT_ERR_INVALID, "ny must be a power of two or 7-smooth, >= 4");
  if (p->nx > (1 << 20) || p->ny > 4096) return fail(PINT_ERR_INVALID, "grid too large");
  if (p->dim == 2 && (p->nx > 4096)) return fail(PINT_ERR_INVALID, "2-D nx must be <= 4096");
  const bool pow2 = is_pow2(p->nx) && (p->dim == 1 || is_pow2(p->ny));
  if (!pow2 && p->nx > 4096) return fail(PINT_ERR_INVALID, "non-power-of-two grids: nx <= 4096");
  if (!pow2 && d && d->nranks > 1) return fail(PINT_ERR_INVALID, "non-power-of-two grids run on one rank");
  if (p->op < PINT_OP_HEAT || p->op > PINT_OP_UPWIND4) return fail(PINT_ERR_INVALID, "unknown op");
  if (!is_pow2(p->L) || p->L > 1024) return fail(PINT_ERR_INVALID, "L must be a power of two <= 1024 (P:592)");
  if (p->M < 1 || p->M > PINT_MAX_M) return fail(PINT_ERR_INVALID, "M must be in [1, 8]");
  if (!(p->T > 0) || !std::isfinite(p->T)) return fail(PINT_ERR_INVALID, "T must be > 0");
  if (!std::isfinite(p->nu) || !std::isfinite(p->cx) || !std::isfinite(p->cy))
    return fail(PINT_ERR_INVALID, "non-finite coefficient");
  if (d) {
    const int P = d->nranks;
    if (P != 1 && P != 2 && P != 4 && P != 8) return fail(PINT_ERR_INVALID, "nranks must be 1, 2, 4 or 8");
    if (d->rank < 0 || d->rank >= P) return fail(PINT_ERR_INVALID, "rank out of range");
    if (P > 1) {
      if ((p->L / P) % P != 0 || p->L < P * P)
        return fail(PINT_ERR_INVALID, "time sharding needs (L/nranks) % nranks == 0 (four-step FFT, L >= nranks^2)");
      if (p->M * P > 32) return fail(PINT_ERR_INVALID, "time sharding needs M * nranks <= 32");
    }
  }
  return PINT_OK;
}

static Geometry make_geometry(const pint_problem *p, int P) {
  Geometry g{};
  g.dim = p->dim;
  g.nx = p->nx;
  g.ny = p->dim == 2 ? p->ny : 1;
  g.N = g.nx * g.ny;
  g.L = p->L / P;          // local step count (cyclic distribution l = rank + P j)
  g.M = p->M;
  g.op = p->op;
  g.pow2 = is_pow2(g.nx) && is_pow2(g.ny) ? 1 : 0;
  g.logL = ilog2(g.L);
  g.logN = g.pow2 ? ilog2(g.N) : 0;        // generic grids: no log2 plans (generic.cu)
  g.lognx = g.pow2 ? ilog2(g.nx) : 0;
  g.logny = g.pow2 ? ilog2(g.ny) : 0;
  g.dT = p->T / p->L;      // global step size
  // stencil weights (long double rationals rounded once; readings R8, R14)
  AxisStencil sx, sy;
  axis_stencil(p->op, g.nx, op_is_heat(p->op) ? p->nu : p->cx, sx);
  if (g.dim == 2) axis_stencil(p->op, g.ny, op_is_heat(p->op) ? p->nu : p->cy, sy);
  g.hx0 = sx.h0; g.hx1 = sx.h1; g.hy0 = sy.h0; g.hy1 = sy.h1;
  g.hw = std::max(std::max(sx.h0, sx.h1), std::max(sy.h0, sy.h1));
  for (int o = 0; o < 7; ++o) {
    g.wx[o] = (double)(o == 3 ? sx.w[3] + sy.w[3] : sx.w[o]);
    g.wy[o] = o == 3 ? 0.0 : (double)sy.w[o];
  }
  g.nfac = g.dim == 1 && g.pow2 ? stencil_factor_count(p->op, sx) : 1;
  return g;
}

static Layout make_layout(const Geometry &g, const LaunchCfg &lc, int P) {
  Layout L{};
  L.vec_bytes = (size_t)g.L * g.M * g.N * sizeof(double2);
  L.two_vectors = (g.dim == 1 && lc.pcr_mode == 1) || P > 1 || pipe2d_geometry(g);
  size_t off = 0;
  L.off_X = off;
  // 2-D: one extra M x N unit plane group (Hermitian packed mode: units 0..L/2 after Z)
  off = align_up(off + L.vec_bytes + (g.dim == 2 ? (size_t)g.M * g.N * sizeof(double2) : 0), 256);
  L.off_Y = L.two_vectors ? off : L.off_X;
  if (L.two_vectors) off = align_up(off + L.vec_bytes, 256);
  L.halo_bytes = P > 1 ? (size_t)g.L * g.N * sizeof(double2) : 0;
  L.off_hsend = off;
  off = align_up(off + L.halo_bytes, 256);
  L.off_hrecv = off;
  off = align_up(off + L.halo_bytes, 256);
  L.off_r0 = off;
  off = align_up(off + (size_t)g.N * sizeof(double2), 256);
  L.off_static = off;
  const int mb = g.dim == 2 ? spatial_maxb(g) : 4;
  L.static_bytes = (size_t)(g.L + g.nx + g.ny + g.nx + g.ny + g.N + g.L + 8 + pass_twiddle_count(g.lognx, mb) +
                            pass_twiddle_count(g.logny, mb) + pass_twiddle_count(g.lognx, 5) +
                            pass_twiddle_count(g.logny, 5) + pass_twiddle_count(g.logL, 5)) * sizeof(double2);
  off = align_up(off + L.static_bytes, 256);
  L.off_alpha = off;
  const size_t LM = (size_t)g.L * g.M;
  size_t per = 2 * g.L * sizeof(double);                                 // scale_fwd, scale_bwd
  per = align_up(per, 16);
  per += 2 * LM * g.M * sizeof(double2);                                   // Sinv, SG
  per += LM * sizeof(double2);                                             // shift
  per += LM * sizeof(double2);                                             // sig (row sums of S^{-1})
  if (g.dim == 1) per += LM * g.logN * g.nfac * 2 * sizeof(double2) + LM * sizeof(double2);  // pcr, inv_e
  L.alpha_bytes_each = align_up(per, 256);
  off += L.alpha_bytes_each * PINT_MAX_SCHEDULE;
  L.off_red = off;
  L.red_bytes = (size_t)(148 * 8 * 2 + 64 + PINT_MAX_SCHEDULE * 8) * sizeof(double) * 2;
  off = align_up(off + L.red_bytes, 256);
  L.off_sync = off;
  L.sync_bytes = g.dim == 2 ? spatial_sync_bytes(g.L * g.M) : 0;
  off = align_up(off + L.sync_bytes, 256);
  L.off_sym = off;
  off = align_up(off + 2 * (size_t)g.L * sizeof(int), 256);
  L.off_band = off;                                        // P > 1: slot lists of the bands (L ints)
  off = align_up(off + (size_t)g.L * sizeof(int), 256);
  L.off_seq = off;   // 1-D: + the PCR level tables and 1/e of the M shifts
  off = align_up(off + (size_t)(2 * g.M + g.M * g.M) * sizeof(double2), 256);
  if (g.dim == 1) off = align_up(off + ((size_t)g.M * g.logN * g.nfac * 2 + g.M) * sizeof(double2), 256);
  L.total = off;
  return L;
}

#define CUDA_TRY(c, expr)                                                                 \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) {                                                              \
      if (c) (c)->poisoned = true;                                                        \
      return fail(PINT_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));     \
    }                                                                                     \
  } while (0)

// Host wait on the context stream.  On an NCCL rank the wait polls the communicator's asynchronous
// error state (ncclCommGetAsyncError): a failed peer or link surfaces as PINT_ERR_NCCL — the
// communicator is aborted and the context poisoned — instead of leaving the host hanging in
// cudaStreamSynchronize.
static pint_status sync_stream(pint_ctx *c) {
  if (!c->comm) {
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return PINT_OK;
  }
  for (;;) {
    cudaError_t e = cudaStreamQuery(c->stream);
    if (e == cudaSuccess) return PINT_OK;
    if (e != cudaErrorNotReady) {
      c->poisoned = true;
      return fail(PINT_ERR_CUDA, std::string("cudaStreamQuery: ") + cudaGetErrorString(e));
    }
    ncclResult_t async = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError(c->comm, &async);
    if (r != ncclSuccess || (async != ncclSuccess && async != ncclInProgress)) {
      c->poisoned = true;
      ncclCommAbort(c->comm);
      c->comm = nullptr;
      return fail(PINT_ERR_NCCL, std::string("asynchronous communicator error: ") +
                                     ncclGetErrorString(r != ncclSuccess ? r : async));
    }
    std::this_thread::yield();
  }
}
#define PINT_SYNC(c)                       \
  do {                                     \
    pint_status _s = sync_stream(c);       \
    if (_s != PINT_OK) return _s;          \
  } while (0)

// pint_create error paths: free the half-built context and its communicator (nothing leaks)
static pint_status create_abort(pint_ctx *c, pint_status st) {
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
  return st;
}
#define CREATE_TRY(c, expr)                                                                       \
  do {                                                                                            \
    cudaError_t _e = (expr);                                                                      \
    if (_e != cudaSuccess)                                                                        \
      return create_abort(c, fail(PINT_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e))); \
  } while (0)

// entry points that enqueue work bind the context's device first (cheap when already current), so
// a thread driving contexts on several devices never launches on the wrong one
#define BIND_DEVICE(c)                                                                            \
  do {                                                                                            \
    cudaError_t _e = cudaSetDevice((c)->dist.device);                                             \
    if (_e != cudaSuccess) return fail(PINT_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(_e)); \
  } while (0)

extern "C" {

int32_t pint_abi_version(void) { return PINT_ABI_VERSION; }

int32_t pint_experiments_enabled(void) {
#ifdef PINT_EXPERIMENTS
  return 1;
#else
  return 0;
#endif
}

const char *pint_last_error(void) { return g_err.c_str(); }

size_t pint_workspace_bytes(const pint_problem *p, const pint_dist *d) {
  if (validate(p, d) != PINT_OK) return 0;
  const int P = d ? d->nranks : 1;
  Geometry g = make_geometry(p, P);
  return make_layout(g, choose_launch(g), P).total;
}

pint_status pint_tableau(int32_t M, double *t, double *Q) {
  if (M < 1 || M > PINT_MAX_M) return fail(PINT_ERR_INVALID, "M must be in [1, 8]");
  std::vector<ld> tt, QQ;
  if (!radau_tableau(M, tt, QQ)) return fail(PINT_ERR_NUMERIC, "Radau root finding failed");
  for (int i = 0; i < M; ++i) if (t) t[i] = (double)tt[i];
  for (int i = 0; i < M * M; ++i) if (Q) Q[i] = (double)QQ[i];
  return PINT_OK;
}

pint_status pint_adaptive_schedule(int32_t L, double w_inf, double m0, double eps, double tau,
                                   int32_t K, double *alpha_out, double *m_out) {
  if (K < 0 || K > 4096 || (K > 0 && !alpha_out)) return fail(PINT_ERR_INVALID, "bad K / output");
  std::vector<double> a, m;
  std::string err;
  if (!adaptive_schedule(L, w_inf, m0, eps, tau, K, a, m, err)) return fail(PINT_ERR_SCHEDULE, err);
  for (int i = 0; i < K; ++i) alpha_out[i] = a[i];
  if (m_out) for (int i = 0; i <= K; ++i) m_out[i] = m[i];
  return PINT_OK;
}

pint_status pint_create(const pint_problem *p, const pint_dist *d, void *u_dev, void *work_dev,
                        size_t work_bytes, const double *u0_host, const double *forcing_host,
                        pint_ctx **out) {
  if (!out) return fail(PINT_ERR_INVALID, "out is NULL");
  *out = nullptr;
  pint_status s = validate(p, d);
  if (s != PINT_OK) return s;
  if (!d) return fail(PINT_ERR_INVALID, "dist is NULL");
  if (!u_dev || !work_dev || !u0_host) return fail(PINT_ERR_INVALID, "NULL buffer");
  for (size_t i = 0; i < 2 * (size_t)p->nx * (p->dim == 2 ? p->ny : 1); ++i)
    if (!std::isfinite(u0_host[i])) return fail(PINT_ERR_NUMERIC, "u0 has a non-finite entry");
  if (forcing_host) return fail(PINT_ERR_INVALID, "forcing_host must be NULL (attach a forcing with pint_set_forcing)");
  if (((uintptr_t)u_dev) % 16) return fail(PINT_ERR_INVALID, "u_dev must be 16-byte aligned");
  if (((uintptr_t)work_dev) % 256) return fail(PINT_ERR_INVALID, "work_dev must be 256-byte aligned");
  const int P = d->nranks, rank = d->rank;
  Geometry g = make_geometry(p, P);
  LaunchCfg lc = choose_launch(g);
  Layout lay = make_layout(g, lc, P);
  if (work_bytes < lay.total) return fail(PINT_ERR_INVALID, "work_bytes < pint_workspace_bytes");

  pint_ctx *c = new pint_ctx();
  c->prob = *p;
  c->dist = *d;
  c->P = P;
  c->rank = rank;
  c->g = g;
  c->lc = lc;
  c->lay = lay;
  c->stream = (cudaStream_t)d->stream;
  c->work = (char *)work_dev;
  c->u = (double2 *)u_dev;
  if (!radau_tableau(p->M, c->t, c->Q)) {
    delete c;
    return fail(PINT_ERR_NUMERIC, "Radau root finding failed");
  }
  for (int m = 0; m < p->M; ++m)
    for (int j = 0; j < p->M; ++j) c->g.dTQ[m * p->M + j] = (double)((ld)p->T / p->L * c->Q[m * p->M + j]);

  cudaError_t e = cudaSetDevice(d->device);
  if (e != cudaSuccess) { delete c; return fail(PINT_ERR_CUDA, cudaGetErrorString(e)); }

  // static tables: twiddles, symbols, u0
  std::vector<double2> host(lay.static_bytes / sizeof(double2));
  size_t o = 0;
  auto tw = [&](int n) {
    for (int q = 0; q < n; ++q) {
      cld w = unit_root(q, n, -1);
      host[o++] = make_double2((double)w.real(), (double)w.imag());
    }
  };
  size_t o_twL = o; tw(g.L);
  size_t o_twx = o; tw(g.nx);
  size_t o_twy = o; tw(g.ny);
  auto lam = [&](int n, double coef) {
    for (int k = 0; k < n; ++k) {
      const cld v = axis_symbol(p->op, n, k, coef);
      host[o++] = make_double2((double)v.real(), (double)v.imag());
    }
  };
  const bool heat = op_is_heat(p->op);
  size_t o_lx = o; lam(g.nx, heat ? p->nu : p->cx);
  size_t o_ly = o; lam(g.ny, heat ? p->nu : p->cy);
  if (g.dim == 1) for (size_t i = o_ly; i < o_ly + g.ny; ++i) host[i] = make_double2(0, 0);
  size_t o_u0 = o;
  c->u0.assign(u0_host, u0_host + 2 * (size_t)g.N);
  for (int n = 0; n < g.N; ++n) host[o++] = make_double2(u0_host[2 * n], u0_host[2 * n + 1]);
  // four-step tables (P > 1): twr[p] = e^{-2 pi i rank bitrev_Ll(p) / L}, twP[q] = e^{-2 pi i q / P}
  size_t o_twr = o;
  for (int q = 0; q < g.L; ++q) {
    cld w = unit_root((long long)rank * bitrev(q, g.logL), p->L, -1);
    host[o++] = make_double2((double)w.real(), (double)w.imag());
  }
  size_t o_twP = o;
  for (int q = 0; q < 8; ++q) {
    cld w = unit_root(q % P, P, -1);
    host[o++] = make_double2((double)w.real(), (double)w.imag());
  }
  const int mb = g.dim == 2 ? spatial_maxb(g) : 4;   // plan of the spatial FFT kernels
  auto ptw = [&](int logn) {
    std::vector<cld> v;
    pass_twiddles(logn, mb, v);
    for (const cld &w : v) host[o++] = make_double2((double)w.real(), (double)w.imag());
  };
  size_t o_px = o; ptw(g.lognx);
  size_t o_py = o; ptw(g.logny);
  auto ptw5 = [&](int logn) {   // radix-32 plans of the pipelined plane passes
    std::vector<cld> v;
    pass_twiddles(logn, 5, v);
    for (const cld &w : v) host[o++] = make_double2((double)w.real(), (double)w.imag());
  };
  size_t o_px5 = o; ptw5(g.lognx);
  size_t o_py5 = o; ptw5(g.logny);
  size_t o_pL5 = o; ptw5(g.logL);
  double2 *sbase = (double2 *)(c->work + lay.off_static);
  CREATE_TRY(c, cudaMemcpyAsync(sbase, host.data(), o * sizeof(double2), cudaMemcpyHostToDevice, c->stream));
  c->st.twL = sbase + o_twL;
  c->st.twx = sbase + o_twx;
  c->st.twy = sbase + o_twy;
  c->st.lamx = sbase + o_lx;
  c->st.lamy = sbase + o_ly;
  c->st.u0 = sbase + o_u0;
  c->st.ptwx = sbase + o_px;
  c->st.ptwy = sbase + o_py;
  c->st.ptwx5 = sbase + o_px5;
  c->st.ptwy5 = sbase + o_py5;
  c->st.ptwL = sbase + o_pL5;
  c->st.P = P;
  c->st.rank = rank;
  if (P == 1) {
    c->st.prev_base = c->u + (size_t)(g.M - 1) * g.N;
    c->st.prev_stride = (long long)g.M * g.N;
    c->st.prev_shift = 1;
    c->st.twr = nullptr;
    c->st.twP = nullptr;
  } else {
    c->st.prev_base = (const double2 *)(c->work + lay.off_hrecv);
    c->st.prev_stride = g.N;
    c->st.prev_shift = rank == 0 ? 1 : 0;
    c->st.twr = sbase + o_twr;
    c->st.twP = sbase + o_twP;
    if (d->nccl_unique_id) {
      ncclUniqueId id;
      std::memcpy(&id, d->nccl_unique_id, sizeof id);
      ncclResult_t r = ncclCommInitRank(&c->comm, P, id, rank);
      if (r != ncclSuccess) {
        c->comm = nullptr;
        return create_abort(c, fail(PINT_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)));
      }
    } else {
      c->loopback = true;
    }
  }
  {
    std::vector<int> sym(2 * (size_t)g.L);
    for (int q = 0; q < g.L; ++q) { sym[q] = q; sym[g.L + q] = q; }
    int *dsym = (int *)(c->work + lay.off_sym);
    CREATE_TRY(c, cudaMemcpyAsync(dsym, sym.data(), sym.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    c->st.slots = dsym;
    c->st.unitof = dsym + g.L;
    c->st.nsolve = g.L;
    c->st.packed = 0;
    c->st.v = nullptr;
    c->st.sm_reserve = (P > 1 && !c->loopback) ? 16 : 0;   // SMs left to NCCL's kernels (overlap)
  }
  if (P > 1) {
    // overlapped schedule: bands of the chunk slots pl (the 2-D plane passes of spatial2d.cu address
    // planes by slot, so a band's slot list {q Lc + pl : q < P, pl in band} is enough; the 1-D PCR
    // and the generic row / column kernels work on whole slot ranges: one band)
    const int Lc = g.L / P;
    int B = g.dim == 2 && reg2d_path(g) ? 4 : 1;
    while (B > 1 && Lc % B) B >>= 1;
    c->bands = B;
    std::vector<int> band((size_t)g.L);
    const int nb = Lc / B;
    size_t o2 = 0;
    for (int bb = 0; bb < B; ++bb)
      for (int q = 0; q < P; ++q)
        for (int pl = bb * nb; pl < (bb + 1) * nb; ++pl) band[o2++] = q * Lc + pl;
    CREATE_TRY(c, cudaMemcpyAsync(c->work + lay.off_band, band.data(), band.size() * sizeof(int),
                                  cudaMemcpyHostToDevice, c->stream));
    if (!c->loopback) {
      CREATE_TRY(c, cudaStreamCreateWithFlags(&c->commstream, cudaStreamNonBlocking));
      c->commstream_owned = true;
    }
    c->ev.resize(1 + 3 * B);
    for (auto &e : c->ev) CREATE_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  Buffers b{c->u, (double2 *)(c->work + lay.off_X), (double2 *)(c->work + lay.off_Y),
            (double *)(c->work + lay.off_red), (unsigned *)(c->work + lay.off_sync)};
  CREATE_TRY(c, launch_init_iterate(c->g, c->st, b, c->stream));
  CREATE_TRY(c, cudaStreamSynchronize(c->stream));  // host staging buffer goes out of scope
  *out = c;
  return PINT_OK;
}

static Buffers buffers(pint_ctx *c) {
  return Buffers{c->u, (double2 *)(c->work + c->lay.off_X), (double2 *)(c->work + c->lay.off_Y),
                 (double *)(c->work + c->lay.off_red), (unsigned *)(c->work + c->lay.off_sync)};
}

pint_status pint_w_inf(pint_ctx *c, double *w_inf) {
  if (!c || !w_inf) return fail(PINT_ERR_INVALID, "NULL argument");
  if (!c->st.v) {   // b == 0: w = (u0 replicated, 0, ..., 0)
    double m = 0;
    for (int n = 0; n < c->g.N; ++n) m = std::fmax(m, std::hypot(c->u0[2 * n], c->u0[2 * n + 1]));
    *w_inf = m;
    return PINT_OK;
  }
  // forcing attached: w = (u0 + v_0, v_1, ..., v_{L-1}) reduced on the device
  BIND_DEVICE(c);
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  double *slot = (double *)(c->work + c->lay.off_red) + 148 * 8 * 2 + 64 + PINT_MAX_SCHEDULE;
  CUDA_TRY(c, launch_w_inf(c->g, c->st, slot, c->stream));
  if (c->P > 1) {
    if (!c->comm) return fail(PINT_ERR_STATE, "loopback (virtual-rank) context: ||w|| needs every rank");
    ncclResult_t r = ncclAllReduce(slot, slot, 1, ncclDouble, ncclMax, c->comm, c->stream);
    if (r != ncclSuccess) { c->poisoned = true; return fail(PINT_ERR_NCCL, ncclGetErrorString(r)); }
  }
  double h = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&h, slot, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  PINT_SYNC(c);
  if (!std::isfinite(h)) return fail(PINT_ERR_NUMERIC, "non-finite ||w||_inf");
  *w_inf = h;
  return PINT_OK;
}

// 1-D: I - s A = lead prod_f T_f (host_numerics: factor_shifted); row-sum-carrying PCR
// coefficients per factor (reading R6), levels interleaved: lev[(j F + f) 2 + {0, 1}] =
// (p_j, q_j) of factor f; *inv_e = 1 / (lead prod_f e_f,final)
static bool pcr_tables(const pint_ctx *c, const AxisStencil &sx, cld s, double2 *lev, double2 *inv_e,
                       std::string &err) {
  const Geometry &g = c->g;
  const int F = g.nfac;
  std::vector<TriFactor> fac;
  cld lead;
  if (!factor_shifted(c->prob.op, sx, s, fac, lead, err) || (int)fac.size() != F) {
    if (err.empty()) err = "unexpected factor count";
    return false;
  }
  cld ie = 1.0L / lead;
  for (int f = 0; f < F; ++f) {
    cld ca = fac[f].a, cc = fac[f].c, e = fac[f].e;
    cld cb = e - ca - cc;
    for (int j = 0; j < g.logN - 1; ++j) {
      cld pj = ca / cb, qj = cc / cb;
      lev[(j * F + f) * 2] = make_double2((double)pj.real(), (double)pj.imag());
      lev[(j * F + f) * 2 + 1] = make_double2((double)qj.real(), (double)qj.imag());
      cld e2 = e * (e - 2.0L * (ca + cc)) / cb;
      cld a2 = -ca * ca / cb, c2 = -cc * cc / cb;
      ca = a2; cc = c2; e = e2; cb = e - ca - cc;
    }
    cld pl = (ca + cc) / cb;                        // pair level: i-h == i+h
    lev[((g.logN - 1) * F + f) * 2] = make_double2((double)pl.real(), (double)pl.imag());
    lev[((g.logN - 1) * F + f) * 2 + 1] = make_double2(0.0, 0.0);
    e = e * (e - 2.0L * (ca + cc)) / cb;
    ie /= e;
  }
  *inv_e = make_double2((double)ie.real(), (double)ie.imag());
  return true;
}

pint_status pint_set_alpha_schedule(pint_ctx *c, const double *alpha, int32_t K) {
  if (!c) return fail(PINT_ERR_INVALID, "ctx is NULL");
  BIND_DEVICE(c);
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  if (K < 0 || K > PINT_MAX_SCHEDULE || (K > 0 && !alpha))
    return fail(PINT_ERR_INVALID, "K must be in [0, PINT_MAX_SCHEDULE]");
  for (int a = 0; a < K; ++a)
    if (!(alpha[a] > 0.0 && alpha[a] < 1.0)) return fail(PINT_ERR_SCHEDULE, "alpha must be in (0, 1)");
  const Geometry &g = c->g;
  const int L = g.L, M = g.M;            // L: local step / frequency-slot count
  const int Lg = c->prob.L, P = c->P, rank = c->rank;
  const ld dT = (ld)c->prob.T / Lg;
  // A's stencil along x for the 1-D PCR factors (host_numerics: factor_shifted)
  AxisStencil sx;
  axis_stencil(c->prob.op, g.nx, op_is_heat(c->prob.op) ? c->prob.nu : c->prob.cx, sx);
  const int F = g.nfac;
  std::vector<AlphaTables> tabs(K);
  std::vector<std::vector<cld>> hS(K), hSi(K), hD(K), hdk(K);
  // every blob is built and validated on the host before any upload: a failing entry leaves the
  // context's current schedule and its device tables untouched
  std::vector<std::vector<char>> blobs(K, std::vector<char>(c->lay.alpha_bytes_each, 0));
  std::vector<size_t> offs_pcr(K, 0), offs_inv(K, 0);
  for (int a = 0; a < K; ++a) {
    std::vector<char> &blob = blobs[a];
    const ld al = alpha[a];
    double *sf = (double *)blob.data();
    double *sb = sf + L;
    size_t off = align_up(2 * L * sizeof(double), 16);
    double2 *Sinv = (double2 *)(blob.data() + off); off += (size_t)L * M * M * sizeof(double2);
    double2 *SG = (double2 *)(blob.data() + off); off += (size_t)L * M * M * sizeof(double2);
    double2 *shift = (double2 *)(blob.data() + off); off += (size_t)L * M * sizeof(double2);
    double2 *sig = (double2 *)(blob.data() + off); off += (size_t)L * M * sizeof(double2);
    double2 *pcr = nullptr, *inv_e = nullptr;
    size_t off_pcr = 0, off_inv = 0;
    if (g.dim == 1) {
      off_pcr = off;
      pcr = (double2 *)(blob.data() + off); off += (size_t)L * M * g.logN * F * 2 * sizeof(double2);
      off_inv = off;
      inv_e = (double2 *)(blob.data() + off); off += (size_t)L * M * sizeof(double2);
    }
    for (int j = 0; j < L; ++j) {
      const ld lgl = (ld)(rank + (long long)P * j);      // global step of local step j
      sf[j] = (double)powl(al, lgl / Lg);                // alpha^{l/L}
      sb[j] = (double)(powl(al, -lgl / Lg) / Lg);        // alpha^{-l/L} / L
    }
    hS[a].assign((size_t)Lg * M * M, cld(0));
    hSi[a].assign((size_t)Lg * M * M, cld(0));
    hD[a].assign((size_t)Lg * M, cld(0));
    hdk[a].assign(Lg, cld(0));
    const ld aroot = powl(al, 1.0L / Lg);
    for (int p = 0; p < L; ++p) {
      // frequency of local slot p: 1 rank: bit-reversed order; P ranks: slot q*Lc + pl holds
      // kappa + Ll q with kappa = bitrev_Ll(rank*Lc + pl)  (four-step order, kernels.cu)
      int k;
      if (P == 1) {
        k = bitrev(p, g.logL);
      } else {
        const int Lc = L / P, q = p / Lc, pl = p % Lc;
        k = bitrev(rank * Lc + pl, g.logL) + L * q;
      }
      const cld dk = -aroot * unit_root(k, Lg, -1);       // d_k = -alpha^{1/L} e^{-2 pi i k/L}
      const cld rk = dk / (1.0L + dk);                     // r_k = d_k / (1 + d_k)
      hdk[a][k] = dk;
      std::vector<cld> B((size_t)M * M);
      for (int m = 0; m < M; ++m)
        for (int j = 0; j < M; ++j)
          B[(size_t)m * M + j] = c->Q[(size_t)m * M + j] - (j == M - 1 ? rk * c->t[m] : cld(0));  // Q - r D_t H
      std::vector<cld> lam, S, Si;
      ld cond, gap;
      if (!eig_diagonalize(M, B, lam, S, Si, cond, gap)) {
        char buf[256];
        snprintf(buf, sizeof buf, "Q G_k^{-1} not safely diagonalisable for alpha=%.6g, k=%d (cond=%.3Lg gap=%.3Lg)",
                 (double)al, k, cond, gap);
        return fail(PINT_ERR_NOT_DIAGONALIZABLE, buf);
      }
      for (int i = 0; i < M * M; ++i) { hS[a][(size_t)k * M * M + i] = S[i]; hSi[a][(size_t)k * M * M + i] = Si[i]; }
      for (int m = 0; m < M; ++m) hD[a][(size_t)k * M + m] = lam[m];
      for (int m = 0; m < M; ++m) {
        cld rs = 0;
        for (int j = 0; j < M; ++j) rs += Si[(size_t)m * M + j];
        sig[(size_t)p * M + m] = make_double2((double)rs.real(), (double)rs.imag());
      }
      for (int m = 0; m < M; ++m)
        for (int j = 0; j < M; ++j) {
          cld v = Si[(size_t)m * M + j];
          Sinv[((size_t)p * M + m) * M + j] = make_double2((double)v.real(), (double)v.imag());
          cld w = S[(size_t)m * M + j] - rk * S[(size_t)(M - 1) * M + j];   // (I - r H_M) S
          SG[((size_t)p * M + m) * M + j] = make_double2((double)w.real(), (double)w.imag());
        }
      for (int m = 0; m < M; ++m) {
        const cld s = lam[m] * dT;                          // (I - d_km dT A)
        shift[(size_t)p * M + m] = make_double2((double)s.real(), (double)s.imag());
        if (g.dim == 1 && g.pow2) {
          std::string ferr;
          if (!pcr_tables(c, sx, s, pcr + ((size_t)p * M + m) * g.logN * F * 2, inv_e + (size_t)p * M + m, ferr)) {
            char buf[256];
            snprintf(buf, sizeof buf, "1-D spatial factorisation failed for alpha=%.6g, k=%d, m=%d: %s",
                     (double)al, k, m, ferr.c_str());
            return fail(PINT_ERR_NUMERIC, buf);
          }
        }
      }
    }
    offs_pcr[a] = off_pcr;
    offs_inv[a] = off_inv;
  }
  // commit: the old schedule is dropped first, so a failed upload leaves no schedule (ERR_SCHEDULE)
  c->at.clear();
  c->alphas.clear();
  for (int a = 0; a < K; ++a) {
    const ld al = alpha[a];
    const size_t off_pcr = offs_pcr[a], off_inv = offs_inv[a];
    char *dst = c->work + c->lay.off_alpha + (size_t)a * c->lay.alpha_bytes_each;
    CUDA_TRY(c, cudaMemcpyAsync(dst, blobs[a].data(), blobs[a].size(), cudaMemcpyHostToDevice, c->stream));
    AlphaTables &t = tabs[a];
    t.scale_fwd = (const double *)dst;
    t.scale_bwd = (const double *)dst + L;
    size_t o2 = align_up(2 * L * sizeof(double), 16);
    t.Sinv = (const double2 *)(dst + o2); o2 += (size_t)L * M * M * sizeof(double2);
    t.SG = (const double2 *)(dst + o2); o2 += (size_t)L * M * M * sizeof(double2);
    t.shift = (const double2 *)(dst + o2); o2 += (size_t)L * M * sizeof(double2);
    t.sig = (const double2 *)(dst + o2); o2 += (size_t)L * M * sizeof(double2);
    t.alpha = (double)al;
    t.pcr = g.dim == 1 ? (const double2 *)(dst + off_pcr) : nullptr;
    t.inv_e = g.dim == 1 ? (const double2 *)(dst + off_inv) : nullptr;
  }
  PINT_SYNC(c);   // host blobs go out of scope
  c->at = tabs;
  c->alphas.assign(alpha, alpha + K);
  c->h_S = hS;
  c->h_Sinv = hSi;
  c->h_dkm = hD;
  c->h_dk = hdk;
  c->k = 0;
  return PINT_OK;
}

static double2 *hsend(pint_ctx *c) { return (double2 *)(c->work + c->lay.off_hsend); }
static double2 *hrecv(pint_ctx *c) { return (double2 *)(c->work + c->lay.off_hrecv); }
static size_t chunk_elems(pint_ctx *c) { return (size_t)(c->g.L / c->P) * c->g.M * c->g.N; }

// ---- phases of one iteration.  1 rank: forward -> solve -> backward on one GPU.  P ranks
// (DESIGN.md §7): [pack halo] -> ring exchange -> forward (residual with the received halo,
// local FFT, four-step twiddle) -> all-to-all -> cross-rank DFT + S^{-1} -> solves ->
// G^{-1}S + inverse cross-rank DFT -> all-to-all -> backward.
enum Phase { PH_PRE, PH_FWD, PH_MID, PH_BWD };

struct IterState {
  double2 *solved = nullptr;     // buffer holding the solve output (P > 1: then the A2A-back target)
  double2 *send_back = nullptr;  // P > 1: inverse cross-rank DFT output (send chunks)
};

// NVTX range of one step group of the iteration (host-side markers, no device work)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static pint_status run_phase(pint_ctx *c, Phase ph, int a, double *diff_slot, IterState &is) {
  static const char *kPhaseName[] = {"pint halo (ring exchange pack)", "pint (i)-(ii) residual + time DFT",
                                     "pint (iii)-(iv) node transforms + spatial solves",
                                     "pint (v) inverse transforms + update"};
  NvtxRange range(kPhaseName[ph]);
  Buffers b = buffers(c);
  const AlphaTables &at = c->at[a];
  switch (ph) {
    case PH_PRE:
      if (c->P > 1) CUDA_TRY(c, launch_halo_pack(c->g, b, hsend(c), c->stream));
      break;
    case PH_FWD:
      CUDA_TRY(c, launch_forward(c->g, c->lc, c->st, at, b, c->stream));
      break;
    case PH_MID: {
      if (c->P > 1) CUDA_TRY(c, launch_xdft(c->g, c->st, at, b.Y, b.X, false, c->stream));
      double2 *x2 = nullptr;
      CUDA_TRY(c, launch_solve(c->g, c->lc, c->st, at, b, c->stream, &x2));
      if (c->P > 1) {
        double2 *other = (x2 == b.X) ? b.Y : b.X;
        CUDA_TRY(c, launch_xdft(c->g, c->st, at, x2, other, true, c->stream));
        is.send_back = other;
        is.solved = x2;        // A2A back lands here (its contents are no longer needed)
      } else {
        is.solved = x2;
      }
      break;
    }
    case PH_BWD:
      CUDA_TRY(c, launch_backward(c->g, c->lc, c->st, at, b, is.solved, diff_slot, c->stream, 0));
      break;
  }
  return PINT_OK;
}

// NCCL exchanges of one rank (all on the context stream)
static pint_status nccl_halo(pint_ctx *c) {
  const size_t cnt = (size_t)c->g.L * c->g.N * 2;
  const int next = (c->rank + 1) % c->P, prev = (c->rank + c->P - 1) % c->P;
  ncclResult_t r = ncclGroupStart();
  if (r == ncclSuccess) r = ncclSend(hsend(c), cnt, ncclDouble, next, c->comm, c->stream);
  if (r == ncclSuccess) r = ncclRecv(hrecv(c), cnt, ncclDouble, prev, c->comm, c->stream);
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess) {
    c->poisoned = true;
    return fail(PINT_ERR_NCCL, std::string("halo exchange: ") + ncclGetErrorString(r != ncclSuccess ? r : r2));
  }
  return PINT_OK;
}

// band bb of every peer chunk: chunk slots pl in [bb nb, (bb + 1) nb), contiguous in both buffers
static size_t band_elems(pint_ctx *c) { return chunk_elems(c) / c->bands; }

static pint_status nccl_alltoall(pint_ctx *c, const double2 *send, double2 *recv, int bb) {
  const size_t ce = chunk_elems(c), be = band_elems(c), off = (size_t)bb * be;
  ncclResult_t r = ncclGroupStart();
  for (int d = 0; d < c->P && r == ncclSuccess; ++d) {
    r = ncclSend(send + d * ce + off, be * 2, ncclDouble, d, c->comm, c->commstream);
    if (r == ncclSuccess) r = ncclRecv(recv + d * ce + off, be * 2, ncclDouble, d, c->comm, c->commstream);
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess) {
    c->poisoned = true;
    return fail(PINT_ERR_NCCL, std::string("all-to-all: ") + ncclGetErrorString(r != ncclSuccess ? r : r2));
  }
  return PINT_OK;
}

// P > 1: the middle of one band (chunk slots pl in band bb): cross-rank DFT + S^{-1} (Y -> X),
// the spatial solves of the band's slots, G^{-1} S + inverse cross-rank DFT (X -> Y send chunks)
static pint_status run_mid_band(pint_ctx *c, int a, int bb, IterState &is) {
  Buffers b = buffers(c);
  const AlphaTables &at = c->at[a];
  const int Lc = c->g.L / c->P, nb = Lc / c->bands;
  CUDA_TRY(c, launch_xdft(c->g, c->st, at, b.Y, b.X, false, c->stream, bb * nb, nb));
  StaticTables sb = c->st;
  sb.slots = (const int *)(c->work + c->lay.off_band) + (size_t)bb * c->P * nb;
  sb.nsolve = c->P * nb;
  double2 *x2 = nullptr;
  CUDA_TRY(c, launch_solve(c->g, c->lc, sb, at, b, c->stream, &x2));
  double2 *other = (x2 == b.X) ? b.Y : b.X;
  CUDA_TRY(c, launch_xdft(c->g, c->st, at, x2, other, true, c->stream, bb * nb, nb));
  is.send_back = other;
  is.solved = x2;
  return PINT_OK;
}

// P > 1, direct form: the middle of every rank once r0 (broadcast from rank P - 1) is in place:
// x1_sigma = sig_sigma r0 synthesized in the local slot order (the alpha-scaled time DFT of the
// single non-zero block r0 is r0 at every frequency), the spatial solves, G^{-1} S + inverse
// cross-rank DFT into the send chunks
static pint_status run_direct_mid(pint_ctx *c, int a, IterState &is) {
  Buffers b = buffers(c);
  const AlphaTables &at = c->at[a];
  double2 *r0 = (double2 *)(c->work + c->lay.off_r0);
  CUDA_TRY(c, launch_direct_spectrum(c->g, c->lc, c->st, at, b, r0, c->stream));
  double2 *x2 = nullptr;
  CUDA_TRY(c, launch_direct_solve(c->g, c->lc, c->st, at, b, r0, c->stream, &x2));
  double2 *other = (x2 == b.X) ? b.Y : b.X;
  CUDA_TRY(c, launch_xdft(c->g, c->st, at, x2, other, true, c->stream));
  is.send_back = other;
  is.solved = x2;
  return PINT_OK;
}

static pint_status run_iteration(pint_ctx *c, int a, double *diff_slot) {
  NvtxRange range("pint iteration");
  IterState is;
  pint_status st;
  if (c->form == PINT_FORM_DIRECT && c->P > 1) {   // time-sharded direct form
    if (!c->comm) return fail(PINT_ERR_STATE, "loopback (virtual-rank) context: use pint_group_iterate");
    Buffers b = buffers(c);
    const AlphaTables &at = c->at[a];
    double2 *r0 = (double2 *)(c->work + c->lay.off_r0);
    const bool pt = c->phase_timing;   // phases: halo = the broadcast, no forward, no all-to-all #1
    if (pt) CUDA_TRY(c, cudaEventRecord(c->tev[0], c->stream));
    if (c->rank == c->P - 1) CUDA_TRY(c, launch_direct_r0(c->g, c->st, at, b, r0, c->stream));
    ncclResult_t r = ncclBroadcast(r0, r0, (size_t)c->g.N * 2, ncclDouble, c->P - 1, c->comm, c->stream);
    if (r != ncclSuccess) { c->poisoned = true; return fail(PINT_ERR_NCCL, std::string("broadcast: ") + ncclGetErrorString(r)); }
    if (pt)
      for (int i : {1, 2, 3, 4}) CUDA_TRY(c, cudaEventRecord(c->tev[i], c->stream));
    if ((st = run_direct_mid(c, a, is)) != PINT_OK) return st;
    CUDA_TRY(c, cudaEventRecord(c->ev[0], c->stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->commstream, c->ev[0], 0));
    for (int bb = 0; bb < c->bands; ++bb)
      if ((st = nccl_alltoall(c, is.send_back, is.solved, bb)) != PINT_OK) return st;
    CUDA_TRY(c, cudaEventRecord(c->ev[1], c->commstream));
    if (pt) CUDA_TRY(c, cudaEventRecord(c->tev[6], c->commstream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev[1], 0));
    if (pt) CUDA_TRY(c, cudaEventRecord(c->tev[5], c->stream));
    CUDA_TRY(c, launch_backward(c->g, c->lc, c->st, at, b, is.solved, c->rank == c->P - 1 ? diff_slot : nullptr,
                                c->stream, 1));
    if (pt) CUDA_TRY(c, cudaEventRecord(c->tev[7], c->stream));
    return PINT_OK;
  }
  if (c->form == PINT_FORM_DIRECT) {  // Alg. 1 as printed: u = C_a^{-1}((C_a - C) u + w), 1 rank
    Buffers b = buffers(c);
    const AlphaTables &at = c->at[a];
    double2 *r0 = (double2 *)(c->work + c->lay.off_r0);
    CUDA_TRY(c, launch_direct_front(c->g, c->lc, c->st, at, b, r0, c->stream));
    double2 *x2 = nullptr;
    CUDA_TRY(c, launch_direct_solve(c->g, c->lc, c->st, at, b, r0, c->stream, &x2));
    CUDA_TRY(c, launch_backward(c->g, c->lc, c->st, at, b, x2, diff_slot, c->stream, 1));
    return PINT_OK;
  }
  if (c->P == 1) {
    if ((st = run_phase(c, PH_FWD, a, nullptr, is)) != PINT_OK) return st;
    if ((st = run_phase(c, PH_MID, a, nullptr, is)) != PINT_OK) return st;
    return run_phase(c, PH_BWD, a, diff_slot, is);
  }
  if (!c->comm) return fail(PINT_ERR_STATE, "loopback (virtual-rank) context: use pint_group_iterate");
  Buffers b = buffers(c);
  const bool pt = c->phase_timing;
  if (pt) CUDA_TRY(c, cudaEventRecord(c->tev[0], c->stream));
  if ((st = run_phase(c, PH_PRE, a, nullptr, is)) != PINT_OK) return st;
  if ((st = nccl_halo(c)) != PINT_OK) return st;
  if (pt) CUDA_TRY(c, cudaEventRecord(c->tev[1], c->stream));
  if ((st = run_phase(c, PH_FWD, a, nullptr, is)) != PINT_OK) return st;
  if (pt) CUDA_TRY(c, cudaEventRecord(c->tev[2], c->stream));
  // overlapped middle: all-to-all #1 of every band on the comm stream; band b's
  // cross-rank DFT + solves + inverse DFT on the compute stream as soon as its data arrived, its
  // all-to-all #2 right after it, overlapping band b + 1's compute
  const int B = c->bands;
  CUDA_TRY(c, cudaEventRecord(c->ev[0], c->stream));
  CUDA_TRY(c, cudaStreamWaitEvent(c->commstream, c->ev[0], 0));
  if (pt) CUDA_TRY(c, cudaEventRecord(c->tev[3], c->commstream));
  for (int bb = 0; bb < B; ++bb) {
    if ((st = nccl_alltoall(c, b.X, b.Y, bb)) != PINT_OK) return st;
    CUDA_TRY(c, cudaEventRecord(c->ev[1 + 3 * bb], c->commstream));
  }
  if (pt) CUDA_TRY(c, cudaEventRecord(c->tev[4], c->commstream));
  for (int bb = 0; bb < B; ++bb) {
    CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev[1 + 3 * bb], 0));
    if ((st = run_mid_band(c, a, bb, is)) != PINT_OK) return st;
    CUDA_TRY(c, cudaEventRecord(c->ev[2 + 3 * bb], c->stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->commstream, c->ev[2 + 3 * bb], 0));
    if ((st = nccl_alltoall(c, is.send_back, is.solved, bb)) != PINT_OK) return st;
    CUDA_TRY(c, cudaEventRecord(c->ev[3 + 3 * bb], c->commstream));
  }
  if (pt) {
    CUDA_TRY(c, cudaEventRecord(c->tev[5], c->stream));
    CUDA_TRY(c, cudaEventRecord(c->tev[6], c->commstream));
  }
  CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev[3 * B], 0));   // the comm stream is in order
  // last-step diff: only the rank holding global step L-1 (rank P-1) reports it
  if ((st = run_phase(c, PH_BWD, a, c->rank == c->P - 1 ? diff_slot : nullptr, is)) != PINT_OK) return st;
  if (pt) CUDA_TRY(c, cudaEventRecord(c->tev[7], c->stream));
  return PINT_OK;
}

pint_status pint_iterate(pint_ctx *c, int32_t n_iter, double *last_step_diff_inf) {
  if (!c) return fail(PINT_ERR_INVALID, "ctx is NULL");
  BIND_DEVICE(c);
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  if (n_iter < 0) return fail(PINT_ERR_INVALID, "n_iter < 0");
  if (c->loopback) return fail(PINT_ERR_STATE, "loopback (virtual-rank) context: use pint_group_iterate");
  if (c->k + n_iter > (int)c->alphas.size())
    return fail(PINT_ERR_SCHEDULE, "alpha schedule exhausted (call pint_set_alpha_schedule)");
  double *slots = nullptr;
  if (last_step_diff_inf && n_iter > 0) {
    slots = (double *)(c->work + c->lay.off_red) + 148 * 8 * 2 + 64;
    if (n_iter > PINT_MAX_SCHEDULE) return fail(PINT_ERR_INVALID, "n_iter too large");
    CUDA_TRY(c, cudaMemsetAsync(slots, 0, n_iter * sizeof(double), c->stream));
  }
  for (int i = 0; i < n_iter; ++i) {
    pint_status s = run_iteration(c, c->k, slots ? slots + i : nullptr);
    if (s != PINT_OK) return s;
    c->k++;
  }
  if (slots) {
    if (c->P > 1) {  // only rank P-1 wrote its slots; max over ranks gives everyone the value
      ncclResult_t r = ncclAllReduce(slots, slots, n_iter, ncclDouble, ncclMax, c->comm, c->stream);
      if (r != ncclSuccess) { c->poisoned = true; return fail(PINT_ERR_NCCL, ncclGetErrorString(r)); }
    }
    CUDA_TRY(c, cudaMemcpyAsync(last_step_diff_inf, slots, n_iter * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    PINT_SYNC(c);
    for (int i = 0; i < n_iter; ++i)   // the device max propagates NaN (nanmax): a diverged iterate
      if (!std::isfinite(last_step_diff_inf[i])) return fail(PINT_ERR_NUMERIC, "non-finite last-step difference");
  }
  return PINT_OK;
}

pint_status pint_nccl_unique_id(void *out128) {
  if (!out128) return fail(PINT_ERR_INVALID, "NULL argument");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(PINT_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof id);
  return PINT_OK;
}

pint_status pint_local_steps(pint_ctx *c, int32_t *first, int32_t *stride, int32_t *count) {
  if (!c) return fail(PINT_ERR_INVALID, "ctx is NULL");
  if (first) *first = c->rank;
  if (stride) *stride = c->P;
  if (count) *count = c->g.L;
  return PINT_OK;
}

pint_status pint_group_iterate(pint_ctx *const *ctxs, int32_t P, int32_t n_iter, double *last_step_diff_inf) {
  if (!ctxs || P < 2) return fail(PINT_ERR_INVALID, "need the P >= 2 contexts of one virtual group");
  for (int r = 0; r < P; ++r) {
    pint_ctx *c = ctxs[r];
    if (!c || !c->loopback || c->P != P || c->rank != r)
      return fail(PINT_ERR_INVALID, "ctxs[r] must be the loopback context of rank r of a P-rank group");
    if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
    if (c->stream != ctxs[0]->stream || c->dist.device != ctxs[0]->dist.device)
      return fail(PINT_ERR_INVALID, "virtual ranks must share one device and one stream");
    if (c->k != ctxs[0]->k || c->alphas.size() != ctxs[0]->alphas.size() || c->form != ctxs[0]->form)
      return fail(PINT_ERR_STATE, "virtual ranks out of step (schedule position or form)");
    if (c->k + n_iter > (int)c->alphas.size())
      return fail(PINT_ERR_SCHEDULE, "alpha schedule exhausted (call pint_set_alpha_schedule)");
  }
  if (n_iter < 0) return fail(PINT_ERR_INVALID, "n_iter < 0");
  cudaStream_t s = ctxs[0]->stream;
  const size_t ce = chunk_elems(ctxs[0]) * sizeof(double2);
  const size_t hb = ctxs[0]->lay.halo_bytes;
  double *slots = nullptr;
  pint_ctx *last = ctxs[P - 1];
  if (last_step_diff_inf && n_iter > 0) {
    if (n_iter > PINT_MAX_SCHEDULE) return fail(PINT_ERR_INVALID, "n_iter too large");
    slots = (double *)(last->work + last->lay.off_red) + 148 * 8 * 2 + 64;
    CUDA_TRY(last, cudaMemsetAsync(slots, 0, n_iter * sizeof(double), s));
  }
  // second (copy) stream of the group and its events (the virtual ranks' own ones are unused)
  cudaStream_t cs = nullptr;
  std::vector<cudaEvent_t> gev(1 + 3 * ctxs[0]->bands, nullptr);
  struct Cleanup {
    cudaStream_t &cs;
    std::vector<cudaEvent_t> &ev;
    ~Cleanup() {
      if (cs) { cudaStreamSynchronize(cs); cudaStreamDestroy(cs); }
      for (cudaEvent_t e : ev) if (e) cudaEventDestroy(e);
    }
  } cleanup{cs, gev};
  CUDA_TRY(last, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  for (auto &e : gev) CUDA_TRY(last, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (int it = 0; it < n_iter; ++it) {
    std::vector<IterState> is(P);
    const int a = ctxs[0]->k;
    pint_status st;
    if (last->form == PINT_FORM_DIRECT) {   // the time-sharded direct form of run_iteration
      double2 *r0l = (double2 *)(last->work + last->lay.off_r0);
      CUDA_TRY(last, launch_direct_r0(last->g, last->st, last->at[a], buffers(last), r0l, s));
      for (int r = 0; r < P - 1; ++r)   // "broadcast" from rank P - 1
        CUDA_TRY(ctxs[r], cudaMemcpyAsync(ctxs[r]->work + ctxs[r]->lay.off_r0, r0l,
                                          (size_t)last->g.N * sizeof(double2), cudaMemcpyDeviceToDevice, s));
      for (int r = 0; r < P; ++r)
        if ((st = run_direct_mid(ctxs[r], a, is[r])) != PINT_OK) return st;
      for (int src = 0; src < P; ++src)
        for (int dst = 0; dst < P; ++dst)
          CUDA_TRY(ctxs[src], cudaMemcpyAsync((char *)is[dst].solved + src * ce, (const char *)is[src].send_back + dst * ce,
                                              ce, cudaMemcpyDeviceToDevice, s));
      for (int r = 0; r < P; ++r)
        CUDA_TRY(ctxs[r], launch_backward(ctxs[r]->g, ctxs[r]->lc, ctxs[r]->st, ctxs[r]->at[a], buffers(ctxs[r]),
                                          is[r].solved, (r == P - 1 && slots) ? slots + it : nullptr, s, 1));
      for (int r = 0; r < P; ++r) ctxs[r]->k++;
      continue;
    }
    for (int r = 0; r < P; ++r)
      if ((st = run_phase(ctxs[r], PH_PRE, a, nullptr, is[r])) != PINT_OK) return st;
    for (int r = 0; r < P; ++r)  // ring: rank r -> rank r+1
      CUDA_TRY(ctxs[r], cudaMemcpyAsync(hrecv(ctxs[(r + 1) % P]), hsend(ctxs[r]), hb, cudaMemcpyDeviceToDevice, s));
    for (int r = 0; r < P; ++r)
      if ((st = run_phase(ctxs[r], PH_FWD, a, nullptr, is[r])) != PINT_OK) return st;
    // the overlapped middle of run_iteration with device copies on a second stream: every band's
    // all-to-all #1, then per band the middle of every rank and its all-to-all #2
    const int B = ctxs[0]->bands;
    const size_t be = ce / B;
    CUDA_TRY(last, cudaEventRecord(gev[0], s));
    CUDA_TRY(last, cudaStreamWaitEvent(cs, gev[0], 0));
    for (int bb = 0; bb < B; ++bb) {
      for (int src = 0; src < P; ++src)
        for (int dst = 0; dst < P; ++dst)
          CUDA_TRY(ctxs[src], cudaMemcpyAsync((char *)buffers(ctxs[dst]).Y + src * ce + bb * be,
                                              (const char *)buffers(ctxs[src]).X + dst * ce + bb * be, be,
                                              cudaMemcpyDeviceToDevice, cs));
      CUDA_TRY(last, cudaEventRecord(gev[1 + 3 * bb], cs));
    }
    for (int bb = 0; bb < B; ++bb) {
      CUDA_TRY(last, cudaStreamWaitEvent(s, gev[1 + 3 * bb], 0));
      for (int r = 0; r < P; ++r)
        if ((st = run_mid_band(ctxs[r], a, bb, is[r])) != PINT_OK) return st;
      CUDA_TRY(last, cudaEventRecord(gev[2 + 3 * bb], s));
      CUDA_TRY(last, cudaStreamWaitEvent(cs, gev[2 + 3 * bb], 0));
      for (int src = 0; src < P; ++src)
        for (int dst = 0; dst < P; ++dst)
          CUDA_TRY(ctxs[src], cudaMemcpyAsync((char *)is[dst].solved + src * ce + bb * be,
                                              (const char *)is[src].send_back + dst * ce + bb * be, be,
                                              cudaMemcpyDeviceToDevice, cs));
      CUDA_TRY(last, cudaEventRecord(gev[3 + 3 * bb], cs));
    }
    CUDA_TRY(last, cudaStreamWaitEvent(s, gev[3 * B], 0));
    for (int r = 0; r < P; ++r)
      if ((st = run_phase(ctxs[r], PH_BWD, a, (r == P - 1 && slots) ? slots + it : nullptr, is[r])) != PINT_OK)
        return st;
    for (int r = 0; r < P; ++r) ctxs[r]->k++;
  }
  if (slots) {
    CUDA_TRY(last, cudaMemcpyAsync(last_step_diff_inf, slots, n_iter * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(last, cudaStreamSynchronize(s));
  }
  return PINT_OK;
}

pint_status pint_group_residual_norm(pint_ctx *const *ctxs, int32_t P, double *l2, double *linf) {
  if (!ctxs || P < 2) return fail(PINT_ERR_INVALID, "need the P >= 2 contexts of one virtual group");
  for (int r = 0; r < P; ++r)
    if (!ctxs[r] || !ctxs[r]->loopback || ctxs[r]->P != P || ctxs[r]->rank != r)
      return fail(PINT_ERR_INVALID, "ctxs[r] must be the loopback context of rank r of a P-rank group");
  cudaStream_t s = ctxs[0]->stream;
  const size_t hb = ctxs[0]->lay.halo_bytes;
  for (int r = 0; r < P; ++r) CUDA_TRY(ctxs[r], launch_halo_pack(ctxs[r]->g, buffers(ctxs[r]), hsend(ctxs[r]), s));
  for (int r = 0; r < P; ++r)
    CUDA_TRY(ctxs[r], cudaMemcpyAsync(hrecv(ctxs[(r + 1) % P]), hsend(ctxs[r]), hb, cudaMemcpyDeviceToDevice, s));
  double sum2 = 0.0, mx = 0.0;
  for (int r = 0; r < P; ++r) {
    pint_ctx *c = ctxs[r];
    double *out2 = (double *)(c->work + c->lay.off_red) + 148 * 8 * 2;
    CUDA_TRY(c, launch_residual_norm(c->g, c->st, buffers(c), out2, s));
    double h[2];
    CUDA_TRY(c, cudaMemcpyAsync(h, out2, sizeof h, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    sum2 += h[0] * h[0];
    mx = std::fmax(mx, h[1]);
  }
  if (l2) *l2 = std::sqrt(sum2);
  if (linf) *linf = mx;
  if (!std::isfinite(sum2) || !std::isfinite(mx)) return fail(PINT_ERR_NUMERIC, "non-finite residual");
  return PINT_OK;
}

pint_status pint_residual_norm(pint_ctx *c, double *l2, double *linf) {
  if (!c) return fail(PINT_ERR_INVALID, "ctx is NULL");
  BIND_DEVICE(c);
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  Buffers b = buffers(c);
  double *out2 = (double *)(c->work + c->lay.off_red) + 148 * 8 * 2;
  if (c->P > 1) {
    if (c->loopback) return fail(PINT_ERR_STATE, "loopback (virtual-rank) context: use pint_group_residual_norm");
    CUDA_TRY(c, launch_halo_pack(c->g, b, hsend(c), c->stream));
    pint_status st = nccl_halo(c);
    if (st != PINT_OK) return st;
  }
  CUDA_TRY(c, launch_residual_norm(c->g, c->st, b, out2, c->stream));
  if (c->P > 1) {  // global: sum of squares and max over ranks
    double *sq = out2 + 2;
    CUDA_TRY(c, launch_square_first(out2, sq, c->stream));
    ncclResult_t r = ncclGroupStart();
    if (r == ncclSuccess) r = ncclAllReduce(sq, sq, 1, ncclDouble, ncclSum, c->comm, c->stream);
    if (r == ncclSuccess) r = ncclAllReduce(out2 + 1, out2 + 1, 1, ncclDouble, ncclMax, c->comm, c->stream);
    ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess) { c->poisoned = true; return fail(PINT_ERR_NCCL, "residual allreduce"); }
    CUDA_TRY(c, launch_sqrt_into(sq, out2, c->stream));
  }
  double h[2];
  CUDA_TRY(c, cudaMemcpyAsync(h, out2, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  PINT_SYNC(c);
  if (l2) *l2 = h[0];
  if (linf) *linf = h[1];
  if (!std::isfinite(h[0]) || !std::isfinite(h[1])) return fail(PINT_ERR_NUMERIC, "non-finite residual");
  return PINT_OK;
}

pint_status pint_get_iterate(pint_ctx *c, double *u_host) {
  if (!c || !u_host) return fail(PINT_ERR_INVALID, "NULL argument");
  BIND_DEVICE(c);
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  if (c->hermitian) {   // real storage: the first L M N doubles, expanded to (re, 0)
    const size_t n = (size_t)c->g.L * c->g.M * c->g.N;
    CUDA_TRY(c, cudaMemcpyAsync(u_host, c->u, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    PINT_SYNC(c);
    for (size_t i = n; i-- > 0;) {   // back to front: u_host[2i] never overwrites an unread u_host[j > i]
      u_host[2 * i] = u_host[i];
      u_host[2 * i + 1] = 0.0;
    }
    return PINT_OK;
  }
  CUDA_TRY(c, cudaMemcpyAsync(u_host, c->u, c->lay.vec_bytes, cudaMemcpyDeviceToHost, c->stream));
  PINT_SYNC(c);
  return PINT_OK;
}

pint_status pint_get_final_value(pint_ctx *c, double *u_host) {
  if (!c || !u_host) return fail(PINT_ERR_INVALID, "NULL argument");
  BIND_DEVICE(c);
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  const size_t off = ((size_t)(c->g.L - 1) * c->g.M + (c->g.M - 1)) * c->g.N;
  if (c->hermitian) {
    const size_t n = (size_t)c->g.N;
    CUDA_TRY(c, cudaMemcpyAsync(u_host, (const double *)c->u + off, n * sizeof(double), cudaMemcpyDeviceToHost,
                                c->stream));
    PINT_SYNC(c);
    for (size_t i = n; i-- > 0;) {
      u_host[2 * i] = u_host[i];
      u_host[2 * i + 1] = 0.0;
    }
    return PINT_OK;
  }
  CUDA_TRY(c, cudaMemcpyAsync(u_host, c->u + off, (size_t)c->g.N * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
  PINT_SYNC(c);
  return PINT_OK;
}

pint_status pint_set_initial_value(pint_ctx *c, const double *u0_host, int32_t reset_iterate) {
  if (!c || !u0_host) return fail(PINT_ERR_INVALID, "NULL argument");
  BIND_DEVICE(c);
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  for (size_t i = 0; i < 2 * (size_t)c->g.N; ++i)
    if (!std::isfinite(u0_host[i])) return fail(PINT_ERR_NUMERIC, "u0 has a non-finite entry");
  if (c->hermitian)
    for (int n = 0; n < c->g.N; ++n)
      if (u0_host[2 * n + 1] != 0.0) return fail(PINT_ERR_INVALID, "Hermitian mode needs a real u0");
  c->u0.assign(u0_host, u0_host + 2 * (size_t)c->g.N);
  CUDA_TRY(c, cudaMemcpyAsync((void *)c->st.u0, u0_host, (size_t)c->g.N * sizeof(double2), cudaMemcpyHostToDevice, c->stream));
  if (reset_iterate) {
    CUDA_TRY(c, launch_init_iterate(c->g, c->st, buffers(c), c->stream));
    c->k = 0;
  }
  return PINT_OK;
}

pint_status pint_next_window(pint_ctx *c) {
  if (!c) return fail(PINT_ERR_INVALID, "ctx is NULL");
  BIND_DEVICE(c);
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  if (c->P != 1) return fail(PINT_ERR_INVALID, "windowed stepping is single-rank only");
  const Geometry &g = c->g;
  if (c->hermitian) {   // real storage: u0 := (u_{L-1, M-1}, 0) through the host copy
    pint_status st = pint_get_final_value(c, c->u0.data());
    if (st != PINT_OK) return st;
    CUDA_TRY(c, cudaMemcpyAsync((void *)c->st.u0, c->u0.data(), (size_t)g.N * sizeof(double2),
                                cudaMemcpyHostToDevice, c->stream));
  } else {
    const double2 *last = c->u + ((size_t)(g.L - 1) * g.M + (g.M - 1)) * g.N;
    CUDA_TRY(c, cudaMemcpyAsync((void *)c->st.u0, last, (size_t)g.N * sizeof(double2), cudaMemcpyDeviceToDevice,
                                c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->u0.data(), last, (size_t)g.N * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_TRY(c, launch_init_iterate(c->g, c->st, buffers(c), c->stream));
  PINT_SYNC(c);
  c->k = 0;
  return PINT_OK;
}

pint_status pint_destroy(pint_ctx *c) {
  if (c && c->comm) ncclCommDestroy(c->comm);
  if (c) {
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    for (cudaEvent_t e : c->tev) if (e) cudaEventDestroy(e);
    if (c->commstream_owned) cudaStreamDestroy(c->commstream);
  }
  delete c;
  return PINT_OK;
}

pint_status pint_graph_create(pint_ctx *c, int32_t n_iter, void **graph_exec) {
  if (!c || !graph_exec || n_iter < 1) return fail(PINT_ERR_INVALID, "NULL argument or n_iter < 1");
  BIND_DEVICE(c);
  *graph_exec = nullptr;
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  if (c->P > 1) return fail(PINT_ERR_INVALID, "graph capture: one rank (the NCCL calls are not captured here)");
  if (c->k + n_iter > (int)c->alphas.size())
    return fail(PINT_ERR_SCHEDULE, "alpha schedule exhausted (call pint_set_alpha_schedule)");
  cudaGraph_t graph = nullptr;
  CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  pint_status st = PINT_OK;
  for (int i = 0; i < n_iter && st == PINT_OK; ++i) {
    st = run_iteration(c, c->k, nullptr);
    if (st == PINT_OK) c->k++;
  }
  cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
  if (st != PINT_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (e != cudaSuccess) { c->poisoned = true; return fail(PINT_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(e)); }
  cudaGraphExec_t ex = nullptr;
  e = cudaGraphInstantiate(&ex, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(PINT_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
  *graph_exec = (void *)ex;
  return PINT_OK;
}

pint_status pint_graph_launch(pint_ctx *c, void *graph_exec) {
  if (!c || !graph_exec) return fail(PINT_ERR_INVALID, "NULL argument");
  BIND_DEVICE(c);
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  CUDA_TRY(c, cudaGraphLaunch((cudaGraphExec_t)graph_exec, c->stream));
  return PINT_OK;
}

pint_status pint_graph_destroy(void *graph_exec) {
  if (graph_exec && cudaGraphExecDestroy((cudaGraphExec_t)graph_exec) != cudaSuccess)
    return fail(PINT_ERR_CUDA, "cudaGraphExecDestroy failed");
  return PINT_OK;
}

pint_status pint_set_phase_timing(pint_ctx *c, int32_t on) {
  if (!c) return fail(PINT_ERR_INVALID, "ctx is NULL");
  BIND_DEVICE(c);
  if (c->P == 1 || !c->comm) return fail(PINT_ERR_INVALID, "phase timing: NCCL ranks (nranks > 1) only");
  if (on && !c->tev[0])
    for (auto &e : c->tev) CUDA_TRY(c, cudaEventCreate(&e));
  c->phase_timing = on != 0;
  return PINT_OK;
}

pint_status pint_phase_times(pint_ctx *c, double *ms) {
  if (!c || !ms) return fail(PINT_ERR_INVALID, "NULL argument");
  BIND_DEVICE(c);
  if (!c->phase_timing) return fail(PINT_ERR_STATE, "phase timing is off (pint_set_phase_timing)");
  CUDA_TRY(c, cudaEventSynchronize(c->tev[7]));
  float t[7];
  const int from[7] = {0, 1, 3, 2, 5, 2, 0}, to[7] = {1, 2, 4, 5, 7, 6, 7};
  for (int i = 0; i < 7; ++i) CUDA_TRY(c, cudaEventElapsedTime(&t[i], c->tev[from[i]], c->tev[to[i]]));
  for (int i = 0; i < 7; ++i) ms[i] = t[i];
  return PINT_OK;
}

pint_status pint_iterate_profiled(pint_ctx *c, int32_t n_iter, double *kernel_ms) {
  if (!c || !kernel_ms) return fail(PINT_ERR_INVALID, "NULL argument");
  BIND_DEVICE(c);
  if (c->P > 1) return fail(PINT_ERR_INVALID, "per-launch profiling is single-rank only");
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  if (c->k + n_iter > (int)c->alphas.size())
    return fail(PINT_ERR_SCHEDULE, "alpha schedule exhausted (call pint_set_alpha_schedule)");
  const int nk = pint_launches_per_iteration(c);
  std::vector<cudaEvent_t> ev(nk + 1);
  for (auto &e : ev) CUDA_TRY(c, cudaEventCreate(&e));
  for (int i = 0; i < nk; ++i) kernel_ms[i] = 0.0;
  pint_status st = PINT_OK;
  for (int it = 0; it < n_iter && st == PINT_OK; ++it) {
    Recorder r{ev.data() + 1, 0, nk};
    CUDA_TRY(c, cudaEventRecord(ev[0], c->stream));
    set_recorder(&r);
    st = run_iteration(c, c->k, nullptr);
    set_recorder(nullptr);
    if (st != PINT_OK) break;
    c->k++;
    CUDA_TRY(c, cudaEventSynchronize(ev[nk]));
    for (int i = 0; i < nk; ++i) {
      float ms = 0.f;
      CUDA_TRY(c, cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      kernel_ms[i] += ms;
    }
  }
  for (auto &e : ev) cudaEventDestroy(e);
  if (st == PINT_OK && n_iter > 0)
    for (int i = 0; i < nk; ++i) kernel_ms[i] /= n_iter;
  return st;
}

const char *pint_kernel_name(pint_ctx *c, int32_t i) {
  if (!c) return "";
  if (c->form == PINT_FORM_DIRECT) return kernel_name_direct(c->g, c->lc, c->st, i);
  return kernel_name(c->g, c->lc, c->st, i);
}

int32_t pint_launches_per_iteration(pint_ctx *c) {
  if (!c) return -1;
  if (c->form == PINT_FORM_DIRECT) return launches_per_iteration_direct(c->g, c->lc, c->st);
  return launches_per_iteration(c->g, c->lc, c->st);
}

pint_status pint_set_form(pint_ctx *c, int32_t form) {
  if (!c) return fail(PINT_ERR_INVALID, "ctx is NULL");
  if (form != PINT_FORM_CORRECTION && form != PINT_FORM_DIRECT) return fail(PINT_ERR_INVALID, "unknown form");
  if (form == PINT_FORM_DIRECT && c->st.v) return fail(PINT_ERR_INVALID, "the direct form assumes b == 0");
  if (form == PINT_FORM_DIRECT && !c->g.pow2)
    return fail(PINT_ERR_INVALID, "non-power-of-two grids: correction form only (generic path)");
  c->form = form;
  return PINT_OK;
}

pint_status pint_set_hermitian(pint_ctx *c, int32_t on) {
  if (!c) return fail(PINT_ERR_INVALID, "ctx is NULL");
  BIND_DEVICE(c);
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  const Geometry &g = c->g;
  if (on) {
    if (!g.pow2) return fail(PINT_ERR_INVALID, "Hermitian mode: power-of-two grids only");
    if (g.dim == 2 && (!reg2d_path(g) || g.ny < 2))
      return fail(PINT_ERR_INVALID, "Hermitian mode: 2-D grids of the register FFT engine, 4 <= L <= 1024, only");
    if (g.dim == 1 && (g.N < 8 || g.L < 2)) return fail(PINT_ERR_INVALID, "Hermitian mode needs N >= 8 and L >= 2");
    if (c->P != 1) return fail(PINT_ERR_INVALID, "Hermitian mode is single-rank only");
    if (c->st.v) return fail(PINT_ERR_INVALID, "Hermitian mode assumes b == 0");
    for (int n = 0; n < g.N; ++n)
      if (c->u0[2 * n + 1] != 0.0) return fail(PINT_ERR_INVALID, "Hermitian mode needs a real u0");
  }
  // slot p holds frequency k = bitrev(p) (1 rank).  Units: the slots with k <= L/2 in slot order.
  std::vector<int> sym(2 * (size_t)g.L, 0);
  int ns = 0;
  if (!on) {
    for (int p = 0; p < g.L; ++p) { sym[p] = p; sym[g.L + p] = p; }
    ns = g.L;
  } else {
    std::vector<int> unit_of_k(g.L, -1);
    for (int p = 0; p < g.L; ++p) {
      const int k = bitrev(p, g.logL);
      if (k <= g.L / 2) { unit_of_k[k] = ns; sym[ns++] = p; }
    }
    for (int p = 0; p < g.L; ++p) {
      const int k = bitrev(p, g.logL);
      sym[g.L + p] = k <= g.L / 2 ? unit_of_k[k] : -1 - unit_of_k[g.L - k];
    }
  }
  int *dsym = (int *)(c->work + c->lay.off_sym);
  CUDA_TRY(c, cudaMemcpyAsync(dsym, sym.data(), sym.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
  PINT_SYNC(c);
  c->st.nsolve = ns;
  c->st.packed = on ? 1 : 0;
  c->st.xpair = on && hermitian_pipe_path(g) ? 1 : 0;
  if ((on != 0) != c->hermitian) {
    // iterate storage: real fp64 in the Hermitian mode (its imaginary parts are zero in exact
    // arithmetic; roundoff-level ones are dropped), complex128 otherwise
    CUDA_TRY(c, launch_storage_convert(g, buffers(c), on != 0, c->stream));
    PINT_SYNC(c);
  }
  c->hermitian = on != 0;
  return PINT_OK;
}

pint_status pint_solve(pint_ctx *c, double m0, double eps, double tau, double tol, int32_t max_iter,
                       int32_t *iters, double *diffs, double *m_out, int32_t *stop_reason) {
  if (!c || !iters) return fail(PINT_ERR_INVALID, "NULL argument");
  if (!(m0 > 0) || !(tol > 0) || max_iter < 1 || max_iter > PINT_MAX_SCHEDULE || !(eps >= 0) || !(tau >= 0))
    return fail(PINT_ERR_INVALID, "need m0 > 0, tol > 0, eps, tau >= 0, 1 <= max_iter <= PINT_MAX_SCHEDULE");
  double w_inf = 0;   // ||w||_inf of the assembled w, forcing included
  {
    pint_status sw = pint_w_inf(c, &w_inf);
    if (sw != PINT_OK) return sw;
  }
  const ld gam = (ld)c->prob.L * (3.0L * eps + tau) * w_inf;          // Alg. 2 line 1
  if (!(gam > 0)) return fail(PINT_ERR_INVALID, "gamma = L(3 eps + tau)||w||_inf must be > 0");
  std::vector<double> alphas, ms{m0};
  int reason = 2;
  ld mk = m0;
  while ((int)alphas.size() < max_iter) {
    if (mk <= tol) { reason = 1; break; }                              // while m_k > tol
    if (4 * gam > mk) { reason = 3; break; }                           // alpha would exceed 1/2
    alphas.push_back((double)sqrtl(gam / mk));                         // alpha_{k+1} = sqrt(gamma/m_k)
    mk = 2 * sqrtl(mk * gam);                                          // m_{k+1} = 2 sqrt(m_k gamma)
    ms.push_back((double)mk);
  }
  *iters = 0;
  if (!alphas.empty()) {
    pint_status st = pint_set_alpha_schedule(c, alphas.data(), (int32_t)alphas.size());
    if (st != PINT_OK) return st;
  }
  for (size_t i = 0; i < alphas.size(); ++i) {
    double d = 0;
    pint_status st = pint_iterate(c, 1, &d);
    if (st != PINT_OK) return st;
    if (diffs) diffs[i] = d;
    *iters = (int32_t)i + 1;
    if (d <= tol) { reason = 0; break; }                              // ||u_L^{k+1} - u_L^k|| <= tol
  }
  if (m_out)
    for (int i = 0; i <= *iters; ++i) m_out[i] = ms[i];
  if (stop_reason) *stop_reason = reason;
  return PINT_OK;
}

pint_status pint_set_forcing(pint_ctx *c, const void *v_dev) {
  if (!c) return fail(PINT_ERR_INVALID, "ctx is NULL");
  if (((uintptr_t)v_dev) % 16) return fail(PINT_ERR_INVALID, "v_dev must be 16-byte aligned");
  if (v_dev && c->form == PINT_FORM_DIRECT) return fail(PINT_ERR_INVALID, "forcing needs the correction form");
  if (v_dev && c->hermitian) return fail(PINT_ERR_INVALID, "forcing is not combinable with the Hermitian mode");
  c->st.v = (const double2 *)v_dev;
  return PINT_OK;
}

pint_status pint_sequential(pint_ctx *c) {
  if (!c) return fail(PINT_ERR_INVALID, "ctx is NULL");
  BIND_DEVICE(c);
  if (c->st.v) return fail(PINT_ERR_INVALID, "the sequential baseline assumes b == 0");
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  const Geometry &g = c->g;
  if (c->P != 1 || !g.pow2 || (g.dim == 2 && !reg2d_path(g)))
    return fail(PINT_ERR_INVALID, "sequential baseline: power-of-two grids (2-D: of the spatial pipeline), one rank");
  if (c->hermitian) return fail(PINT_ERR_INVALID, "sequential baseline: complex storage only (pint_set_hermitian(0))");
  const int M = g.M;
  // Q = V diag(lambda) V^{-1} (Radau IIA): step l solves (I - dT Q (x) A) U_l = 1 (x) u_{l-1,M-1}
  // as z_m = (V^{-1} 1)_m (I - dT lambda_m A)^{-1} u_{l-1,M-1}, U_l = (V (x) I) z
  std::vector<cld> B((size_t)M * M), lam, S, Si;
  for (int i = 0; i < M * M; ++i) B[i] = c->Q[i];
  ld cond, gap;
  if (!eig_diagonalize(M, B, lam, S, Si, cond, gap)) return fail(PINT_ERR_NOT_DIAGONALIZABLE, "Q not diagonalisable");
  const ld dT = (ld)c->prob.T / c->prob.L;
  const size_t npcr = g.dim == 1 ? (size_t)M * g.logN * g.nfac * 2 : 0;
  std::vector<double2> tab(2 * M + M * M + npcr + (g.dim == 1 ? M : 0));
  AxisStencil sx;
  if (g.dim == 1) axis_stencil(c->prob.op, g.nx, op_is_heat(c->prob.op) ? c->prob.nu : c->prob.cx, sx);
  for (int m = 0; m < M; ++m) {
    cld rs = 0;
    for (int j = 0; j < M; ++j) rs += Si[(size_t)m * M + j];
    tab[m] = make_double2((double)rs.real(), (double)rs.imag());                       // sig
    const cld sh = lam[m] * dT;
    tab[M + m] = make_double2((double)sh.real(), (double)sh.imag());                   // shift
    for (int j = 0; j < M; ++j) {
      const cld v = S[(size_t)m * M + j];
      tab[2 * M + m * M + j] = make_double2((double)v.real(), (double)v.imag());       // V
    }
    if (g.dim == 1) {   // PCR tables of the shifted system I - dT lambda_m A (line m)
      std::string ferr;
      if (!pcr_tables(c, sx, sh, tab.data() + 2 * M + M * M + (size_t)m * g.logN * g.nfac * 2,
                      tab.data() + 2 * M + M * M + npcr + m, ferr))
        return fail(PINT_ERR_NUMERIC, "sequential baseline: 1-D spatial factorisation failed: " + ferr);
    }
  }
  double2 *dtab = (double2 *)(c->work + c->lay.off_seq);
  CUDA_TRY(c, cudaMemcpyAsync(dtab, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice, c->stream));
  AlphaTables at{};
  at.sig = dtab;
  at.shift = dtab + M;
  at.SG = dtab + 2 * M;
  if (g.dim == 1) {
    at.pcr = dtab + 2 * M + M * M;
    at.inv_e = dtab + 2 * M + M * M + npcr;
  }
  StaticTables st = c->st;       // one "slot" (slot 0) per step, never packed
  st.nsolve = 1;
  st.packed = 0;
  Buffers b = buffers(c);
  double2 *r0 = (double2 *)(c->work + c->lay.off_r0);
  for (int l = 0; l < g.L; ++l) {
    const double2 *prev = l == 0 ? c->st.u0 : c->u + ((size_t)(l - 1) * M + (M - 1)) * g.N;
    CUDA_TRY(c, cudaMemcpyAsync(r0, prev, (size_t)g.N * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
    if (g.dim == 1)
      CUDA_TRY(c, launch_sequential_step_1d(g, c->lc, st, at, b, r0, c->u + (size_t)l * M * g.N, c->stream));
    else
      CUDA_TRY(c, launch_sequential_step(g, st, at, b, r0, c->u + (size_t)l * M * g.N, c->stream));
  }
  PINT_SYNC(c);
  return PINT_OK;
}

pint_status pint_get_factors(pint_ctx *c, int32_t a, int32_t k, double *d_k, double *S, double *Sinv,
                             double *d_km) {
  if (!c || a < 0 || a >= (int)c->h_S.size() || k < 0 || k >= c->prob.L)
    return fail(PINT_ERR_INVALID, "bad schedule entry / frequency");
  const int M = c->g.M;
  if (d_k) { d_k[0] = (double)c->h_dk[a][k].real(); d_k[1] = (double)c->h_dk[a][k].imag(); }
  for (int i = 0; i < M * M; ++i) {
    if (S) { S[2 * i] = (double)c->h_S[a][(size_t)k * M * M + i].real(); S[2 * i + 1] = (double)c->h_S[a][(size_t)k * M * M + i].imag(); }
    if (Sinv) { Sinv[2 * i] = (double)c->h_Sinv[a][(size_t)k * M * M + i].real(); Sinv[2 * i + 1] = (double)c->h_Sinv[a][(size_t)k * M * M + i].imag(); }
  }
  if (d_km)
    for (int m = 0; m < M; ++m) { d_km[2 * m] = (double)c->h_dkm[a][(size_t)k * M + m].real(); d_km[2 * m + 1] = (double)c->h_dkm[a][(size_t)k * M + m].imag(); }
  return PINT_OK;
}

pint_status pint_debug_stage(pint_ctx *c, int32_t a, int32_t s) {
  if (!c || a < 0 || a >= (int)c->at.size()) return fail(PINT_ERR_INVALID, "bad schedule entry");
  BIND_DEVICE(c);
  if (c->P > 1) return fail(PINT_ERR_INVALID, "debug stages are single-rank only");
  if (c->poisoned) return fail(PINT_ERR_STATE, "context poisoned by an earlier CUDA error");
  Buffers b = buffers(c);
  const AlphaTables &at = c->at[a];
  if (s == 0) CUDA_TRY(c, launch_forward(c->g, c->lc, c->st, at, b, c->stream));
  else if (s == 1) { double2 *x2; CUDA_TRY(c, launch_solve(c->g, c->lc, c->st, at, b, c->stream, &x2)); }
  else if (s == 2) {
    double2 *x2 = (c->g.dim == 1 && c->lc.pcr_mode == 1) ? b.Y : b.X;
    CUDA_TRY(c, launch_backward(c->g, c->lc, c->st, at, b, x2, nullptr, c->stream, 0));
  } else return fail(PINT_ERR_INVALID, "stage must be 0, 1 or 2");
  PINT_SYNC(c);
  return PINT_OK;
}

pint_status pint_debug_get_work(pint_ctx *c, int32_t which, double *host) {
  if (!c || !host) return fail(PINT_ERR_INVALID, "NULL argument");
  BIND_DEVICE(c);
  Buffers b = buffers(c);
  const double2 *src = which == 0 ? b.X : ((c->g.dim == 1 && c->lc.pcr_mode == 1) ? b.Y : b.X);
  CUDA_TRY(c, cudaMemcpyAsync(host, src, c->lay.vec_bytes, cudaMemcpyDeviceToHost, c->stream));
  PINT_SYNC(c);
  return PINT_OK;
}

}  // extern "C"
