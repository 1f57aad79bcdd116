// Host numerics of libpint in long double (see host_numerics.h).
#include "host_numerics.h"
#include "pint.h"

#include <algorithm>
#include <cmath>

namespace pint {

static const ld kPi = 3.141592653589793238462643383279502884L;

cld unit_root(long long q, long long n, int sign) {
  q %= n;
  if (q < 0) q += n;
  // exact values at the quarter points, long double sin/cos elsewhere (index already reduced)
  if (q == 0) return cld(1, 0);
  if (2 * q == n) return cld(-1, 0);
  if (4 * q == n) return cld(0, sign);
  if (4 * q == 3 * n) return cld(0, -sign);
  ld ang = 2 * kPi * (ld)q / (ld)n;
  return cld(cosl(ang), sign * sinl(ang));
}

// ---------------------------------------------------------------------------------------------
// Radau IIA tableau

// R_M(x) = P_{M-1}(x) + P_M(x) and its derivative via the Legendre three-term recurrence
static void radau_poly(int M, ld x, ld &f, ld &df) {
  // P_0 = 1, P_1 = x, (k+1) P_{k+1} = (2k+1) x P_k - k P_{k-1}
  ld p0 = 1, p1 = x, d0 = 0, d1 = 1;
  ld pm1 = 1, dm1 = 0;  // P_{M-1}
  ld pm = x, dm = 1;    // P_M
  if (M == 1) { pm1 = 1; dm1 = 0; pm = x; dm = 1; }
  else {
    for (int k = 1; k < M; ++k) {
      ld p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
      ld d2 = ((2 * k + 1) * (p1 + x * d1) - k * d0) / (k + 1);
      p0 = p1; p1 = p2; d0 = d1; d1 = d2;
    }
    pm = p1; dm = d1; pm1 = p0; dm1 = d0;
  }
  f = pm1 + pm;
  df = dm1 + dm;
}

bool radau_tableau(int M, std::vector<ld> &t, std::vector<ld> &Q) {
  if (M < 1) return false;
  // roots of R_M on [-1, 1]: x = -1 exactly, the other M-1 by Newton with deflation from
  // Chebyshev-like guesses (interior roots interlace with the Chebyshev-Gauss-Radau points)
  std::vector<ld> x;
  x.push_back(-1.0L);
  for (int i = 1; i < M; ++i) {
    ld xi = -cosl(kPi * (2 * i) / (2 * M - 1));
    for (int it = 0; it < 200; ++it) {
      ld f, df;
      radau_poly(M, xi, f, df);
      // deflate known roots: g = f / prod(x - r);  g'/g = f'/f - sum 1/(x - r)
      ld s = 0;
      for (ld r : x) s += 1.0L / (xi - r);
      ld step = f / (df - f * s);
      xi -= step;
      if (fabsl(step) < 1e-19L) break;
    }
    x.push_back(xi);
  }
  t.resize(M);
  for (int i = 0; i < M; ++i) t[i] = (1.0L - x[i]) / 2.0L;   // x = -2t + 1
  std::sort(t.begin(), t.end());
  t[M - 1] = 1.0L;
  for (int i = 1; i < M; ++i)
    if (!(t[i] > t[i - 1])) return false;
  if (!(t[0] > 0)) return false;
  // Q[m][i] = int_0^{t_m} l_i(s) ds by exact integration of the monomial expansion
  Q.assign((size_t)M * M, 0.0L);
  for (int i = 0; i < M; ++i) {
    std::vector<ld> c(1, 1.0L);  // coefficients low -> high
    ld den = 1;
    for (int j = 0; j < M; ++j) {
      if (j == i) continue;
      std::vector<ld> nc(c.size() + 1, 0.0L);
      for (size_t k = 0; k < c.size(); ++k) {
        nc[k + 1] += c[k];
        nc[k] -= c[k] * t[j];
      }
      c.swap(nc);
      den *= (t[i] - t[j]);
    }
    for (int m = 0; m < M; ++m) {
      ld acc = 0, tp = t[m];
      for (size_t k = 0; k < c.size(); ++k) { acc += c[k] / (k + 1) * tp; tp *= t[m]; }
      Q[(size_t)m * M + i] = acc / den;
    }
  }
  return true;
}

// ---------------------------------------------------------------------------------------------
// Algorithm 2

bool adaptive_schedule(int L, double w_inf, double m0, double eps, double tau, int K,
                       std::vector<double> &alpha, std::vector<double> &m, std::string &err) {
  ld g = (ld)L * (3.0L * eps + tau) * w_inf;
  if (!(g > 0)) { err = "gamma = L(3 eps + tau)||w||_inf must be > 0"; return false; }
  if (!(m0 > 0)) { err = "m0 must be > 0"; return false; }
  alpha.clear();
  m.clear();
  ld mk = m0;
  m.push_back((double)mk);
  for (int k = 0; k < K; ++k) {
    if (4 * g > mk) { err = "m_k < 4 gamma: alpha would exceed 1/2 (P:399-401)"; return false; }
    alpha.push_back((double)sqrtl(g / mk));
    mk = 2 * sqrtl(mk * g);
    m.push_back((double)mk);
  }
  return true;
}

// ---------------------------------------------------------------------------------------------
// small complex linear algebra

bool invert(int n, std::vector<cld> &A) {
  std::vector<cld> I((size_t)n * n, cld(0));
  for (int i = 0; i < n; ++i) I[(size_t)i * n + i] = 1;
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::abs(A[(size_t)r * n + col]) > std::abs(A[(size_t)piv * n + col])) piv = r;
    if (std::abs(A[(size_t)piv * n + col]) == 0) return false;
    if (piv != col)
      for (int k = 0; k < n; ++k) {
        std::swap(A[(size_t)piv * n + k], A[(size_t)col * n + k]);
        std::swap(I[(size_t)piv * n + k], I[(size_t)col * n + k]);
      }
    cld inv = 1.0L / A[(size_t)col * n + col];
    for (int k = 0; k < n; ++k) { A[(size_t)col * n + k] *= inv; I[(size_t)col * n + k] *= inv; }
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      cld f = A[(size_t)r * n + col];
      if (f == cld(0)) continue;
      for (int k = 0; k < n; ++k) {
        A[(size_t)r * n + k] -= f * A[(size_t)col * n + k];
        I[(size_t)r * n + k] -= f * I[(size_t)col * n + k];
      }
    }
  }
  A.swap(I);
  return true;
}

// LU solve with partial pivoting (copies A)
static bool lu_solve(int n, std::vector<cld> A, std::vector<cld> &b) {
  std::vector<int> p(n);
  for (int i = 0; i < n; ++i) p[i] = i;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::abs(A[(size_t)r * n + c]) > std::abs(A[(size_t)piv * n + c])) piv = r;
    if (std::abs(A[(size_t)piv * n + c]) == 0) return false;
    if (piv != c) {
      for (int k = 0; k < n; ++k) std::swap(A[(size_t)piv * n + k], A[(size_t)c * n + k]);
      std::swap(b[piv], b[c]);
    }
    for (int r = c + 1; r < n; ++r) {
      cld f = A[(size_t)r * n + c] / A[(size_t)c * n + c];
      for (int k = c; k < n; ++k) A[(size_t)r * n + k] -= f * A[(size_t)c * n + k];
      b[r] -= f * b[c];
    }
  }
  for (int r = n - 1; r >= 0; --r) {
    cld s = b[r];
    for (int k = r + 1; k < n; ++k) s -= A[(size_t)r * n + k] * b[k];
    b[r] = s / A[(size_t)r * n + r];
  }
  return true;
}

// eigenvalues of a complex matrix: Hessenberg reduction + Wilkinson-shifted QR (Givens)
static bool eigenvalues(int n, std::vector<cld> H, std::vector<cld> &lam) {
  auto at = [&](int i, int j) -> cld & { return H[(size_t)i * n + j]; };
  // Householder reduction to upper Hessenberg
  for (int k = 0; k + 2 < n; ++k) {
    ld alpha2 = 0;
    for (int i = k + 1; i < n; ++i) alpha2 += std::norm(at(i, k));
    ld alpha = sqrtl(alpha2);
    if (alpha == 0) continue;
    cld x0 = at(k + 1, k);
    cld ph = (std::abs(x0) == 0) ? cld(1) : x0 / std::abs(x0);
    std::vector<cld> v(n, cld(0));
    v[k + 1] = x0 + ph * alpha;
    for (int i = k + 2; i < n; ++i) v[i] = at(i, k);
    ld vn = 0;
    for (int i = k + 1; i < n; ++i) vn += std::norm(v[i]);
    if (vn == 0) continue;
    // H = (I - 2 v v^H / vn) H (I - 2 v v^H / vn)
    for (int j = 0; j < n; ++j) {
      cld s = 0;
      for (int i = k + 1; i < n; ++i) s += std::conj(v[i]) * at(i, j);
      s *= 2.0L / vn;
      for (int i = k + 1; i < n; ++i) at(i, j) -= v[i] * s;
    }
    for (int i = 0; i < n; ++i) {
      cld s = 0;
      for (int j = k + 1; j < n; ++j) s += at(i, j) * v[j];
      s *= 2.0L / vn;
      for (int j = k + 1; j < n; ++j) at(i, j) -= s * std::conj(v[j]);
    }
  }
  lam.assign(n, cld(0));
  int hi = n - 1;
  int iter = 0;
  const ld eps = 1e-19L;
  while (hi >= 0) {
    if (hi == 0) { lam[0] = at(0, 0); break; }
    int lo = hi;
    while (lo > 0) {
      ld s = std::abs(at(lo, lo)) + std::abs(at(lo - 1, lo - 1));
      if (s == 0) s = 1;
      if (std::abs(at(lo, lo - 1)) <= eps * s) { at(lo, lo - 1) = 0; break; }
      --lo;
    }
    if (lo == hi) { lam[hi] = at(hi, hi); --hi; iter = 0; continue; }
    if (++iter > 500) return false;
    // Wilkinson shift from the trailing 2x2 of the active block
    cld a = at(hi - 1, hi - 1), b = at(hi - 1, hi), c = at(hi, hi - 1), d = at(hi, hi);
    cld tr = a + d, det = a * d - b * c;
    cld disc = std::sqrt(tr * tr / 4.0L - det);
    cld mu1 = tr / 2.0L + disc, mu2 = tr / 2.0L - disc;
    cld mu = (std::abs(mu1 - d) < std::abs(mu2 - d)) ? mu1 : mu2;
    if (iter % 11 == 10) mu = d + cld(std::abs(c), 0);  // exceptional shift
    // QR step on rows/cols lo..hi of (H - mu I) with Givens rotations
    std::vector<cld> cs(hi - lo), sn(hi - lo);
    for (int i = lo; i <= hi; ++i) at(i, i) -= mu;
    for (int k = lo; k < hi; ++k) {
      cld x = at(k, k), y = at(k + 1, k);
      ld r = sqrtl(std::norm(x) + std::norm(y));
      cld cc = (r == 0) ? cld(1) : x / r, ss = (r == 0) ? cld(0) : y / r;
      cs[k - lo] = cc; sn[k - lo] = ss;
      // apply G^H = [[conj(c), conj(s)], [-s, c]] to rows k, k+1
      for (int j = k; j < n; ++j) {
        cld h1 = at(k, j), h2 = at(k + 1, j);
        at(k, j) = std::conj(cc) * h1 + std::conj(ss) * h2;
        at(k + 1, j) = -ss * h1 + cc * h2;
      }
    }
    for (int k = lo; k < hi; ++k) {
      cld cc = cs[k - lo], ss = sn[k - lo];
      // apply G on the right to columns k, k+1
      for (int i = 0; i <= std::min(hi, k + 2); ++i) {
        cld h1 = at(i, k), h2 = at(i, k + 1);
        at(i, k) = h1 * cc + h2 * ss;
        at(i, k + 1) = -h1 * std::conj(ss) + h2 * std::conj(cc);
      }
    }
    for (int i = lo; i <= hi; ++i) at(i, i) += mu;
  }
  return true;
}

static ld norm1(int n, const std::vector<cld> &A) {
  ld best = 0;
  for (int j = 0; j < n; ++j) {
    ld s = 0;
    for (int i = 0; i < n; ++i) s += std::abs(A[(size_t)i * n + j]);
    best = std::max(best, s);
  }
  return best;
}

bool eig_diagonalize(int n, const std::vector<cld> &B, std::vector<cld> &lam, std::vector<cld> &S,
                     std::vector<cld> &Sinv, ld &cond, ld &gap) {
  cond = INFINITY;
  gap = 0;
  if (!eigenvalues(n, B, lam)) return false;
  std::sort(lam.begin(), lam.end(), [](const cld &a, const cld &b) {
    if (a.real() != b.real()) return a.real() < b.real();
    return a.imag() < b.imag();
  });
  ld lmax = 0;
  for (auto &l : lam) lmax = std::max(lmax, std::abs(l));
  gap = INFINITY;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) gap = std::min(gap, std::abs(lam[i] - lam[j]));
  if (n == 1) gap = INFINITY;
  // Rayleigh-style refinement of each eigenvalue + eigenvector by inverse iteration
  S.assign((size_t)n * n, cld(0));
  ld bn = norm1(n, B);
  for (int e = 0; e < n; ++e) {
    std::vector<cld> v(n);
    for (int i = 0; i < n; ++i) v[i] = cld(1.0L + 0.1L * i, 0.05L * (i % 3));
    cld shift = lam[e] + cld(bn * 1e-17L, bn * 1e-17L);
    for (int it = 0; it < 4; ++it) {
      std::vector<cld> A = B;
      for (int i = 0; i < n; ++i) A[(size_t)i * n + i] -= shift;
      if (!lu_solve(n, A, v)) break;  // exact eigenvalue hit: v already converged
      ld nv = 0;
      for (auto &z : v) nv += std::norm(z);
      nv = sqrtl(nv);
      for (auto &z : v) z /= nv;
    }
    // normalise: unit 2-norm, largest component real positive (deterministic)
    int imax = 0;
    for (int i = 1; i < n; ++i) if (std::abs(v[i]) > std::abs(v[imax])) imax = i;
    cld ph = std::abs(v[imax]) > 0 ? std::conj(v[imax]) / std::abs(v[imax]) : cld(1);
    ld nv = 0;
    for (auto &z : v) { z *= ph; nv += std::norm(z); }
    nv = sqrtl(nv);
    for (int i = 0; i < n; ++i) S[(size_t)i * n + e] = v[i] / nv;
  }
  Sinv = S;
  if (!invert(n, Sinv)) return false;
  cond = norm1(n, S) * norm1(n, Sinv);
  if (cond > 1e8L) return false;
  if (n > 1 && gap < 1e-8L * lmax) return false;
  return true;
}

void pass_twiddles(int logn, int maxb, std::vector<cld> &out) {
  out.clear();
  const int b0 = logn < maxb ? logn : maxb;
  const int b1 = (logn - b0) < maxb ? (logn - b0) : maxb;
  const int b[3] = {b0, b1, logn - b0 - b1};
  int logm = logn;
  for (int p = 0; p < 3 && b[p] > 0; ++p) {
    const int logs = logm - b[p], s = 1 << logs;
    for (int k = 0; k < b[p]; ++k)
      for (int j = 0; j < s; ++j)
        out.push_back(unit_root(((long long)j << k) & ((1LL << logm) - 1), 1LL << logm, -1));
    logm -= b[p];
  }
}

size_t pass_twiddle_count(int logn, int maxb) {
  std::vector<cld> v;
  pass_twiddles(logn, maxb, v);
  return v.size();
}

// ---------------------------------------------------------------------------------------------
// Spatial operators.  Centred second differences of order 2, 4, 6 and upwind-biased first
// differences of order 1 .. 5 (c > 0; mirrored for c < 0); exact rational weights.

static const ld kD2[3][4] = {{-2.0L, 1.0L, 0, 0},                                   // kappa 2: d_0, d_1
                             {-5.0L / 2, 4.0L / 3, -1.0L / 12, 0},                  // kappa 4
                             {-49.0L / 18, 3.0L / 2, -3.0L / 20, 1.0L / 90}};       // kappa 6
// upwind (c > 0): offsets -3 .. 2 at index o + 3; orders 1, 3, 5 on -(k+1)/2 .. (k-1)/2 and the
// even orders 2, 4 of Table 1 on -(k/2+1) .. k/2-1 (reading R16)
static const ld kD1[5][6] = {{0, 0, -1.0L, 1.0L, 0, 0},
                             {0, 1.0L / 2, -2.0L, 3.0L / 2, 0, 0},
                             {0, 1.0L / 6, -1.0L, 1.0L / 2, 1.0L / 3, 0},
                             {-1.0L / 12, 1.0L / 2, -3.0L / 2, 5.0L / 6, 1.0L / 4, 0},
                             {-2.0L / 60, 15.0L / 60, -1.0L, 20.0L / 60, 30.0L / 60, -3.0L / 60}};

bool op_is_heat(int op) { return op == PINT_OP_HEAT || op == PINT_OP_HEAT4 || op == PINT_OP_HEAT6; }

static int heat_row(int op) { return op == PINT_OP_HEAT ? 0 : op == PINT_OP_HEAT4 ? 1 : 2; }
static bool op_is_upwind(int op) {
  return op == PINT_OP_UPWIND1 || op == PINT_OP_UPWIND2 || op == PINT_OP_UPWIND3 || op == PINT_OP_UPWIND4 ||
         op == PINT_OP_UPWIND5;
}
static int upwind_row(int op) {
  return op == PINT_OP_UPWIND1 ? 0 : op == PINT_OP_UPWIND2 ? 1 : op == PINT_OP_UPWIND3 ? 2 : op == PINT_OP_UPWIND4 ? 3 : 4;
}

bool axis_stencil(int op, long long n, ld coef, AxisStencil &st) {
  st = AxisStencil{};
  const ld nn = (ld)n;
  if (op_is_heat(op)) {
    const int r = heat_row(op), h = r + 1;
    st.h0 = st.h1 = h;
    for (int o = 0; o <= h; ++o) st.w[3 + o] = st.w[3 - o] = coef * nn * nn * kD2[r][o];
    return true;
  }
  if (op == PINT_OP_ADVECTION) {
    st.h0 = st.h1 = 1;
    st.w[2] = coef * nn / 2;
    st.w[4] = -coef * nn / 2;
    return true;
  }
  if (op_is_upwind(op)) {
    const ld *d = kD1[upwind_row(op)];
    const bool mirror = coef < 0;
    st.h0 = st.h1 = 3;
    for (int o = -3; o <= 2; ++o) {
      const int oo = mirror ? -o : o;                     // c < 0: w(o) = -d(-o)
      st.w[3 + oo] = -coef * nn * (mirror ? -d[o + 3] : d[o + 3]);
    }
    // trim to the nonzero offsets
    while (st.h0 > 0 && st.w[3 - st.h0] == 0) --st.h0;
    while (st.h1 > 0 && st.w[3 + st.h1] == 0) --st.h1;
    if (coef == 0) st.h0 = st.h1 = 0;
    return true;
  }
  return false;
}

// sin^2(pi q / n) and sin(2 pi q / n) from the integer-reduced q (no large-argument rounding)
static ld sin2_pi(long long q, long long n) {
  q %= n;
  if (q < 0) q += n;
  const ld sn = sinl(kPi * (ld)q / (ld)n);
  return sn * sn;
}

cld axis_symbol(int op, long long n, long long k, ld coef) {
  AxisStencil st;
  axis_stencil(op, n, coef, st);
  if (op_is_heat(op)) {
    // sum_o w_o e^{i o theta} = -4 sum_{o >= 1} w_o sin^2(o theta / 2)
    ld acc = 0;
    for (int o = 1; o <= st.h1; ++o) acc += st.w[3 + o] * sin2_pi((long long)o * k, n);
    return cld(-4 * acc, 0);
  }
  // sum_o w_o e^{i o theta} = -2 sum_o w_o sin^2(o theta / 2) + i sum_o w_o sin(o theta)
  ld re = 0, im = 0;
  for (int o = -st.h0; o <= st.h1; ++o) {
    if (o == 0) continue;
    re += -2 * st.w[3 + o] * sin2_pi((long long)o * k, n);
    im += st.w[3 + o] * unit_root((long long)o * k, n, +1).imag();
  }
  return cld(re, im);
}

int stencil_factor_count(int op, const AxisStencil &st) {
  if (st.h0 <= 1 && st.h1 <= 1) return 1;
  if (op_is_heat(op)) return st.h1;
  return std::max(st.h0, st.h1);
}

// roots of sum_j p[j] z^j (p[deg] != 0): Durand-Kerner in long double, then Newton polishing
static void poly_roots(const std::vector<cld> &p, std::vector<cld> &r) {
  const int deg = (int)p.size() - 1;
  std::vector<cld> m(deg + 1);
  for (int j = 0; j <= deg; ++j) m[j] = p[j] / p[deg];
  auto eval = [&](cld z, cld *dp) {
    cld v = m[deg], d = 0;
    for (int j = deg - 1; j >= 0; --j) { d = d * z + v; v = v * z + m[j]; }
    if (dp) *dp = d;
    return v;
  };
  ld rad = 0;
  for (int j = 0; j < deg; ++j) rad = std::max(rad, std::pow(std::abs(m[j]), 1.0L / (deg - j)));
  rad = 2 * rad + 1e-3L;
  r.resize(deg);
  for (int i = 0; i < deg; ++i) r[i] = std::polar(rad * (0.4L + 0.1L * i), 0.9L + 2 * kPi * i / deg);
  for (int it = 0; it < 2000; ++it) {
    ld mv = 0;
    for (int i = 0; i < deg; ++i) {
      cld den = 1;
      for (int j = 0; j < deg; ++j) if (j != i) den *= r[i] - r[j];
      const cld dz = eval(r[i], nullptr) / den;
      r[i] -= dz;
      mv = std::max(mv, std::abs(dz) / std::max(1.0L, std::abs(r[i])));
    }
    if (mv < 1e-30L) break;
  }
  for (int i = 0; i < deg; ++i)
    for (int it = 0; it < 4; ++it) {
      cld d;
      const cld v = eval(r[i], &d);
      if (d == cld(0)) break;
      r[i] -= v / d;
    }
}

bool factor_shifted(int op, const AxisStencil &st, cld s, std::vector<TriFactor> &f, cld &lead,
                    std::string &err) {
  f.clear();
  if (st.h0 <= 1 && st.h1 <= 1) {
    // one factor; A 1 = 0 makes the row sum exactly 1 - s (w_-1 + w_0 + w_1) = 1 (reading R6)
    const cld a = -s * st.w[2], c = -s * st.w[4];
    const cld e = 1.0L - s * (st.w[2] + st.w[3] + st.w[4]);
    f.push_back({a, e - a - c, c, e});
    lead = 1;
    return true;
  }
  if (op_is_heat(op)) {
    // A(tau) = sum_{o>=1} w_o (z^o + z^-o - 2), z^o + z^-o - 2 = tau, tau^2 + 4 tau, tau^3 + 6 tau^2 + 9 tau
    static const int P[4][4] = {{0, 0, 0, 0}, {0, 1, 0, 0}, {0, 4, 1, 0}, {0, 9, 6, 1}};
    const int h = st.h1;
    std::vector<cld> p(h + 1, cld(0));
    p[0] = 1;                                        // 1 - s A(tau)
    for (int o = 1; o <= h; ++o)
      for (int j = 1; j <= h; ++j) p[j] -= s * st.w[3 + o] * (ld)P[o][j];
    std::vector<cld> tau;
    poly_roots(p, tau);
    for (const cld &t : tau) {
      if (std::abs(t) == 0) { err = "zero factor root"; return false; }
      f.push_back({cld(1), -2.0L - t, cld(1), -t});
    }
    lead = p[h];
    return true;
  }
  const int deg = st.h0 + st.h1;
  std::vector<cld> p(deg + 1, cld(0));
  for (int o = -st.h0; o <= st.h1; ++o) p[o + st.h0] = (o == 0 ? cld(1) : cld(0)) - s * st.w[3 + o];
  std::vector<cld> r;
  poly_roots(p, r);
  std::vector<cld> in, out;
  for (const cld &z : r) {
    const ld az = std::abs(z);
    if (std::fabs(az - 1) < 1e-12L) { err = "factor root on the unit circle"; return false; }
    (az < 1 ? in : out).push_back(z);
  }
  if ((int)in.size() != st.h0) { err = "factor roots do not split h0 inside / h1 outside the unit circle"; return false; }
  size_t i = 0;
  for (; i < in.size() && i < out.size(); ++i) {     // z^-1 (z - r_in)(z - r_out)
    const cld ri = in[i], ro = out[i];
    f.push_back({ri * ro, -(ri + ro), cld(1), (1.0L - ri) * (1.0L - ro)});
  }
  for (size_t j = i; j < in.size(); ++j) f.push_back({-in[j], cld(1), cld(0), 1.0L - in[j]});   // 1 - r z^-1
  for (size_t j = i; j < out.size(); ++j) f.push_back({cld(0), -out[j], cld(1), 1.0L - out[j]});  // z - r
  lead = p[deg];
  return true;
}

}  // namespace pint
