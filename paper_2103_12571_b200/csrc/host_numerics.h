// Host-side numerics of libpint (long double): Radau IIA tableau, alpha schedule, per-alpha
// factor tables.  Pure functions; no CUDA.  Independent of the numpy oracle (no shared code).
#pragma once
#include <complex>
#include <string>
#include <vector>

namespace pint {

using ld = long double;
using cld = std::complex<long double>;

// Radau IIA nodes (roots of P_{M-1} + P_M mapped by x = -2t + 1) and
// Q[m][i] = int_0^{t_m} l_i(s) ds.  Returns false on root-finding failure.
bool radau_tableau(int M, std::vector<ld> &t, std::vector<ld> &Q);

// Algorithm 2 recurrence.  Returns false (and a message) if m_k < 4 gamma.
bool adaptive_schedule(int L, double w_inf, double m0, double eps, double tau, int K,
                       std::vector<double> &alpha, std::vector<double> &m, std::string &err);

// Eigendecomposition B = S diag(lam) S^{-1} of a complex M x M matrix (row-major), columns of S
// of unit 2-norm, eigenvalues sorted by (Re, Im).  Returns false if the guard fails
// (cond_1(S) > 1e8 or min eigenvalue gap < 1e-8 * max |lam|); cond/gap reported.
bool eig_diagonalize(int M, const std::vector<cld> &B, std::vector<cld> &lam, std::vector<cld> &S,
                     std::vector<cld> &Sinv, ld &cond, ld &gap);

// In-place inverse (Gauss-Jordan, partial pivoting); false if singular.
bool invert(int M, std::vector<cld> &A);

inline int ilog2(long long n) { int r = 0; while ((1LL << r) < n) ++r; return r; }
inline bool is_pow2(long long n) { return n > 0 && (n & (n - 1)) == 0; }
inline int bitrev(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
  return r;
}

// e^{sign * 2 pi i q / n} for 0 <= q < n, long double
cld unit_root(long long q, long long n, int sign);

// Per-pass twiddle tables of the register FFT plan of fft_reg.cuh for N = 2^logn: passes of
// radix 2^b (b0 = min(B, logn), b1 = min(B, logn - b0), b2 = rest; B = maxb), pass p over blocks of m_p at
// stride s_p = m_p / 2^b_p; entry k s_p + j = e^{-2 pi i j 2^k / m_p}, k < b_p.
void pass_twiddles(int logn, int maxb, std::vector<cld> &out);
size_t pass_twiddle_count(int logn, int maxb);

}  // namespace pint
