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

// ---- spatial operators (readings R8, R14) -----------------------
// Op codes are pint_op's (include/pint.h).  Weights of A along one axis of n points: (A u)_j =
// sum_{o=-h0}^{h1} w[3+o] u_{j+o}; coef = nu (heat family) or the axis velocity c (advection).
struct AxisStencil {
  int h0 = 0, h1 = 0;
  ld w[7] = {0, 0, 0, 0, 0, 0, 0};
};
bool axis_stencil(int op, long long n, ld coef, AxisStencil &st);
bool op_is_heat(int op);
// Fourier symbol of A along one axis at integer wavenumber k (cancellation-free sin^2 forms)
cld axis_symbol(int op, long long n, long long k, ld coef);

// I - s A (1-D) as a product of tridiagonal circulant factors (PCR, kernels.cu):
//   I - s A = lead * prod_f (a_f S^{-1} + b_f + c_f S),   (S u)_j = u_{j+1},
// with e_f = a_f + b_f + c_f (row sum, carried through PCR, reading R6).  3-point operators are
// one factor (a, 1 - s wc, c) with e = 1; the centred heat family is factored in
// tau = z + 1/z - 2 = -4 sin^2(theta/2) (factors S^{-1} + S - 2 - tau_f, e_f = -tau_f exactly);
// other stencils by the roots of z^{h0} (1 - s A(z)), pairing a root inside the unit circle
// with one outside per factor so every PCR level stays diagonally dominated.  Returns false
// (err) if a root lies on the unit circle or the roots do not split h0 inside / h1 outside.
struct TriFactor { cld a, b, c, e; };
int stencil_factor_count(int op, const AxisStencil &st);
bool factor_shifted(int op, const AxisStencil &st, cld s, std::vector<TriFactor> &f, cld &lead,
                    std::string &err);

}  // namespace pint
