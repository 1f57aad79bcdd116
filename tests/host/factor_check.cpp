// Host-logic check of libpint's 1-D spatial factorisation (host_numerics.cpp: factor_shifted),
// compiled and run by tests/test_host_numerics.py (CPU, no GPU).  For every operator and a spread
// of shifts s (including stiff ones), the factors must reproduce the symbol of I - s A:
//   lead * prod_f (a_f z^-1 + b_f + c_f z) == 1 - s * lambda(theta),  z = e^{i theta},
// with e_f = a_f + b_f + c_f, and lambda from axis_symbol (itself pinned to the stencil here by a
// direct sum).  Prints one line per failure; exit code = number of failures.
#include <cstdio>
#include <string>
#include <vector>

#include "host_numerics.h"
#include "pint.h"

using namespace pint;

int main() {
  int fails = 0;
  const int ops[] = {PINT_OP_HEAT, PINT_OP_ADVECTION, PINT_OP_HEAT4, PINT_OP_HEAT6,
                     PINT_OP_UPWIND1, PINT_OP_UPWIND2, PINT_OP_UPWIND3, PINT_OP_UPWIND4, PINT_OP_UPWIND5};
  const long long n = 128;
  const ld coefs[] = {1.0L, -0.7L, 1e-2L};
  const cld shifts[] = {cld(1e-4L, 0), cld(3e-3L, 1e-3L), cld(2e-2L, -4e-2L), cld(0.5L, 0.3L), cld(5.0L, -2.0L)};
  for (int op : ops)
    for (ld coef : coefs) {
      if (op_is_heat(op) && coef < 0) continue;
      AxisStencil st;
      if (!axis_stencil(op, n, coef, st)) { printf("stencil op=%d\n", op); ++fails; continue; }
      // symbol vs direct stencil sum
      ld wsum = 0;
      for (int o = -st.h0; o <= st.h1; ++o) wsum += std::abs(st.w[3 + o]);
      for (long long k = 0; k < n; k += 7) {
        cld direct = 0;
        for (int o = -st.h0; o <= st.h1; ++o) direct += st.w[3 + o] * unit_root(o * k, n, +1);
        const cld sym = axis_symbol(op, n, k, coef);
        if (std::abs(direct - sym) > 1e-15L * wsum) {
          printf("symbol op=%d coef=%Lg k=%lld |d|=%Lg\n", op, coef, k, std::abs(direct - sym));
          ++fails;
        }
      }
      for (cld s : shifts) {
        std::vector<TriFactor> f;
        cld lead;
        std::string err;
        if (!factor_shifted(op, st, s, f, lead, err)) {
          printf("factor op=%d coef=%Lg s=(%Lg,%Lg): %s\n", op, coef, s.real(), s.imag(), err.c_str());
          ++fails;
          continue;
        }
        if ((int)f.size() != stencil_factor_count(op, st)) { printf("count op=%d\n", op); ++fails; }
        for (const TriFactor &t : f)
          if (std::abs(t.a + t.b + t.c - t.e) > 1e-15L * (std::abs(t.a) + std::abs(t.b) + std::abs(t.c))) {
            printf("row sum op=%d\n", op);
            ++fails;
          }
        for (long long k = 0; k < n; ++k) {
          const cld z = unit_root(k, n, +1);
          cld prod = lead;
          for (const TriFactor &t : f) prod *= t.a / z + t.b + t.c * z;
          const cld want = 1.0L - s * axis_symbol(op, n, k, coef);
          const ld scale = 1 + std::abs(s) * wsum;
          if (std::abs(prod - want) > 1e-14L * scale) {
            printf("product op=%d coef=%Lg s=(%Lg,%Lg) k=%lld err=%Lg\n", op, coef, s.real(), s.imag(), k,
                   std::abs(prod - want) / scale);
            ++fails;
            break;
          }
        }
      }
    }
  printf("failures %d\n", fails);
  return fails;
}
