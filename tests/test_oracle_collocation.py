"""Pins for oracle/collocation.py (Radau IIA tableau) — independent of the oracle's own arithmetic."""
import json
import math
import os
from fractions import Fraction

import mpmath as mpm
import numpy as np
import pytest

from oracle.collocation import Tableau, collocation_matrix, radau_nodes

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def _radau_nodes_textbook(M, dps=40):
    """Radau IIA nodes as roots of d^{M-1}/dt^{M-1} [t^{M-1} (t-1)^M] (Hairer-Wanner IV.5) —
    a different characterisation from the paper's P_{M-1}+P_M, in exact integers + mpmath."""
    # coefficients of t^{M-1}(t-1)^M, low -> high, exact
    c = [Fraction(0)] * (2 * M)
    for j in range(M + 1):
        c[M - 1 + j] = Fraction(math.comb(M, j) * (-1) ** (M - j))
    for _ in range(M - 1):
        c = [c[i] * i for i in range(1, len(c))]
    mpm.mp.dps = dps
    coeffs_high = [mpm.mpf(x.numerator) / x.denominator for x in reversed(c)]
    roots = mpm.polyroots(coeffs_high, maxsteps=200, extraprec=200)
    return sorted(float(mpm.re(r)) for r in roots)


@pytest.mark.parametrize("M", range(1, 9))
def test_nodes_match_textbook_characterisation(M):
    t = radau_nodes(M)
    ref = _radau_nodes_textbook(M)
    assert t[-1] == 1.0                                    # right node included exactly
    assert np.all(np.diff(t) > 0) and t[0] > 0
    np.testing.assert_allclose(t, ref, rtol=0, atol=2e-15)


@pytest.mark.parametrize("key,M", [("radau_poly_w2", 2), ("radau_poly_w3", 3)])
def test_nodes_are_roots_of_paper_w(key, M):
    """PAPER.md P:567 / P:573 print w_2, w_3 whose roots are the nodes."""
    coeffs = GOLD[key]["coeffs_high_to_low"]
    t = radau_nodes(M)
    np.testing.assert_allclose(np.polyval(coeffs, t), 0.0, atol=1e-15)
    np.testing.assert_allclose(np.poly(t), coeffs, atol=1e-15)


def test_nodes_M3_closed_form():
    np.testing.assert_allclose(radau_nodes(3), GOLD["nodes_M3"]["t"], atol=1e-16)


def test_Q_M2_values():
    np.testing.assert_allclose(Tableau(2).Q, GOLD["Q_M2"]["Q"], atol=1e-16)


@pytest.mark.parametrize("M", range(1, 9))
def test_Q_integrates_polynomials_exactly(M):
    """Q (p(t_j))_j = int_0^{t_m} p for deg p <= M-1 (Q is the integral of the interpolant)."""
    tab = Tableau(M)
    for k in range(M):
        np.testing.assert_allclose(tab.Q @ tab.t ** k, tab.t ** (k + 1) / (k + 1), atol=5e-15)


@pytest.mark.parametrize("M", range(1, 9))
def test_QH_equals_DtH(M):
    """Q H_M = D_t H_M."""
    tab = Tableau(M)
    np.testing.assert_allclose(tab.Q @ tab.H, tab.Dt @ tab.H, atol=5e-15)


def _pade_R(M, z):
    """(M-1, M) Pade approximant of e^z (textbook closed form) = Radau IIA stability function."""
    k, m = M - 1, M
    P = sum(math.factorial(k + m - j) * math.factorial(k) /
            (math.factorial(k + m) * math.factorial(j) * math.factorial(k - j)) * z ** j for j in range(k + 1))
    Qd = sum(math.factorial(k + m - j) * math.factorial(m) /
             (math.factorial(k + m) * math.factorial(j) * math.factorial(m - j)) * (-z) ** j for j in range(m + 1))
    return P / Qd


@pytest.mark.parametrize("M", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("z", [-0.986167977534, -3.0 + 2.0j, 0.25j, -40.0])
def test_stability_function_is_pade(M, z):
    tab = Tableau(M)
    s = np.linalg.solve(np.eye(M) - z * tab.Q, np.ones(M))
    assert abs(s[-1] - _pade_R(M, z)) <= 1e-13 * max(1.0, abs(s[-1]))


@pytest.mark.parametrize("M", [1, 2, 3, 4])
def test_temporal_order(M):
    """Dahlquist u' = lam u over [0,1]: error of L collocation steps ~ dT^{2M-1}."""
    lam = -1.0 + 2.0j
    errs = []
    Ls = [4, 8]
    for L in Ls:
        tab = Tableau(M)
        dT = 1.0 / L
        s = np.linalg.solve(np.eye(M) - dT * lam * tab.Q, np.ones(M))
        errs.append(abs(s[-1] ** L - np.exp(lam)))
    order = math.log(errs[0] / errs[1], 2)
    assert order >= 2 * M - 1 - 0.5
