"""Radau IIA collocation tableau (oracle; test infrastructure only).

PAPER.md P:91-111 (eq. collocation): q_mi = int_0^{t_m} c_i(s) ds with c_i the
i-th Lagrange polynomial on the nodes; right-included Gauss-Radau nodes.
P:555-557: nodes are the roots of R_M = P_{M-1} + P_M on [-1, 1] (left point
included) mapped by x(t) = -2t + 1.
P:113: H_M has ones in its last column; D_t = diag(t_1..t_M).
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import legendre as npleg
from numpy.polynomial import polynomial as nppoly


def radau_nodes(M: int) -> np.ndarray:
    """Right-included Gauss-Radau nodes on (0, 1], ascending, last == 1 exactly."""
    if M < 1:
        raise ValueError("M >= 1")
    c = np.zeros(M + 1)
    c[M - 1] = 1.0      # P_{M-1}
    c[M] += 1.0         # + P_M
    x = np.sort(npleg.legroots(c).real)
    # x = -1 is an exact root (left point); polish the others with Newton on R_M
    dc = npleg.legder(c)
    out = []
    for xi in x:
        if abs(xi + 1.0) < 1e-8:
            out.append(-1.0)
            continue
        for _ in range(8):
            xi = xi - npleg.legval(xi, c) / npleg.legval(xi, dc)
        out.append(xi)
    t = (1.0 - np.asarray(out)) / 2.0      # x(t) = -2t + 1  <=>  t = (1 - x)/2
    t = np.sort(t)
    t[-1] = 1.0
    return t


def lagrange_coeffs(t: np.ndarray, i: int) -> np.ndarray:
    """Monomial coefficients (low -> high) of the i-th Lagrange polynomial c_i on nodes t."""
    others = np.delete(t, i)
    num = nppoly.polyfromroots(others) if len(others) else np.array([1.0])
    den = np.prod(t[i] - others) if len(others) else 1.0
    return num / den


def collocation_matrix(t: np.ndarray) -> np.ndarray:
    """Q with q_mi = int_0^{t_m} c_i(s) ds, by exact polynomial integration."""
    M = len(t)
    Q = np.zeros((M, M))
    for i in range(M):
        ci = lagrange_coeffs(t, i)
        Ci = nppoly.polyint(ci, lbnd=0.0)     # antiderivative vanishing at 0
        Q[:, i] = nppoly.polyval(t, Ci)
    return Q


def H_matrix(M: int) -> np.ndarray:
    """H_M: zeros except ones in the last column."""
    H = np.zeros((M, M))
    H[:, M - 1] = 1.0
    return H


class Tableau:
    def __init__(self, M: int):
        self.M = M
        self.t = radau_nodes(M)
        self.Q = collocation_matrix(self.t)
        self.H = H_matrix(M)
        self.Dt = np.diag(self.t)
