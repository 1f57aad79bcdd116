"""Adaptive alpha sequence of Algorithm 2 (oracle; test infrastructure only).

PAPER.md P:387-397: gamma := L (3 eps + tau) ||w||_inf;
  alpha_{k+1} = sqrt(gamma / m_k),  m_{k+1} = 2 sqrt(m_k gamma)
P:399-401: the m_k descend (and alpha_k <= 1/2) while 4 gamma <= m_k.
P:402: telescoped m_k = (4 gamma)^{1 - 2^-k} m0^{2^-k}.
DESIGN.md reading R4: eps = 2^-52, tau = 0, m0 = dT, ||w||_inf = ||u0||_inf
when b == 0 (w = (u0 replicated, 0, ..., 0)).
"""
from __future__ import annotations

import math


def gamma(L: int, eps: float, tau: float, w_inf: float) -> float:
    return L * (3.0 * eps + tau) * w_inf


def adaptive_schedule(L: int, w_inf: float, m0: float, K: int, eps: float = 2.0 ** -52,
                      tau: float = 0.0):
    """Returns (alphas[0..K), ms[0..K]) with alphas[k] used by iteration k (Alg. 2 line 4-6)."""
    g = gamma(L, eps, tau, w_inf)
    if not (g > 0.0):
        raise ValueError("gamma must be positive")
    ms = [m0]
    alphas = []
    for _ in range(K):
        mk = ms[-1]
        if 4.0 * g > mk:
            raise ValueError("m_k < 4 gamma: alpha would exceed 1/2 (P:399-401)")
        alphas.append(math.sqrt(g / mk))
        ms.append(2.0 * math.sqrt(mk * g))
    return alphas, ms
