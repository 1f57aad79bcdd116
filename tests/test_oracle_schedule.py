"""Pins for oracle/schedule.py (Algorithm 2)."""
import json
import math
import os

import numpy as np
import pytest

from oracle.schedule import adaptive_schedule, gamma

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_spec_example():
    g = GOLD["spec_schedule_example"]
    # gamma = L (3 eps + tau) w_inf with L = 1, eps = 0, tau = 1: gamma = w_inf
    alphas, ms = adaptive_schedule(1, g["gamma"], g["m0"], 1, eps=0.0, tau=1.0)
    assert alphas[0] == pytest.approx(g["alpha1"], rel=1e-14)
    assert ms[1] == pytest.approx(g["m1"], rel=1e-14)


def test_fig3_sequence_from_first_alpha():
    """Fig. 3: the recurrence is scale-free in rho = gamma/m0; rho = alpha_1^2 reproduces
    the printed alpha_2..alpha_4 (3 printed digits)."""
    g = GOLD["fig3_alpha"]
    a1 = g["alphas"][0]
    alphas, _ = adaptive_schedule(1, 1.0, 1.0 / a1 ** 2, 4, eps=0.0, tau=1.0)
    np.testing.assert_allclose(alphas, g["alphas"], rtol=g["rel_tol"])


@pytest.mark.parametrize("m0,g", [(1e-2, 3e-14), (1.0 / 256, 1.6e-13), (5.0, 1e-12)])
def test_telescoped_m(m0, g):
    """m_k = (4 gamma)^{1 - 2^-k} m0^{2^-k}; alpha_{k+1} = sqrt(gamma/m_k) <= 1/2 ascending."""
    alphas, ms = adaptive_schedule(1, g, m0, 12, eps=0.0, tau=1.0)
    for k in range(1, 13):
        assert ms[k] == pytest.approx((4 * g) ** (1 - 2.0 ** -k) * m0 ** (2.0 ** -k), rel=1e-12)
    assert all(b > a for a, b in zip(alphas, alphas[1:]))
    assert max(alphas) <= 0.5


def test_gamma_definition():
    assert gamma(256, 2.0 ** -52, 0.0, 8.0) == 256 * 3 * 2.0 ** -52 * 8.0


def test_rejects_stagnation():
    with pytest.raises(ValueError):
        adaptive_schedule(1, 1.0, 2.0, 1, eps=0.0, tau=1.0)   # m0 < 4 gamma
