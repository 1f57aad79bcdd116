"""Pins for the oracle's forcing term (b != 0): w = (u0 + v_1, v_2, ..., v_L)
with v_l = dT (Q (x) I) b(t_l + tau dT).  A wrong quadrature or a dropped block
fails the brute-force identity, the fixed point or the Radau IIA order test."""
import numpy as np
import pytest

import workloads as W
from oracle.collocation import Tableau
from oracle.operators import symbol
from oracle.paralpha import (Oracle, brute_force_iterate, brute_force_iterate_direct, forcing_vector,
                             relative_l2, sequential_solution)

TINY = [W.CONFIGS[1]] + [p for p in W.edge_cases() if p.M * p.N <= 512]


def _random_v(p, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((p.L, p.M, p.N)) + 1j * rng.standard_normal((p.L, p.M, p.N))


@pytest.mark.parametrize("p", TINY, ids=lambda p: p.name)
@pytest.mark.parametrize("tier", ["dense", "fourier"])
def test_forcing_brute_force(p, tier):
    """Both forms with forcing equal the dense C_alpha solves with the same w."""
    u0 = p.u0()
    v = _random_v(p, 7)
    o = Oracle(p, u0, tier, v=v)
    tab = Tableau(p.M)
    u = ud = ub = ubd = o.initial()
    for k in range(3):
        a = 1e-2 * (1 + k)
        u = o.iterate(u, a)
        ub = brute_force_iterate(p, tab, ub, u0, a, v)
        ud = o.iterate_direct(ud, a)
        ubd = brute_force_iterate_direct(p, tab, ubd, u0, a, v)
        assert relative_l2(u, ub) < 1e-11 and relative_l2(ud, ubd) < 1e-11


@pytest.mark.parametrize("p", TINY[:3], ids=lambda p: p.name)
def test_forcing_fixed_point_is_sequential_stepping(p):
    """The iteration with forcing converges to sequential collocation stepping with forcing."""
    u0 = p.u0()
    v = _random_v(p, 8)
    o = Oracle(p, u0, "dense", v=v)
    u = o.initial()
    for _ in range(25):
        u = o.iterate(u, 1e-3)
    assert relative_l2(u, sequential_solution(p, Tableau(p.M), u0, v)) < 1e-12


@pytest.mark.parametrize("M", [1, 2, 3])
def test_forcing_quadrature_reaches_radau_order(M):
    """Manufactured single-mode solution: u0 = sin(2 pi x), b = (-sin t - lambda cos t) sin(2 pi x)
    makes the semi-discrete solution cos(t) sin(2 pi x) (lambda = the discrete symbol of the mode),
    so the step-end error of the collocation solution must fall like dT^(2M-1) (Radau IIA order)."""
    base = W.CONFIGS[1].replace(M=M, T=1.0, nx=16, nu=0.05)   # non-stiff: z = dT lambda small (no order reduction)
    errs = []
    for L in (4, 8, 16):
        p = base.replace(L=L)
        x = np.arange(p.nx) / p.nx
        s = np.sin(2 * np.pi * x)
        lam = complex(symbol(p, np.array(1), np.array(0)))
        tab = Tableau(p.M)
        v = forcing_vector(p, tab, lambda t: (-np.sin(t) - lam * np.cos(t)) * s)
        u = sequential_solution(p, tab, s.astype(np.complex128), v)
        errs.append(np.abs(u[-1, -1] - np.cos(p.T) * s).max())
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(rates > 2 * M - 1 - 0.35), (errs, rates)
