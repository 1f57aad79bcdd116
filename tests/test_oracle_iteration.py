"""Pins for oracle/paralpha.py: brute force, residual structure, fixed point, closed form,
contraction, tier agreement and the paper's factorisation identities."""
import json
import os

import numpy as np
import pytest

import workloads as W
from oracle.collocation import Tableau
from oracle.paralpha import (E_matrix, ModeOracle, Oracle, V_inverse, V_matrix, brute_force_iterate,
                             brute_force_iterate_direct,
                             d_values, mode_coefficients, relative_l2, residual, sequential_solution,
                             single_mode_solution, w_vector)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))

TINY = [W.CONFIGS[1]] + W.edge_cases()


@pytest.mark.parametrize("p", TINY, ids=lambda p: p.name)
@pytest.mark.parametrize("tier", ["dense", "fourier"])
def test_brute_force(p, tier):
    """P1: every iteration equals u + solve(C_alpha, w - C u) with C, C_alpha assembled densely."""
    u0 = p.u0()
    o = Oracle(p, u0, tier)
    u = o.initial()
    ub = u.copy()
    for k in range(3):
        a = p.alpha_fixed * (1 + k)
        u = o.iterate(u, a)
        ub = brute_force_iterate(p, o.tab, ub, u0, a)
        assert relative_l2(u, ub) < 1e-11, (k, relative_l2(u, ub))


@pytest.mark.parametrize("p", TINY[:4], ids=lambda p: p.name)
def test_residual_structure(p):
    """P5: w - C u^{k+1} = -alpha e_1 (x) H (u_L^{k+1} - u_L^k): only block 0 is
    non-zero and it holds -alpha times the change of the last node of the last step."""
    u0 = p.u0()
    o = Oracle(p, u0, "dense")
    u = o.initial()
    a = p.alpha_fixed
    un = o.iterate(u, a)
    r = residual(p, o.tab, un, u0)
    expect = -a * (un[-1, -1] - u[-1, -1])
    # roundoff floor of w - C u is eps * ||C|| * ||u||, ||C||_inf <= 2 + dT ||Q||_inf ||A||_inf
    from oracle.operators import dense_A
    normC = 2 + p.dT * np.abs(o.tab.Q).sum(1).max() * np.abs(dense_A(p)).sum(1).max()
    tol = 1e-12 * normC * np.abs(un).max()
    if p.L > 1:
        assert np.abs(r[1:]).max() <= tol
    for m in range(p.M):
        np.testing.assert_allclose(r[0, m], expect, atol=tol)


@pytest.mark.parametrize("p", TINY, ids=lambda p: p.name)
def test_fixed_point_is_sequential_collocation(p):
    """P2: the iteration converges to the solution of L sequential Radau IIA steps."""
    u0 = p.u0()
    o = Oracle(p, u0)
    u = o.initial()
    for k in range(12):
        u = o.iterate(u, min(0.3, p.alpha_fixed * 10 ** (k // 2)))
    us = sequential_solution(p, o.tab, u0)
    assert relative_l2(u, us) < 1e-12


def test_config1_single_mode_closed_form():
    """P3: config 1's u0 = sin(2 pi x) is one spatial mode pair; u* = s_m R(z)^l, z = dT lambda."""
    p = W.CONFIGS[1]
    tab = Tableau(p.M)
    lam = -4 * p.nu * p.nx ** 2 * np.sin(np.pi / p.nx) ** 2
    z = p.dT * lam
    closed = single_mode_solution(tab, z, p.L, 1.0)
    us = sequential_solution(p, tab, p.u0())
    coef = np.fft.fft(us, axis=-1)[:, :, 1] / (p.N / 2j)
    np.testing.assert_allclose(coef, closed, atol=1e-14)
    # the R(z) value for this z by the textbook M=2 Pade form (1 + z/3) / (1 - 2z/3 + z^2/6)
    R = (1 + z / 3) / (1 - 2 * z / 3 + z * z / 6)
    assert closed[3, 1] == pytest.approx(R ** 4, rel=1e-13)


@pytest.mark.parametrize("alpha", [1e-4, 1e-2, 0.1])
def test_contraction(alpha):
    """P4 / Theorem P:279: per spatial mode, ||e^{k+1}|| <= alpha/(1-alpha) ||e^k|| (inf-norm over l, m)."""
    p = W.CONFIGS[2].replace(L=16, nx=64)
    u0 = p.u0()
    kx = np.arange(0, 8)
    ky = np.zeros_like(kx)
    uh0 = mode_coefficients(p, u0, kx, ky)
    mo = ModeOracle(p, uh0, kx, ky)
    ustar = np.stack([single_mode_solution(mo.tab, p.dT * mo.lam[j], p.L, uh0[j]) for j in range(len(kx))], -1)
    u = mo.initial()
    e0 = np.abs(u - ustar).max(axis=(0, 1))
    u = mo.iterate(u, alpha)
    e1 = np.abs(u - ustar).max(axis=(0, 1))
    u = mo.iterate(u, alpha)
    e2 = np.abs(u - ustar).max(axis=(0, 1))
    fac = alpha / (1 - alpha) * 1.1
    floor = 1e-13 * np.abs(ustar).max()
    assert np.all(e1 <= fac * e0 + floor)
    assert np.all(e2 <= fac * e1 + floor)


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_mode_tier_matches_fourier_tier(cfg):
    """The per-mode tier (used for full-size sampled parity) equals the physical-space tier."""
    p = W.reduced(cfg)
    if cfg == 2:
        p = p.replace(L=16)
    u0 = p.u0()
    o = Oracle(p, u0, "fourier")
    rng = np.random.default_rng(7)
    kx = np.concatenate([[0, 1, 2], rng.integers(0, p.nx, 6)])
    ky = np.concatenate([[0, 1, 0] if p.dim == 2 else [0, 0, 0], rng.integers(0, p.ny, 6)])
    mo = ModeOracle(p, mode_coefficients(p, u0, kx, ky), kx, ky)
    u, uh = o.initial(), mo.initial()
    for k in range(2):
        a = 10.0 ** (-4 + 2 * k)
        u, uh = o.iterate(u, a), mo.iterate(uh, a)
        proj = mode_coefficients(p, u, kx, ky)
        assert np.abs(proj - uh).max() <= 1e-10 * np.abs(uh).max()


def test_circulant_diagonalisation():
    """P7 / Lemma P:164-171: E_alpha = V D V^{-1}; |d| = alpha^{1/L}; alpha=1 gives the numpy fft."""
    for L in (1, 2, 4, 8, 16):
        a = 0.3
        V, Vi, d = V_matrix(L, a), V_inverse(L, a), d_values(L, a)
        np.testing.assert_allclose(V @ np.diag(d) @ Vi, E_matrix(L, a), atol=1e-14)
        np.testing.assert_allclose(V @ Vi, np.eye(L), atol=1e-14)
        np.testing.assert_allclose(np.abs(d), a ** (1.0 / L), rtol=1e-15)
        np.testing.assert_allclose(V_inverse(L, 1.0), np.fft.fft(np.eye(L), axis=0), atol=1e-13)
    g = GOLD["spec_d_example"]
    np.testing.assert_allclose(d_values(g["L"], g["alpha"]), g["d"], atol=1e-16)


def test_spec_residual_example():
    """L=2, M=1, N=1, A=0, u0=1, u=(0.5, 2), alpha=0.1: (C_a - C) u + w = (0.8, 0).
    The oracle's residual w - C u plus C_alpha u (assembled) must give it."""
    g = GOLD["spec_residual_example"]
    p = W.Problem("spec", 1, 1, 1, "heat", 0.0, 0, 0, 1.0, 2, 1, "random", "fixed", 0.1, 1)
    tab = Tableau(1)
    u = np.array(g["u"], dtype=complex).reshape(2, 1, 1)
    u0 = np.ones(1, dtype=complex)
    r = residual(p, tab, u, u0).reshape(-1)
    Ca_u = (np.eye(2) + E_matrix(2, g["alpha"])) @ u.reshape(-1)
    np.testing.assert_allclose(r + Ca_u, g["r_direct"], atol=1e-16)


@pytest.mark.parametrize("M", [1, 2, 3, 4])
def test_paper_G_and_QG_identities(M):
    """G^{-1} = I - r H_M with r = d/(1+d); Q G^{-1} = Q - r D_t H_M."""
    tab = Tableau(M)
    for d in d_values(8, 0.37):
        G = np.eye(M) + d * tab.H
        r = d / (1 + d)
        np.testing.assert_allclose(np.linalg.inv(G), np.eye(M) - r * tab.H, atol=1e-14)
        np.testing.assert_allclose(tab.Q @ np.linalg.inv(G), tab.Q - r * tab.Dt @ tab.H, atol=1e-14)


def test_paper_p2_char_poly_sign():
    """P:567's p_2(lambda) = 2 l^2 - (4/3 + 2r) l + (r+1)/3 has the eigenvalues of Q + r D_t H_M,
    i.e. of Q G^{-1} with r -> -r (reading R12: sign slip in Lemma 3.4)."""
    tab = Tableau(2)
    for r in GOLD["p2_char_poly"]["r_sample"]:
        roots = np.sort_complex(np.roots([2.0, -(4.0 / 3 + 2 * r), (r + 1) / 3.0]))
        ev = np.sort_complex(np.linalg.eigvals(tab.Q + r * tab.Dt @ tab.H))
        np.testing.assert_allclose(roots, ev, atol=1e-14)


def test_w_vector_layout():
    p = W.CONFIGS[1]
    w = w_vector(p, p.u0())
    assert np.all(w[1:] == 0) and np.all(w[0, 1] == p.u0())


@pytest.mark.parametrize("p", TINY, ids=lambda p: p.name)
def test_direct_form_brute_force_and_equivalence(p):
    """Alg. 1 as printed (direct form): equals the dense C_a solve of (C_a - C)u + w,
    and agrees with the correction form (reading R1) up to roundoff."""
    u0 = p.u0()
    o = Oracle(p, u0, "dense")
    u = o.initial()
    uc = u.copy()
    for k in range(3):
        a = p.alpha_fixed * (1 + k)
        un = o.iterate_direct(u, a)
        ub = brute_force_iterate_direct(p, o.tab, u, u0, a)
        assert relative_l2(un, ub) < 1e-11
        uc = o.iterate(uc, a)
        assert relative_l2(un, uc) < 1e-9
        u = un


def test_direct_form_mode_tier():
    p = W.reduced(5).replace(L=8)
    u0 = p.u0()
    o = Oracle(p, u0, "fourier")
    kx = np.array([0, 1, 3, 5])
    ky = np.array([0, 2, 1, 7])
    mo = ModeOracle(p, mode_coefficients(p, u0, kx, ky), kx, ky)
    u, uh = o.initial(), mo.initial()
    for a in (1e-3, 1e-2):
        u, uh = o.iterate_direct(u, a), mo.iterate_direct(uh, a)
        proj = mode_coefficients(p, u, kx, ky)
        assert np.abs(proj - uh).max() <= 1e-10 * np.abs(uh).max()
