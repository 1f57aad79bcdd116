"""Pins for oracle/operators.py: stencil definition vs dense matrix vs closed-form symbols."""
import numpy as np
import pytest

import workloads as W
from oracle.operators import apply_A, dense_A, symbol, symbol_grid

SMALL = [
    W.Problem("h1", 1, 16, 1, "heat", 0.7, 0, 0, 1, 2, 1, "random", "fixed", 0.1, 1),
    W.Problem("a1", 1, 16, 1, "advection", 0, 1.3, 0, 1, 2, 1, "random", "fixed", 0.1, 1),
    W.Problem("h2", 2, 8, 4, "heat", 0.3, 0, 0, 1, 2, 1, "random", "fixed", 0.1, 1),
    W.Problem("a2", 2, 8, 16, "advection", 0, 1.0, -0.5, 1, 2, 1, "random", "fixed", 0.1, 1),
]
# the paper's other discretisations: centred kappa 4, 6 and upwind 1, 3, 5 (both flow signs)
SMALL += [W.Problem(op + ("_2d" if d == 2 else ""), d, 16, 8 if d == 2 else 1, op, 0.4,
                    1.1 if op != "heat4" else 0, -0.6 if d == 2 else 0, 1, 2, 1, "random", "fixed", 0.1, 1)
          for op in ("heat4", "heat6", "upwind1", "upwind2", "upwind3", "upwind4", "upwind5") for d in (1, 2)]
SMALL += [W.Problem("up3_neg", 1, 16, 1, "upwind3", 0, -0.8, 0, 1, 2, 1, "random", "fixed", 0.1, 1)]


@pytest.mark.parametrize("p", SMALL, ids=lambda p: p.name)
def test_dense_matches_stencil(p):
    rng = np.random.default_rng(0)
    v = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
    np.testing.assert_allclose(dense_A(p) @ v, apply_A(p, v), rtol=0, atol=1e-12 * np.abs(apply_A(p, v)).max())


@pytest.mark.parametrize("p", SMALL + [W.CONFIGS[2], W.reduced(4), W.reduced(5)], ids=lambda p: p.name)
def test_constants_in_kernel(p):
    """A 1 = 0 for every operator: exact for the 3-point stencils,
    to rounding of the weight sum (|weights|_1 * 8 eps) for the wider ones (thirds, twelfths)."""
    r = np.abs(apply_A(p, np.ones(p.N, dtype=complex))).max()
    if p.op in ("heat", "advection"):
        assert r == 0.0
    else:
        assert r <= 8 * np.finfo(float).eps * np.abs(dense_A(p)).sum(1).max()


@pytest.mark.parametrize("p", SMALL + [W.CONFIGS[2], W.reduced(4), W.reduced(5)], ids=lambda p: p.name)
def test_fourier_modes_are_eigenvectors(p):
    """A e^{2 pi i (kx x + ky y)} = lambda(kx, ky) e^{...} with the closed-form symbols."""
    rng = np.random.default_rng(1)
    xs = np.arange(p.nx)
    ys = np.arange(p.ny)
    for _ in range(6):
        kx, ky = int(rng.integers(p.nx)), int(rng.integers(p.ny))
        qx = (kx * xs[None, :]) % p.nx
        qy = (ky * ys[:, None]) % p.ny
        mode = (np.exp(2j * np.pi * qx / p.nx) * np.exp(2j * np.pi * qy / p.ny)).reshape(-1)
        lam = symbol(p, np.array(kx), np.array(ky))
        Am = apply_A(p, mode)
        scale = max(1.0, np.abs(dense_A(p)).sum(1).max()) if p.N <= 4096 else max(1.0, 4 * abs(lam))
        np.testing.assert_allclose(Am, lam * mode, rtol=0, atol=1e-12 * scale)


def test_heat_symbol_is_nonpositive_and_advection_imaginary():
    p = W.reduced(4)
    lam = symbol_grid(p)
    assert np.all(lam.real <= 0) and np.all(lam.imag == 0)
    q = W.reduced(5)
    lam = symbol_grid(q)
    assert np.all(lam.real == 0)


@pytest.mark.parametrize("op,order", [("heat", 2), ("heat4", 4), ("heat6", 6), ("advection", 2),
                                      ("upwind1", 1), ("upwind2", 2), ("upwind3", 3), ("upwind4", 4),
                                      ("upwind5", 5)])
@pytest.mark.parametrize("sign", [1.0, -1.0])
def test_consistency_order(op, order, sign):
    """A applied to sin(2 pi x) (+ 0.5 cos(4 pi x)) approaches nu u'' (heat) or -c u' (advection,
    upwind) with error ~ n^-order: pins every stencil weight (a wrong weight breaks the rate)."""
    errs = []
    for n in (32, 64, 128):
        p = W.Problem("c", 1, n, 1, op, 0.3, sign * 0.9, 0, 1, 2, 1, "random", "fixed", 0.1, 1)
        x = np.arange(n) / n
        u = np.sin(2 * np.pi * x) + 0.5 * np.cos(4 * np.pi * x)
        if op.startswith("heat"):
            exact = 0.3 * (-(2 * np.pi) ** 2 * np.sin(2 * np.pi * x) - 0.5 * (4 * np.pi) ** 2 * np.cos(4 * np.pi * x))
        else:
            exact = -sign * 0.9 * (2 * np.pi * np.cos(2 * np.pi * x) - 0.5 * 4 * np.pi * np.sin(4 * np.pi * x))
        errs.append(np.abs(apply_A(p, u.astype(complex)) - exact).max())
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(rates - order) < 0.3), (errs, rates)


def test_upwind_damps_and_centred_heat_is_real():
    """Upwind symbols have Re lambda <= 0 (dissipative, flow-sign independent); centred heat symbols
    of every order are real and non-positive."""
    for op in ("upwind1", "upwind2", "upwind3", "upwind4", "upwind5"):
        for c in (1.0, -1.0):
            p = W.Problem("u", 2, 16, 8, op, 0, c, 0.5 * c, 1, 2, 1, "random", "fixed", 0.1, 1)
            assert np.all(symbol_grid(p).real <= 1e-12)
    for op in ("heat4", "heat6"):
        p = W.Problem("h", 2, 16, 8, op, 0.5, 0, 0, 1, 2, 1, "random", "fixed", 0.1, 1)
        lam = symbol_grid(p)
        assert np.all(lam.imag == 0) and np.all(lam.real <= 0)
