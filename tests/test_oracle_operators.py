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


@pytest.mark.parametrize("p", SMALL, ids=lambda p: p.name)
def test_dense_matches_stencil(p):
    rng = np.random.default_rng(0)
    v = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
    np.testing.assert_allclose(dense_A(p) @ v, apply_A(p, v), rtol=0, atol=1e-12 * np.abs(apply_A(p, v)).max())


@pytest.mark.parametrize("p", SMALL + [W.CONFIGS[2], W.reduced(4), W.reduced(5)], ids=lambda p: p.name)
def test_constants_in_kernel(p):
    """A 1 = 0 for both operators."""
    assert np.abs(apply_A(p, np.ones(p.N, dtype=complex))).max() == 0.0


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
