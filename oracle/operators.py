"""Spatial operators A of u_t = A u + b for the configs (oracle; test infrastructure only).

Periodic grid x_j = j/n on [0,1) (2-D: n = y*nx + x).  SURVEY.md §8(c) C9 reading:
  heat:       (A u)_j = nu * n^2 (u_{j-1} - 2 u_j + u_{j+1})        per axis, summed in 2-D
  advection:  (A u)_j = -c * n/2 (u_{j+1} - u_{j-1})                per axis (c = cx, cy)
Fourier symbols (A e^{2 pi i k j/n} = lambda(k) e^{2 pi i k j/n}), cancellation-free forms
(SURVEY §8(c) C6):
  heat:       lambda = -4 nu (nx^2 sin^2(pi kx/nx) + ny^2 sin^2(pi ky/ny))
  advection:  lambda = -i (cx nx sin(2 pi kx/nx) + cy ny sin(2 pi ky/ny))
"""
from __future__ import annotations

import numpy as np


def apply_A(p, v: np.ndarray) -> np.ndarray:
    """A applied along the trailing spatial axis (length N = nx*ny) of v."""
    nx, ny = p.nx, p.ny
    shp = v.shape
    w = v.reshape(shp[:-1] + (ny, nx))
    out = np.zeros_like(w)
    if p.op == "heat":
        out += p.nu * nx * nx * (np.roll(w, 1, axis=-1) - 2.0 * w + np.roll(w, -1, axis=-1))
        if p.dim == 2:
            out += p.nu * ny * ny * (np.roll(w, 1, axis=-2) - 2.0 * w + np.roll(w, -1, axis=-2))
    elif p.op == "advection":
        # np.roll(w, -1)[j] = w[j+1]
        out += -p.cx * nx / 2.0 * (np.roll(w, -1, axis=-1) - np.roll(w, 1, axis=-1))
        if p.dim == 2:
            out += -p.cy * ny / 2.0 * (np.roll(w, -1, axis=-2) - np.roll(w, 1, axis=-2))
    else:
        raise ValueError(p.op)
    return out.reshape(shp)


def dense_A(p) -> np.ndarray:
    """A as an explicit N x N matrix, entry by entry from the stencil definition (tiny N only)."""
    nx, ny = p.nx, p.ny
    N = nx * ny
    A = np.zeros((N, N), dtype=np.complex128)
    for y in range(ny):
        for x in range(nx):
            i = y * nx + x
            xm, xp = y * nx + (x - 1) % nx, y * nx + (x + 1) % nx
            if p.op == "heat":
                A[i, xm] += p.nu * nx * nx
                A[i, i] += -2.0 * p.nu * nx * nx
                A[i, xp] += p.nu * nx * nx
            else:
                A[i, xp] += -p.cx * nx / 2.0
                A[i, xm] += p.cx * nx / 2.0
            if p.dim == 2:
                ym, yp = ((y - 1) % ny) * nx + x, ((y + 1) % ny) * nx + x
                if p.op == "heat":
                    A[i, ym] += p.nu * ny * ny
                    A[i, i] += -2.0 * p.nu * ny * ny
                    A[i, yp] += p.nu * ny * ny
                else:
                    A[i, yp] += -p.cy * ny / 2.0
                    A[i, ym] += p.cy * ny / 2.0
    return A


def symbol_1d(op: str, n: int, k: np.ndarray, coef: float) -> np.ndarray:
    """Per-axis symbol for integer wavenumbers k (coef = nu for heat, c for advection)."""
    k = np.asarray(k, dtype=np.int64) % n
    if op == "heat":
        s = np.sin(np.pi * k.astype(np.float64) / n)
        return np.asarray(-4.0 * coef * n * n * s * s, dtype=np.complex128)
    # sin(2 pi k/n) from the reduced index k mod n
    return np.asarray(-1j * coef * n * np.sin(2.0 * np.pi * k.astype(np.float64) / n), dtype=np.complex128)


def symbol(p, kx: np.ndarray, ky: np.ndarray) -> np.ndarray:
    """lambda(kx, ky) for mode exp(2 pi i (kx x + ky y)) (broadcasting)."""
    if p.op == "heat":
        lam = symbol_1d("heat", p.nx, kx, p.nu)
        if p.dim == 2:
            lam = lam + symbol_1d("heat", p.ny, ky, p.nu)
    else:
        lam = symbol_1d("advection", p.nx, kx, p.cx)
        if p.dim == 2:
            lam = lam + symbol_1d("advection", p.ny, ky, p.cy)
    return lam


def symbol_grid(p) -> np.ndarray:
    """lambda on the numpy-fft grid, shape (ny, nx) flattened to (N,), index n = ky*nx + kx."""
    kx = np.arange(p.nx)[None, :]
    ky = np.arange(p.ny)[:, None]
    return np.broadcast_to(symbol(p, kx, ky), (p.ny, p.nx)).reshape(-1).copy()
