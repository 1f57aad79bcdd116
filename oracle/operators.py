"""Spatial operators A of u_t = A u + b (oracle; test infrastructure only).

Periodic grid x_j = j/n on [0,1) (2-D: n = y*nx + x); 2-D sums the two axes.
reading for the configs, plus the paper's other discretisations (
DESIGN.md reading R14): centred differences of order kappa = 2, 4, 6 for the second derivative
and upwind differences of order 1, 2, 3, 4, 5 for the first derivative.
  heat  (kappa):   (A u)_j = nu n^2 sum_s d2[s] u_{j+s}
  advection:       (A u)_j = -c n/2 (u_{j+1} - u_{j-1})                      (centred, kappa 2)
  upwind (kappa):  (A u)_j = -c n sum_s d1[s] u_{j+s},  d1 biased against the flow (c > 0: left)
Stencil weights (exact rationals):
  d2, kappa 2: (1, -2, 1);  4: (-1/12, 4/3, -5/2, 4/3, -1/12);  6: (1/90, -3/20, 3/2, -49/18, ...)
  d1 (c > 0), kappa 1: {-1: -1, 0: 1};  3: (u_{j-2} - 6u_{j-1} + 3u_j + 2u_{j+1})/6;
              5: (-2u_{j-3} + 15u_{j-2} - 60u_{j-1} + 20u_j + 30u_{j+1} - 3u_{j+2})/60;  c < 0: mirrored.
  Table 1 also lists upwind kappa = 2 and 4 without printing them (DESIGN.md reading
  R16): the unique (kappa+1)-point stencils of order kappa on the offsets -(kappa/2 + 1) ..
  kappa/2 - 1 (one point more upwind than downwind, as for the odd orders):
              2: (u_{j-2} - 4u_{j-1} + 3u_j)/2;  4: (-u_{j-3} + 6u_{j-2} - 18u_{j-1} + 10u_j + 3u_{j+1})/12.
Fourier symbols (A e^{2 pi i k j/n} = lambda(k) e^{2 pi i k j/n}) in cancellation-free forms
(SURVEY §8(c) C6): with theta = 2 pi k/n (index reduced mod n),
  symmetric d2:  lambda = -4 nu n^2 sum_{s>=1} d2[s] sin^2(s theta/2)
  d1:            sum_s d1[s] e^{i s theta} = -2 sum_s d1[s] sin^2(s theta/2) + i sum_s d1[s] sin(s theta)
  advection:     lambda = -i c n sin(theta)
"""
from __future__ import annotations

import numpy as np


D2 = {2: {-1: 1.0, 0: -2.0, 1: 1.0},
      4: {-2: -1 / 12, -1: 4 / 3, 0: -5 / 2, 1: 4 / 3, 2: -1 / 12},
      6: {-3: 1 / 90, -2: -3 / 20, -1: 3 / 2, 0: -49 / 18, 1: 3 / 2, 2: -3 / 20, 3: 1 / 90}}
D1_LEFT = {1: {-1: -1.0, 0: 1.0},
           2: {-2: 1 / 2, -1: -2.0, 0: 3 / 2},
           3: {-2: 1 / 6, -1: -1.0, 0: 1 / 2, 1: 1 / 3},
           4: {-3: -1 / 12, -2: 1 / 2, -1: -3 / 2, 0: 5 / 6, 1: 1 / 4},
           5: {-3: -2 / 60, -2: 15 / 60, -1: -60 / 60, 0: 20 / 60, 1: 30 / 60, 2: -3 / 60}}
HEAT_OPS = {"heat": 2, "heat4": 4, "heat6": 6}
UPWIND_OPS = {"upwind1": 1, "upwind2": 2, "upwind3": 3, "upwind4": 4, "upwind5": 5}


def axis_stencil(op: str, n: int, coef: float) -> dict:
    """{offset s: weight} of A along one axis of n points (coef = nu for heat, c for advection)."""
    if op in HEAT_OPS:
        return {s: coef * n * n * w for s, w in D2[HEAT_OPS[op]].items()}
    if op == "advection":
        return {-1: coef * n / 2.0, 1: -coef * n / 2.0}
    if op in UPWIND_OPS:
        d = D1_LEFT[UPWIND_OPS[op]]
        if coef < 0:
            d = {-s: -w for s, w in d.items()}           # flow to the left: mirrored stencil
        return {s: -coef * n * w for s, w in d.items()}
    raise ValueError(op)


def _axes(p):
    if p.op in HEAT_OPS:
        cx, cy = p.nu, p.nu
    else:
        cx, cy = p.cx, p.cy
    out = [(-1, axis_stencil(p.op, p.nx, cx))]
    if p.dim == 2:
        out.append((-2, axis_stencil(p.op, p.ny, cy)))
    return out


def apply_A(p, v: np.ndarray) -> np.ndarray:
    """A applied along the trailing spatial axis (length N = nx*ny) of v: the stencil sum with
    np.roll (np.roll(w, -s)[j] = w[j+s])."""
    shp = v.shape
    w = v.reshape(shp[:-1] + (p.ny, p.nx))
    out = np.zeros_like(w)
    for axis, st in _axes(p):
        for sft, wt in st.items():
            out += wt * np.roll(w, -sft, axis=axis)
    return out.reshape(shp)


def dense_A(p) -> np.ndarray:
    """A as an explicit N x N matrix, entry by entry from the stencil definition (tiny N only)."""
    nx, ny = p.nx, p.ny
    A = np.zeros((nx * ny, nx * ny), dtype=np.complex128)
    axes = dict(_axes(p))
    for y in range(ny):
        for x in range(nx):
            i = y * nx + x
            for sft, wt in axes[-1].items():
                A[i, y * nx + (x + sft) % nx] += wt
            if p.dim == 2:
                for sft, wt in axes[-2].items():
                    A[i, ((y + sft) % ny) * nx + x] += wt
    return A


def symbol_1d(op: str, n: int, k: np.ndarray, coef: float) -> np.ndarray:
    """Per-axis symbol for integer wavenumbers k (coef = nu for heat, c for advection)."""
    k = np.asarray(k, dtype=np.int64) % n
    th = 2.0 * np.pi * k.astype(np.float64) / n
    if op in HEAT_OPS:
        acc = np.zeros_like(th)
        for sft, w in D2[HEAT_OPS[op]].items():
            if sft > 0:
                acc = acc + w * np.sin(sft * th / 2) ** 2
        return np.asarray(-4.0 * coef * n * n * acc, dtype=np.complex128)
    if op == "advection":
        # sin(2 pi k/n) from the reduced index k mod n
        return np.asarray(-1j * coef * n * np.sin(th), dtype=np.complex128)
    st = axis_stencil(op, n, coef)
    re = np.zeros_like(th)
    im = np.zeros_like(th)
    for sft, w in st.items():
        re = re - 2.0 * w * np.sin(sft * th / 2) ** 2
        im = im + w * np.sin(sft * th)
    return re + 1j * im


def symbol(p, kx: np.ndarray, ky: np.ndarray) -> np.ndarray:
    """lambda(kx, ky) for mode exp(2 pi i (kx x + ky y)) (broadcasting)."""
    cx, cy = (p.nu, p.nu) if p.op in HEAT_OPS else (p.cx, p.cy)
    lam = symbol_1d(p.op, p.nx, kx, cx)
    if p.dim == 2:
        lam = lam + symbol_1d(p.op, p.ny, ky, cy)
    return lam


def symbol_grid(p) -> np.ndarray:
    """lambda on the numpy-fft grid, shape (ny, nx) flattened to (N,), index n = ky*nx + kx."""
    kx = np.arange(p.nx)[None, :]
    ky = np.arange(p.ny)[:, None]
    return np.broadcast_to(symbol(p, kx, ky), (p.ny, p.nx)).reshape(-1).copy()
