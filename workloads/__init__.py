"""Seeded synthetic workloads shared by the oracle tests and the CUDA path.

This module is the ONLY code both sides import.  It holds problem definitions
(the five BASELINE.json configs and reduced parity cases) and the seeded
initial-value generators u0, and NONE of the method's arithmetic: no residual,
no transforms, no solves, no alpha schedule.

Conventions (SURVEY.md §8 notation):
  * periodic grid x_j = j / nx on [0, 1) (2-D: [0, 1)^2, n = y*nx + x, x fastest);
  * u0 is complex128 (imaginary part zero), shape (N,) with N = nx*ny;
  * "op" is "heat" (A = nu * centred Laplacian) or "advection"
    (A = -(cx d/dx + cy d/dy), centred), both 2nd order.

Config recipe citations: BASELINE.json "configs"; generators for configs 3-4
follow SURVEY.md §8(d) (the BASELINE text only says "16 sine modes with seeded
N(0,1) amplitudes" / "random Fourier modes |k|<=32 with N(0,1) coefficients").
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, Optional

import numpy as np


@dataclasses.dataclass(frozen=True)
class Problem:
    name: str
    dim: int            # 1 or 2
    nx: int
    ny: int             # 1 in 1-D
    op: str             # "heat" | "advection"
    nu: float
    cx: float
    cy: float
    T: float
    L: int              # time steps (power of two)
    M: int              # Radau IIA nodes
    u0_kind: str        # generator name, see make_u0
    alpha_mode: str     # "fixed" | "adaptive"
    alpha_fixed: Optional[float]
    iters: int
    # adaptive-alpha constants: eps = 2^-52, tau = 0, m0 = dT
    eps: float = 2.0 ** -52
    tau: float = 0.0
    m0_over_dT: float = 1.0

    @property
    def N(self) -> int:
        return self.nx * self.ny

    @property
    def U(self) -> int:
        """Space-time unknowns L*M*N (the metric's unit count)."""
        return self.L * self.M * self.N

    @property
    def dT(self) -> float:
        return self.T / self.L

    @property
    def m0(self) -> float:
        return self.m0_over_dT * self.dT

    def u0(self) -> np.ndarray:
        return make_u0(self)

    def replace(self, **kw) -> "Problem":
        return dataclasses.replace(self, **kw)


def _grid_angle_exp(k: int, n: int) -> np.ndarray:
    """exp(2*pi*i*k*j/n) for j in [0, n), from the integer-reduced index (k*j mod n)."""
    j = np.arange(n, dtype=np.int64)
    q = (k * j) % n
    ang = 2.0 * np.pi * q.astype(np.float64) / n
    return np.cos(ang) + 1j * np.sin(ang)


def make_u0(p: Problem) -> np.ndarray:
    nx, ny = p.nx, p.ny
    x = np.arange(nx, dtype=np.float64) / nx
    kind = p.u0_kind
    if kind == "sin1":                      # config 1: sin(2 pi x)
        v = _grid_angle_exp(1, nx).imag
    elif kind == "gauss1d":                 # config 2: exp(-((x-0.5)/0.05)^2)
        v = np.exp(-(((x - 0.5) / 0.05) ** 2))
    elif kind == "sines16":                 # config 3: sum_{k=1}^{16} a_k sin(2 pi k x)
        a = np.random.default_rng(3).standard_normal(16)
        v = np.zeros(nx)
        for k in range(1, 17):
            v += a[k - 1] * _grid_angle_exp(k, nx).imag
    elif kind == "fourier2d":               # config 4: random modes 1 <= |k| <= 32 (half plane)
        v = _fourier2d(nx, ny, seed=4, kmax=32)
    elif kind == "fourier2d_small":         # reduced config 4: same recipe, |k| <= 8 on a small grid
        v = _fourier2d(nx, ny, seed=4, kmax=8)
    elif kind == "gauss2d":                 # config 5: exp(-((x-.5)^2+(y-.5)^2)/0.05^2)
        y = np.arange(ny, dtype=np.float64) / ny
        v = np.exp(-(((x[None, :] - 0.5) ** 2 + (y[:, None] - 0.5) ** 2) / 0.05 ** 2))
    elif kind == "random":                  # parity edge cases: seeded N(0,1), complex
        rng = np.random.default_rng(12345 + p.N)
        v = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
        return np.ascontiguousarray(v.astype(np.complex128))
    else:
        raise ValueError(f"unknown u0 kind {kind!r}")
    return np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1).astype(np.complex128))


def fourier2d_wavevectors(kmax: int = 32):
    """Half-plane wavevectors 1 <= kx^2+ky^2 <= kmax^2, (ky > 0 or ky == 0 < kx), (ky, kx) lexicographic."""
    out = []
    for ky in range(0, kmax + 1):
        for kx in range(-kmax, kmax + 1):
            r2 = kx * kx + ky * ky
            if r2 < 1 or r2 > kmax * kmax:
                continue
            if ky > 0 or kx > 0:
                out.append((kx, ky))
    return out


def _fourier2d(nx: int, ny: int, seed: int, kmax: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    ks = fourier2d_wavevectors(kmax)
    coef = np.zeros((kmax + 1, 2 * kmax + 1), dtype=np.complex128)  # [ky][kx+kmax]
    for kx, ky in ks:
        a, b = rng.standard_normal(2)
        # a cos(th) + b sin(th) = Re((a - i b) e^{i th})
        coef[ky, kx + kmax] = a - 1j * b
    ex = np.stack([_grid_angle_exp(kx, nx) for kx in range(-kmax, kmax + 1)])   # (2k+1, nx)
    ey = np.stack([_grid_angle_exp(ky, ny) for ky in range(0, kmax + 1)])       # (k+1, ny)
    field = ey.T @ coef @ ex                                                     # (ny, nx)
    return field.real


# --- the five BASELINE.json configs -------------------------------------------------------------

CONFIGS = {
    1: Problem("cfg1_heat1d_N64_M2_L4", 1, 64, 1, "heat", 1.0, 0.0, 0.0, 0.1, 4, 2,
               "sin1", "fixed", 1e-4, 5),
    2: Problem("cfg2_adv1d_N1024_M3_L64", 1, 1024, 1, "advection", 0.0, 1.0, 0.0, 1.0, 64, 3,
               "gauss1d", "fixed", 1e-5, 10),
    3: Problem("cfg3_heat1d_N65536_M3_L256", 1, 65536, 1, "heat", 1e-2, 0.0, 0.0, 1.0, 256, 3,
               "sines16", "adaptive", None, 8),
    4: Problem("cfg4_heat2d_512x512_M3_L128", 2, 512, 512, "heat", 1e-2, 0.0, 0.0, 1.0, 128, 3,
               "fourier2d", "adaptive", None, 8),
    5: Problem("cfg5_adv2d_1024x1024_M4_L512", 2, 1024, 1024, "advection", 0.0, 1.0, 0.5, 1.0, 512, 4,
               "gauss2d", "adaptive", None, 10),
}


def reduced(cfg: int) -> Problem:
    """Same PDE/method/u0 recipe as config `cfg` at a size the oracle finishes in seconds,
    still spanning several kernel tiles (parity tests)."""
    p = CONFIGS[cfg]
    if cfg in (1, 2):
        return p
    if cfg == 3:
        return p.replace(name="red3_heat1d_N4096_M3_L32", nx=4096, L=32)
    if cfg == 4:
        return p.replace(name="red4_heat2d_64x64_M3_L16", nx=64, ny=64, L=16, u0_kind="fourier2d_small")
    if cfg == 5:
        return p.replace(name="red5_adv2d_64x64_M4_L32", nx=64, ny=64, L=32)
    raise KeyError(cfg)


def edge_cases():
    """Degenerate / ragged parity cases (all small)."""
    base = Problem("edge", 1, 16, 1, "heat", 1.0, 0.0, 0.0, 0.5, 4, 2, "random", "fixed", 1e-3, 3)
    return [
        base.replace(name="edge_M1_implicit_euler", M=1),
        base.replace(name="edge_L1", L=1, alpha_fixed=0.2),
        base.replace(name="edge_L2_N4", L=2, nx=4),
        base.replace(name="edge_adv_M3_L8_N8", op="advection", cx=-0.7, nu=0.0, M=3, L=8, nx=8),
        base.replace(name="edge_M5_L16_N32", M=5, L=16, nx=32, alpha_fixed=1e-2),
        base.replace(name="edge_2d_heat_4x8", dim=2, nx=8, ny=4, M=2, L=4),
        base.replace(name="edge_2d_adv_16x8_M3", dim=2, nx=16, ny=8, op="advection", nu=0.0,
                     cx=1.0, cy=-0.5, M=3, L=8),
    ]


def discretisation_cases():
    """The paper's other spatial discretisations (Tables 1-2; reading R14) at
    parity size: the Table 2 pairings (heat: kappa 2/4/6 with M 1/2/3; advection u_t + u_x + u_y = 0
    (P:715-718), upwind kappa 1/3/5 with M 1/2/3) on small periodic grids, L = 16 steps of
    dT = T_64/64, plus 1-D variants, a two-pass 1-D size, a smem-engine 2-D shape and a mirrored
    (c < 0) upwind stencil.  Seeded random u0 (complex) unless stated."""
    heat = Problem("disc", 2, 32, 32, "heat", 1.0, 0.0, 0.0, 0.16 / 4, 16, 2, "random", "fixed", 1e-3, 3)
    adv = heat.replace(op="upwind1", nu=0.0, cx=1.0, cy=1.0)
    out = []
    for op, M, T64 in (("heat", 1, 0.32), ("heat4", 2, 0.16), ("heat6", 3, 0.16)):
        out.append(heat.replace(name=f"disc_{op}_2d_M{M}", op=op, M=M, T=T64 / 4))
        out.append(heat.replace(name=f"disc_{op}_1d_M{M}", op=op, M=M, T=T64 / 4, dim=1, nx=128, ny=1))
    for op, M, T64 in (("upwind1", 1, 0.00016), ("upwind3", 2, 0.00064), ("upwind5", 3, 0.0128)):
        out.append(adv.replace(name=f"disc_{op}_2d_M{M}", op=op, M=M, T=T64 / 4))
        out.append(adv.replace(name=f"disc_{op}_1d_M{M}", op=op, M=M, T=T64 / 4, dim=1, nx=128, ny=1, cy=0.0))
    # stiffer advection (|s c n| ~ 10) and flow to the left (mirrored stencils)
    out.append(adv.replace(name="disc_upwind5_1d_neg_stiff", op="upwind5", M=3, T=1.0, cx=-1.0, cy=0.0,
                           dim=1, nx=128, ny=1))
    out.append(adv.replace(name="disc_upwind3_2d_mixed_sign", op="upwind3", M=2, T=0.05, cx=0.8, cy=-0.6))
    # two-pass 1-D PCR (class pass + chunk pass with halo F R) and a 2-D shape served by the
    # smem-engine kernels (|log nx - log ny| > 1)
    out.append(heat.replace(name="disc_heat6_1d_N16384", op="heat6", M=2, T=0.01, dim=1, nx=16384, ny=1,
                            L=4, nu=1e-2))
    out.append(adv.replace(name="disc_upwind5_1d_N16384", op="upwind5", M=2, T=0.01, dim=1, nx=16384, ny=1,
                           L=4, cy=0.0))
    out.append(heat.replace(name="disc_heat4_2d_64x8", op="heat4", M=2, nx=64, ny=8))
    out.append(heat.replace(name="disc_heat6_2d_M8", op="heat6", M=8, nx=16, ny=16, L=4, T=0.01))
    return out


def halo_box_cases():
    """2-D grids wide and tall enough (256 x 32, residual blocks of 64 x 8) to have residual blocks
    whose halo does not wrap the periodic boundary next to blocks whose halo does, for every halo
    width of the paper's stencils (1: kappa 2, upwind 1; 2: kappa 4, upwind 3; 3: kappa 6, upwind 5,
    with a mirrored one): the two staging paths of the residual kernel side by side.  L = 4, seeded
    random complex u0."""
    base = Problem("halo", 2, 256, 32, "heat", 1e-2, 0.0, 0.0, 0.02, 4, 2, "random", "fixed", 1e-3, 2)
    out = [base.replace(name=f"halo_{op}_M{M}", op=op, M=M) for op, M in (("heat", 1), ("heat4", 2), ("heat6", 3))]
    adv = base.replace(nu=0.0, cx=1.0, cy=-0.5, T=0.002)
    out += [adv.replace(name=f"halo_{op}_M{M}", op=op, M=M) for op, M in (("upwind1", 4), ("upwind3", 2), ("upwind5", 3))]
    return out


def table_cases():
    """The paper's own test problems at their Table 1/2 sizes:
    heat u_t = Laplace(u) (nu = 1, centred kappa 2/4/6) and advection u_t + u_x + u_y = 0 (upwind
    kappa 1..5) on the periodic unit square, with the printed N (7-smooth, mostly not
    powers of two: 300, 350, 400, 450, 490, 700, 800), kappa, M, L and T (Table 1) or dT = T_64/64
    (Table 2).  2-D grids are N x N, the 1-D variants N points.  Seeded random complex u0 (every
    spatial mode excited; the forcing of P:706-712 is not needed for parity), fixed alpha."""
    heat = Problem("tab", 2, 8, 8, "heat", 1.0, 0.0, 0.0, 0.1, 32, 1, "random", "fixed", 1e-3, 2)
    adv = heat.replace(op="upwind2", nu=0.0, cx=1.0, cy=1.0)
    out = []
    # Table 1: heat T = 0.1, advection T = 1e-2
    for N, kap, M, L in ((450, 2, 1, 32), (400, 4, 2, 32), (300, 6, 3, 16)):
        op = {2: "heat", 4: "heat4", 6: "heat6"}[kap]
        out.append(heat.replace(name=f"t1_heat_k{kap}_N{N}", op=op, nx=N, ny=N, M=M, L=L, T=0.1))
    for N, kap, M, L in ((350, 2, 2, 8), (350, 4, 2, 16), (490, 5, 3, 32)):
        out.append(adv.replace(name=f"t1_adv_k{kap}_N{N}", op=f"upwind{kap}", nx=N, ny=N, M=M, L=L, T=1e-2))
    # Table 2: dT = T_64 / 64, here L = 8 steps of it
    for N, kap, M, T64 in ((350, 2, 1, 0.32), (400, 4, 2, 0.16), (350, 6, 3, 0.16)):
        op = {2: "heat", 4: "heat4", 6: "heat6"}[kap]
        out.append(heat.replace(name=f"t2_heat_k{kap}_N{N}", op=op, nx=N, ny=N, M=M, L=8, T=8 * T64 / 64))
    for N, kap, M, T64 in ((800, 1, 1, 0.00016), (800, 3, 2, 0.00064), (700, 5, 3, 0.0128)):
        out.append(adv.replace(name=f"t2_adv_k{kap}_N{N}", op=f"upwind{kap}", nx=N, ny=N, M=M, L=8, T=8 * T64 / 64))
    # 1-D variants of every entry (N points)
    out += [p.replace(name=p.name + "_1d", dim=1, ny=1, cy=0.0) for p in list(out)]
    return out

