"""One alpha-circulant preconditioned Richardson iteration (oracle; test infrastructure only).

Definition (PAPER.md, with the block matrix of P:115-135 — DESIGN.md reading R2):
    C     = I_L (x) C_coll + E (x) H,      C_coll = I_MN - dT Q (x) A,  H = H_M (x) I_N
    C_a   = I_L (x) C_coll + E_a (x) H     (eq. prec)
    w     = (u0 + v_1, v_2, ..., v_L),     v_l = dT (Q (x) I) b_l, b_l[m] = b(t_l + tau_m dT)
            (P:105); v = 0 in every config (b == 0), optional forcing otherwise
and the iteration, in correction form (reading R1; algebraically eq. Riteration):
    u^{k+1} = u^k + C_{a_k}^{-1} (w - C u^k).
C_a^{-1} is applied exactly as the paper's three steps s1-s3 with
V^{-1} = F* J^{-1}, V = J F / L (Lemma P:164-171; 0-based index reading R3), and the
block-diagonal step s2 solved DIRECTLY per frequency, (G_k (x) I_N - dT Q (x) A) y_k = x_k
with G_k = I_M + d_k H_M (eq. inner1) — by dense LU ("dense" tier), by spatial FFT +
M x M LU per mode ("fourier" tier, exact because A is circulant), or for a subset of spatial
Fourier modes only ("mode" tier: every spatial mode is an independent L*M problem).
The oracle never forms S_k, never uses PCR and never uses an FFT in time: the time transforms
are naive L x L DFT matrices with integer-reduced twiddles (reading R5).

Array layout: u[l][m][n], complex128, l in [0,L), m in [0,M), n = y*nx + x.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .collocation import Tableau
from .operators import apply_A, dense_A, symbol


# ---------------------------------------------------------------------------------------------
# time transforms (Lemma P:164-171)

def twiddle(L: int, sign: int) -> np.ndarray:
    """T[k, l] = exp(sign * 2 pi i ((l k) mod L) / L), index reduced in integers (reading R5)."""
    l = np.arange(L, dtype=np.int64)
    q = np.outer(l, l) % L
    ang = 2.0 * np.pi * q.astype(np.float64) / L
    return np.cos(ang) + 1j * sign * np.sin(ang)


def V_inverse(L: int, alpha: float) -> np.ndarray:
    """V^{-1}[k, l] = exp(-2 pi i k l / L) alpha^{l/L}   (V^{-1} = F* J^{-1}, J = diag(alpha^{-l/L}))."""
    scale = alpha ** (np.arange(L) / L)
    return twiddle(L, -1) * scale[None, :]


def V_matrix(L: int, alpha: float) -> np.ndarray:
    """V[l, k] = alpha^{-l/L} exp(+2 pi i l k / L) / L   (V = J F / L)."""
    scale = alpha ** (-np.arange(L) / L) / L
    return twiddle(L, +1) * scale[:, None]


def d_values(L: int, alpha: float) -> np.ndarray:
    """d_k = -alpha^{1/L} exp(-2 pi i k / L), k = 0..L-1 (Lemma P:167, 0-based)."""
    k = np.arange(L)
    ang = 2.0 * np.pi * k / L
    return -(alpha ** (1.0 / L)) * (np.cos(ang) - 1j * np.sin(ang))


def time_apply(T: np.ndarray, v: np.ndarray) -> np.ndarray:
    """(T (x) I) v for an L x L matrix T acting on the leading (time) axis of v[l][...]: one complex
    GEMM (L x L) . (L x M*N) — the naive DFT of SURVEY §8(c) O2/O4 (no FFT)."""
    return (T @ v.reshape(v.shape[0], -1)).reshape((T.shape[0],) + v.shape[1:])


def E_matrix(L: int, alpha: float | None = None) -> np.ndarray:
    """E (alpha None): -1 on the sub-diagonal; E_alpha: plus -alpha in the corner."""
    E = np.zeros((L, L))
    for l in range(1, L):
        E[l, l - 1] = -1.0
    if alpha is not None:
        E[0, L - 1] += -alpha
    return E


# ---------------------------------------------------------------------------------------------
# residual (step (i))

def w_vector(p, u0: np.ndarray, v: np.ndarray | None = None) -> np.ndarray:
    """w = (u0 replicated over the M nodes + v_1, v_2, ..., v_L); v = None: b == 0."""
    w = np.zeros((p.L, p.M, p.N), dtype=np.complex128) if v is None else np.array(v, dtype=np.complex128)
    w[0, :, :] += u0[None, :]
    return w


def forcing_vector(p, tab: Tableau, b) -> np.ndarray:
    """v_l = dT (Q (x) I) b_l with b_l[m] = b(t_l + tau_m dT) (collocation integral of the forcing,
    P:105); b(t) returns the N-vector b(., t)."""
    bl = np.array([[b((l + tab.t[m]) * p.dT) for m in range(p.M)] for l in range(p.L)], dtype=np.complex128)
    return p.dT * np.einsum("mj,ljn->lmn", tab.Q, bl)


def apply_C(p, tab: Tableau, u: np.ndarray) -> np.ndarray:
    """C u = (I_L (x) C_coll + E (x) H) u, block by block."""
    Au = apply_A(p, u)                                       # (L, M, N)
    QAu = np.matmul(tab.Q, Au)                               # Q (x) I over the node axis
    Cu = u - p.dT * QAu
    Hu_prev = np.zeros_like(u)
    Hu_prev[1:, :, :] = u[:-1, p.M - 1, :][:, None, :]       # H u_{l-1}: last node to every node
    return Cu - Hu_prev                                      # E has -1 on the sub-diagonal


def residual(p, tab: Tableau, u: np.ndarray, u0: np.ndarray, v: np.ndarray | None = None) -> np.ndarray:
    """r = w - C u."""
    return w_vector(p, u0, v) - apply_C(p, tab, u)


# ---------------------------------------------------------------------------------------------
# block-diagonal solve (step s2 / eq. inner1)

class DenseBlockSolver:
    """(G_k (x) I_N - dT Q (x) A) y_k = x_k by dense LU on the MN x MN block (tiny N)."""

    def __init__(self, p, tab: Tableau):
        self.p, self.tab = p, tab
        self.A = dense_A(p)
        self._cache = {}

    def solve(self, alpha: float, x: np.ndarray) -> np.ndarray:
        p, tab = self.p, self.tab
        d = d_values(p.L, alpha)
        y = np.empty_like(x)
        I_N = np.eye(p.N)
        for k in range(p.L):
            key = (alpha, k)
            if key not in self._cache:
                G = np.eye(p.M) + d[k] * tab.H
                B = np.kron(G, I_N) - p.dT * np.kron(tab.Q, self.A)
                self._cache[key] = sla.lu_factor(B)
            y[k] = sla.lu_solve(self._cache[key], x[k].reshape(-1)).reshape(p.M, p.N)
        return y


class FourierBlockSolver:
    """Same block solve via the spatial DFT: A is circulant, so each spatial mode kappa gives
    an independent M x M system (G_k - dT lambda_kappa Q) yhat = xhat (LU with pivoting)."""

    def __init__(self, p, tab: Tableau):
        self.p, self.tab = p, tab
        kx = np.arange(p.nx)[None, :]
        ky = np.arange(p.ny)[:, None]
        self.lam = np.broadcast_to(symbol(p, kx, ky), (p.ny, p.nx)).reshape(-1)

    def solve(self, alpha: float, x: np.ndarray) -> np.ndarray:
        p, tab = self.p, self.tab
        d = d_values(p.L, alpha)
        xs = x.reshape(p.L, p.M, p.ny, p.nx)
        xh = np.fft.fft2(xs, axes=(-2, -1)).reshape(p.L, p.M, p.N)
        yh = np.empty_like(xh)
        for k in range(p.L):
            G = np.eye(p.M) + d[k] * tab.H
            B = G[None, :, :] - p.dT * self.lam[:, None, None] * tab.Q[None, :, :]   # (N, M, M)
            yh[k] = np.linalg.solve(B, xh[k].T[:, :, None])[:, :, 0].T
        y = np.fft.ifft2(yh.reshape(p.L, p.M, p.ny, p.nx), axes=(-2, -1))
        return y.reshape(p.L, p.M, p.N)


# ---------------------------------------------------------------------------------------------
# one iteration (Alg. 1 order: residual, J^-1 + DFT, block solves, inverse DFT + J, update)

class Oracle:
    def __init__(self, p, u0: np.ndarray, tier: str = "auto", v: np.ndarray | None = None):
        self.p = p
        self.tab = Tableau(p.M)
        self.u0 = np.asarray(u0, dtype=np.complex128)
        self.v = v                                          # forcing part of w (None: b == 0)
        if tier == "auto":
            tier = "dense" if p.M * p.N <= 2048 else "fourier"
        self.tier = tier
        self.solver = DenseBlockSolver(p, self.tab) if tier == "dense" else FourierBlockSolver(p, self.tab)

    def initial(self) -> np.ndarray:
        """u^(0) = u0 replicated over all (l, m)."""
        return np.broadcast_to(self.u0, (self.p.L, self.p.M, self.p.N)).copy()

    def iterate(self, u: np.ndarray, alpha: float) -> np.ndarray:
        p = self.p
        r = residual(p, self.tab, u, self.u0, self.v)                       # (i)
        x = time_apply(V_inverse(p.L, alpha), r)              # (ii)  eq. s1
        y = self.solver.solve(alpha, x)                                     # (iii)-(iv) eq. s2
        c = time_apply(V_matrix(p.L, alpha), y)               # (v)   eq. s3
        return u + c

    def iterate_direct(self, u: np.ndarray, alpha: float) -> np.ndarray:
        """Alg. 1 as printed (eq. Riteration): u^{k+1} = C_a^{-1} ((C_a - C) u + w).
        (C_a - C) u + w = w - alpha e_1 (x) H u_L: only block 0 of (C_a - C) u is non-zero."""
        p = self.p
        r = w_vector(p, self.u0, self.v)
        r[0, :, :] -= alpha * u[p.L - 1, p.M - 1, :][None, :]
        x = time_apply(V_inverse(p.L, alpha), r)
        y = self.solver.solve(alpha, x)
        return time_apply(V_matrix(p.L, alpha), y)

    def residual_norms(self, u: np.ndarray):
        r = residual(self.p, self.tab, u, self.u0, self.v)
        return float(np.linalg.norm(r.ravel())), float(np.abs(r).max())


# ---------------------------------------------------------------------------------------------
# per-mode tier: the whole iteration for selected spatial Fourier modes

def mode_coefficients(p, v: np.ndarray, kx: np.ndarray, ky: np.ndarray) -> np.ndarray:
    """vhat(kappa) = sum_n v[..., n] exp(-2 pi i (kx x/nx + ky y/ny)) (numpy fft convention),
    evaluated directly (one O(N) sum per mode)."""
    xs = np.arange(p.nx, dtype=np.int64)
    ys = np.arange(p.ny, dtype=np.int64)
    out = []
    vv = v.reshape(v.shape[:-1] + (p.ny, p.nx))
    for a, b in zip(np.atleast_1d(kx), np.atleast_1d(ky)):
        ex = np.exp(-2j * np.pi * ((int(a) * xs) % p.nx) / p.nx)
        ey = np.exp(-2j * np.pi * ((int(b) * ys) % p.ny) / p.ny)
        out.append(np.einsum("...yx,y,x->...", vv, ey, ex))
    return np.stack(out, axis=-1)


class ModeOracle:
    """The iteration restricted to spatial modes kappa: each is the L*M problem with A -> lambda_kappa
    (exact by linearity since A is circulant).  uhat[l][m][j] for mode j."""

    def __init__(self, p, u0hat: np.ndarray, kx, ky):
        self.p = p
        self.tab = Tableau(p.M)
        self.kx = np.atleast_1d(np.asarray(kx))
        self.ky = np.atleast_1d(np.asarray(ky))
        self.lam = symbol(p, self.kx, self.ky)
        self.u0hat = np.asarray(u0hat, dtype=np.complex128)

    def initial(self) -> np.ndarray:
        return np.broadcast_to(self.u0hat, (self.p.L, self.p.M, len(self.lam))).copy()

    def residual(self, uh: np.ndarray) -> np.ndarray:
        p, tab = self.p, self.tab
        w = np.zeros_like(uh)
        w[0] = self.u0hat[None, :]
        Cu = uh - p.dT * self.lam[None, None, :] * np.matmul(tab.Q, uh)
        Cu[1:] -= uh[:-1, p.M - 1, :][:, None, :]
        return w - Cu

    def iterate_direct(self, uh: np.ndarray, alpha: float) -> np.ndarray:
        """Direct form for the sampled modes: uh^{k+1} = C_a(lam)^{-1} (w - alpha e_1 (x) H uh_L)."""
        p = self.p
        r = np.zeros_like(uh)
        r[0] = self.u0hat[None, :] - alpha * uh[p.L - 1, p.M - 1, :][None, :]
        return self._solve_ca(r, alpha)

    def _solve_ca(self, r: np.ndarray, alpha: float) -> np.ndarray:
        p, tab = self.p, self.tab
        x = time_apply(V_inverse(p.L, alpha), r)
        d = d_values(p.L, alpha)
        y = np.empty_like(x)
        for k in range(p.L):
            G = np.eye(p.M) + d[k] * tab.H
            B = G[None, :, :] - p.dT * self.lam[:, None, None] * tab.Q[None, :, :]
            y[k] = np.linalg.solve(B, x[k].T[:, :, None])[:, :, 0].T
        return time_apply(V_matrix(p.L, alpha), y)

    def iterate(self, uh: np.ndarray, alpha: float) -> np.ndarray:
        p, tab = self.p, self.tab
        r = self.residual(uh)
        x = time_apply(V_inverse(p.L, alpha), r)
        d = d_values(p.L, alpha)
        y = np.empty_like(x)
        for k in range(p.L):
            G = np.eye(p.M) + d[k] * tab.H
            B = G[None, :, :] - p.dT * self.lam[:, None, None] * tab.Q[None, :, :]
            y[k] = np.linalg.solve(B, x[k].T[:, :, None])[:, :, 0].T
        c = time_apply(V_matrix(p.L, alpha), y)
        return uh + c


# ---------------------------------------------------------------------------------------------
# independent pins: brute force, sequential stepping, closed form

def assemble_C(p, tab: Tableau, alpha: float | None = None) -> np.ndarray:
    """Dense C (alpha None) or C_alpha from their Kronecker definitions; tiny sizes only."""
    A = dense_A(p)
    Ccoll = np.eye(p.M * p.N) - p.dT * np.kron(tab.Q, A)
    H = np.kron(tab.H, np.eye(p.N))
    return np.kron(np.eye(p.L), Ccoll) + np.kron(E_matrix(p.L, alpha), H)


def brute_force_iterate_direct(p, tab: Tableau, u: np.ndarray, u0: np.ndarray, alpha: float,
                               v: np.ndarray | None = None) -> np.ndarray:
    """u^{k+1} = solve(C_a, (C_a - C) u + w) with C, C_a assembled densely (eq. Riteration)."""
    C = assemble_C(p, tab)
    Ca = assemble_C(p, tab, alpha)
    w = w_vector(p, u0, v).reshape(-1)
    return np.linalg.solve(Ca, (Ca - C) @ u.reshape(-1) + w).reshape(u.shape)


def brute_force_iterate(p, tab: Tableau, u: np.ndarray, u0: np.ndarray, alpha: float,
                        v: np.ndarray | None = None) -> np.ndarray:
    C = assemble_C(p, tab)
    Ca = assemble_C(p, tab, alpha)
    w = w_vector(p, u0, v).reshape(-1)
    uf = u.reshape(-1)
    return (uf + np.linalg.solve(Ca, w - C @ uf)).reshape(u.shape)


def sequential_solution(p, tab: Tableau, u0: np.ndarray, v: np.ndarray | None = None) -> np.ndarray:
    """u* of C u = w by L sequential collocation steps:
    (I - dT Q (x) A) u_l = 1 (x) u_{l-1, M-1} + v_l,  u_{-1, M-1} := u0.  Spatial-FFT solve per step."""
    lam = FourierBlockSolver(p, tab).lam
    B = np.eye(p.M)[None] - p.dT * lam[:, None, None] * tab.Q[None]      # (N, M, M)
    out = np.empty((p.L, p.M, p.N), dtype=np.complex128)
    prev = np.asarray(u0, dtype=np.complex128)
    for l in range(p.L):
        rhs = np.fft.fft2(prev.reshape(p.ny, p.nx)).reshape(-1)
        rhs = np.repeat(rhs[:, None], p.M, axis=1)                        # (N, M)
        if v is not None:
            rhs = rhs + np.fft.fft2(v[l].reshape(p.M, p.ny, p.nx), axes=(-2, -1)).reshape(p.M, p.N).T
        yh = np.linalg.solve(B, rhs[:, :, None])[:, :, 0]
        y = np.fft.ifft2(yh.T.reshape(p.M, p.ny, p.nx), axes=(-2, -1)).reshape(p.M, p.N)
        out[l] = y
        prev = y[p.M - 1]
    return out


def single_mode_solution(tab: Tableau, z: complex, L: int, uhat0: complex) -> np.ndarray:
    """u*_{l,m} = [(I - zQ)^{-1} 1]_m R(z)^{l+1} / R(z) * uhat0 for one spatial eigenmode, z = dT lambda:
    stage values s = (I - zQ)^{-1} 1 of one collocation step, R(z) = s_{M-1} (stability function)."""
    M = tab.M
    s = np.linalg.solve(np.eye(M) - z * tab.Q, np.ones(M))
    R = s[M - 1]
    return np.array([[s[m] * R ** l * uhat0 for m in range(M)] for l in range(L)])


def relative_l2(a: np.ndarray, b: np.ndarray) -> float:
    """||a - b||_2 / ||b||_2 over all entries."""
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))
