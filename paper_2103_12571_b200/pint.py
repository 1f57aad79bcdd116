"""Thin ctypes binding of libpint (include/pint.h).  Argument marshalling only: every step of the
iteration runs in the library's CUDA kernels.  PyTorch supplies device memory and the stream.

There is NO fallback: if libpint.so is missing or no CUDA device is present the product path
raises.  (The CPU oracle lives in oracle/ and is test infrastructure only.)
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PINT_LIBRARY selects another build of the same ABI (A/B runs against libpint_exp.so only);
# bench.py records pint_experiments_enabled() and refuses an experiments build by default
LIB_PATH = os.environ.get("PINT_LIBRARY") or os.path.join(HERE, "libpint.so")

PINT_OK = 0
STATUS = {0: "PINT_OK", 1: "PINT_ERR_INVALID", 2: "PINT_ERR_SCHEDULE", 3: "PINT_ERR_NOT_DIAGONALIZABLE",
          4: "PINT_ERR_NUMERIC", 5: "PINT_ERR_CUDA", 6: "PINT_ERR_NCCL", 7: "PINT_ERR_STATE"}
OPS = {"heat": 0, "advection": 1, "heat4": 2, "heat6": 3, "upwind1": 4, "upwind3": 5, "upwind5": 6,
       "upwind2": 7, "upwind4": 8}
MAX_SCHEDULE = 64

# every symbol include/pint.h declares (checked by tests/test_abi.py)
EXPORTS = ["pint_workspace_bytes", "pint_create", "pint_adaptive_schedule", "pint_w_inf",
           "pint_set_alpha_schedule", "pint_iterate", "pint_residual_norm", "pint_get_iterate",
           "pint_get_final_value", "pint_set_initial_value", "pint_destroy", "pint_last_error",
           "pint_abi_version", "pint_launches_per_iteration", "pint_get_factors", "pint_tableau",
           "pint_debug_stage", "pint_debug_get_work", "pint_iterate_profiled", "pint_kernel_name",
           "pint_nccl_unique_id", "pint_local_steps", "pint_group_iterate", "pint_group_residual_norm",
           "pint_set_form", "pint_set_hermitian", "pint_solve", "pint_sequential", "pint_set_forcing",
           "pint_next_window", "pint_experiments_enabled", "pint_graph_create", "pint_graph_launch",
           "pint_graph_destroy", "pint_set_phase_timing", "pint_phase_times"]
FORMS = {"correction": 0, "direct": 1}


class PintError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Problem(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("op", ctypes.c_int32), ("nu", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("T", ctypes.c_double), ("L", ctypes.c_int32),
                ("M", ctypes.c_int32)]


class Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p),
                ("device", ctypes.c_int32), ("stream", ctypes.c_void_p)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Loads libpint.so (raises if missing — there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libpint.so not built at {path}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, D, vp, dp = ctypes.POINTER(Problem), ctypes.POINTER(Dist), ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)
    i32 = ctypes.c_int32
    sig = {
        "pint_workspace_bytes": (ctypes.c_size_t, [P, D]),
        "pint_create": (i32, [P, D, vp, vp, ctypes.c_size_t, dp, dp, ctypes.POINTER(vp)]),
        "pint_adaptive_schedule": (i32, [i32, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                         i32, dp, dp]),
        "pint_w_inf": (i32, [vp, dp]),
        "pint_set_alpha_schedule": (i32, [vp, dp, i32]),
        "pint_iterate": (i32, [vp, i32, dp]),
        "pint_residual_norm": (i32, [vp, dp, dp]),
        "pint_get_iterate": (i32, [vp, dp]),
        "pint_get_final_value": (i32, [vp, dp]),
        "pint_set_initial_value": (i32, [vp, dp, i32]),
        "pint_destroy": (i32, [vp]),
        "pint_last_error": (ctypes.c_char_p, []),
        "pint_abi_version": (i32, []),
        "pint_experiments_enabled": (i32, []),
        "pint_launches_per_iteration": (i32, [vp]),
        "pint_get_factors": (i32, [vp, i32, i32, dp, dp, dp, dp]),
        "pint_tableau": (i32, [i32, dp, dp]),
        "pint_debug_stage": (i32, [vp, i32, i32]),
        "pint_debug_get_work": (i32, [vp, i32, dp]),
        "pint_iterate_profiled": (i32, [vp, i32, dp]),
        "pint_kernel_name": (ctypes.c_char_p, [vp, i32]),
        "pint_nccl_unique_id": (i32, [vp]),
        "pint_local_steps": (i32, [vp, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)]),
        "pint_group_iterate": (i32, [ctypes.POINTER(vp), i32, i32, dp]),
        "pint_group_residual_norm": (i32, [ctypes.POINTER(vp), i32, dp, dp]),
        "pint_set_form": (i32, [vp, i32]),
        "pint_set_hermitian": (i32, [vp, i32]),
        "pint_solve": (i32, [vp, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, i32,
                             ctypes.POINTER(i32), dp, dp, ctypes.POINTER(i32)]),
        "pint_sequential": (i32, [vp]),
        "pint_set_forcing": (i32, [vp, vp]),
        "pint_next_window": (i32, [vp]),
        "pint_graph_create": (i32, [vp, i32, ctypes.POINTER(vp)]),
        "pint_graph_launch": (i32, [vp, vp]),
        "pint_graph_destroy": (i32, [vp]),
        "pint_set_phase_timing": (i32, [vp, i32]),
        "pint_phase_times": (i32, [vp, dp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def experiments_enabled() -> bool:
    """True for an A/B build with the PINT_* environment switches compiled in (never the product)."""
    return bool(load_library().pint_experiments_enabled())


def _check(st: int):
    if st != PINT_OK:
        raise PintError(st, _lib.pint_last_error().decode())


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def make_problem(p) -> Problem:
    """p: any object with dim, nx, ny, op, nu, cx, cy, T, L, M (e.g. workloads.Problem)."""
    return Problem(p.dim, p.nx, p.ny if p.dim == 2 else 1, OPS[p.op], p.nu, p.cx, p.cy, p.T, p.L, p.M)


def tableau(M: int):
    lib = load_library()
    t = np.zeros(M)
    Q = np.zeros((M, M))
    _check(lib.pint_tableau(M, _dp(t), _dp(Q)))
    return t, Q


def adaptive_schedule(L: int, w_inf: float, m0: float, K: int, eps: float = 2.0 ** -52, tau: float = 0.0):
    lib = load_library()
    a = np.zeros(max(K, 1))
    m = np.zeros(K + 1)
    _check(lib.pint_adaptive_schedule(L, w_inf, m0, eps, tau, K, _dp(a), _dp(m)))
    return a[:K].copy(), m


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; the caller broadcasts it)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(lib.pint_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


class Solver:
    """One Paralpha context on one GPU (one rank).  Device buffers are torch tensors (complex128).

    nranks > 1 shards the time steps cyclically (rank r owns global steps r + nranks*j); with an
    nccl_id the ranks exchange over NCCL, without one the context is a virtual rank of a
    single-process loopback Group."""

    def __init__(self, problem, u0: np.ndarray, device: int = 0, stream=None, rank: int = 0, nranks: int = 1,
                 nccl_id: Optional[bytes] = None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("pint needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.problem = problem
        self.cp = make_problem(problem)
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._id = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        self.dist = Dist(rank, nranks, ctypes.cast(self._id, ctypes.c_void_p) if self._id is not None else None,
                         device, ctypes.c_void_p(self.stream.cuda_stream))
        self.rank, self.nranks = rank, nranks
        nbytes = self.lib.pint_workspace_bytes(ctypes.byref(self.cp), ctypes.byref(self.dist))
        if nbytes == 0:
            raise PintError(1, self.lib.pint_last_error().decode())
        self.L, self.M, self.N = problem.L // nranks, problem.M, problem.nx * (problem.ny if problem.dim == 2 else 1)
        self.u = torch.empty((self.L, self.M, self.N), dtype=torch.complex128, device=self.device)
        self.work = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        u0h = np.ascontiguousarray(np.asarray(u0, dtype=np.complex128)).view(np.float64)
        ctx = ctypes.c_void_p()
        _check(self.lib.pint_create(ctypes.byref(self.cp), ctypes.byref(self.dist), ctypes.c_void_p(self.u.data_ptr()),
                                    ctypes.c_void_p(self.work.data_ptr()), nbytes, _dp(u0h), None, ctypes.byref(ctx)))
        self.ctx = ctx
        self.workspace_bytes = nbytes

    # -- schedule
    def w_inf(self) -> float:
        v = ctypes.c_double()
        _check(self.lib.pint_w_inf(self.ctx, ctypes.byref(v)))
        return v.value

    def set_alpha_schedule(self, alphas: Sequence[float]):
        a = np.ascontiguousarray(np.asarray(alphas, dtype=np.float64))
        _check(self.lib.pint_set_alpha_schedule(self.ctx, _dp(a), len(a)))

    def set_form(self, form: str):
        """"correction" (default, u += C_a^{-1}(w - C u)) or "direct" (Alg. 1: u = C_a^{-1}((C_a - C)u + w))."""
        _check(self.lib.pint_set_form(self.ctx, FORMS[form]))

    def solve(self, m0: float, tol: float, max_iter: int, eps: float = 2.0 ** -52, tau: float = 0.0):
        """Algorithm 2: adaptive alphas, stop on consecutive iterates <= tol (C ABI)."""
        it, why = ctypes.c_int32(0), ctypes.c_int32(0)
        d = np.zeros(max_iter)
        m = np.zeros(max_iter + 1)
        _check(self.lib.pint_solve(self.ctx, m0, eps, tau, tol, max_iter, ctypes.byref(it), _dp(d), _dp(m),
                                   ctypes.byref(why)))
        n = it.value
        return {"iters": n, "diffs": d[:n], "m": m[:n + 1],
                "stop": ["consecutive iterates", "m_k <= tol", "max_iter", "m_k < 4 gamma"][why.value]}

    def set_forcing(self, v: Optional[np.ndarray]):
        """Attach w's forcing part v[l][m][n] (complex128, this rank's local steps; None removes it)."""
        import torch
        if v is None:
            _check(self.lib.pint_set_forcing(self.ctx, None))
            self.v = None
            return
        vv = np.ascontiguousarray(np.asarray(v, dtype=np.complex128).reshape(self.L, self.M, self.N))
        self.v = torch.from_numpy(vv).to(self.device)
        _check(self.lib.pint_set_forcing(self.ctx, ctypes.c_void_p(self.v.data_ptr())))

    def next_window(self):
        """Start the next window of L steps from the final value (windowed Paralpha)."""
        _check(self.lib.pint_next_window(self.ctx))

    def sequential(self):
        """Overwrite the iterate with the sequential Radau IIA solution (baseline)."""
        _check(self.lib.pint_sequential(self.ctx))

    def set_hermitian(self, on: bool = True):
        """Real-data fast path: solve only the frequencies k <= L/2 (y_{L-k} = conj(y_k)); while on,
        the device iterate is stored as real fp64 (see iterate_view)."""
        _check(self.lib.pint_set_hermitian(self.ctx, 1 if on else 0))
        self.hermitian = bool(on)

    def iterate_view(self):
        """The device iterate as a torch view: complex128 (L, M, N), or float64 (L, M, N) in the
        Hermitian mode (real storage in the first L*M*N doubles of the buffer)."""
        import torch
        if getattr(self, "hermitian", False):
            return self.u.view(-1).view(torch.float64)[: self.L * self.M * self.N].view(self.L, self.M, self.N)
        return self.u

    # -- iteration
    def iterate(self, n: int = 1, want_diff: bool = False):
        if want_diff:
            d = np.zeros(n)
            _check(self.lib.pint_iterate(self.ctx, n, _dp(d)))
            return d
        _check(self.lib.pint_iterate(self.ctx, n, None))
        return None

    PHASES = ("halo", "forward", "alltoall1_span", "middle", "midend_to_end", "fwd_end_to_alltoall2_done", "total")

    def set_phase_timing(self, on: bool = True):
        _check(self.lib.pint_set_phase_timing(self.ctx, 1 if on else 0))

    def phase_times(self) -> dict:
        """Per-phase ms of the last iteration (NCCL ranks, see include/pint.h)."""
        out = np.zeros(7)
        _check(self.lib.pint_phase_times(self.ctx, _dp(out)))
        return dict(zip(self.PHASES, out.tolist()))

    def graph_create(self, n: int):
        """Capture n iterations into a CUDA graph (launch-bound problems); returns a handle."""
        h = ctypes.c_void_p()
        _check(self.lib.pint_graph_create(self.ctx, n, ctypes.byref(h)))
        return h

    def graph_launch(self, h):
        _check(self.lib.pint_graph_launch(self.ctx, h))

    def graph_destroy(self, h):
        _check(self.lib.pint_graph_destroy(h))

    def residual_norm(self):
        a, b = ctypes.c_double(), ctypes.c_double()
        _check(self.lib.pint_residual_norm(self.ctx, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def get_iterate(self) -> np.ndarray:
        out = np.empty((self.L, self.M, self.N), dtype=np.complex128)
        _check(self.lib.pint_get_iterate(self.ctx, _dp(out.view(np.float64))))
        return out

    def get_final_value(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.N, dtype=np.complex128)
        _check(self.lib.pint_get_final_value(self.ctx, _dp(out.view(np.float64))))
        return out

    def set_initial_value(self, u0: np.ndarray, reset: bool = True):
        u0h = np.ascontiguousarray(np.asarray(u0, dtype=np.complex128)).view(np.float64)
        _check(self.lib.pint_set_initial_value(self.ctx, _dp(u0h), 1 if reset else 0))

    def launches_per_iteration(self) -> int:
        return int(self.lib.pint_launches_per_iteration(self.ctx))

    def kernel_names(self):
        return [self.lib.pint_kernel_name(self.ctx, i).decode() for i in range(self.launches_per_iteration())]

    def iterate_profiled(self, n: int) -> np.ndarray:
        """Average per-launch device time (ms) of each kernel of an iteration over n iterations."""
        out = np.zeros(self.launches_per_iteration())
        _check(self.lib.pint_iterate_profiled(self.ctx, n, _dp(out)))
        return out

    def factors(self, a: int, k: int):
        M = self.M
        dk = np.zeros(2)
        S = np.zeros(2 * M * M)
        Si = np.zeros(2 * M * M)
        dkm = np.zeros(2 * M)
        _check(self.lib.pint_get_factors(self.ctx, a, k, _dp(dk), _dp(S), _dp(Si), _dp(dkm)))
        c = lambda v: v.view(np.complex128)
        return c(dk)[0], c(S).reshape(M, M), c(Si).reshape(M, M), c(dkm)

    def debug_stage(self, a: int, s: int):
        _check(self.lib.pint_debug_stage(self.ctx, a, s))

    def debug_work(self, which: int) -> np.ndarray:
        out = np.empty((self.L, self.M, self.N), dtype=np.complex128)
        _check(self.lib.pint_debug_get_work(self.ctx, which, _dp(out.view(np.float64))))
        return out

    def local_steps(self):
        a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(self.lib.pint_local_steps(self.ctx, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.pint_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Group:
    """Single-process loopback group of P virtual ranks on one GPU (tests of the sharded path):
    the same kernels and phase sequence as the NCCL ranks, chunks moved by device copies."""

    def __init__(self, problem, u0: np.ndarray, P: int, device: int = 0):
        import torch
        self.P = P
        self.problem = problem
        stream = torch.cuda.current_stream(torch.device("cuda", device))
        self.ranks = [Solver(problem, u0, device=device, stream=stream, rank=r, nranks=P) for r in range(P)]
        self.lib = self.ranks[0].lib
        self._ctxs = (ctypes.c_void_p * P)(*[s.ctx.value for s in self.ranks])

    def set_alpha_schedule(self, alphas):
        for s in self.ranks:
            s.set_alpha_schedule(alphas)

    def set_form(self, form: str):
        for s in self.ranks:
            s.set_form(form)

    def iterate(self, n: int = 1, want_diff: bool = False):
        d = np.zeros(n) if want_diff else None
        _check(self.lib.pint_group_iterate(self._ctxs, self.P, n, _dp(d)))
        return d

    def residual_norm(self):
        a, b = ctypes.c_double(), ctypes.c_double()
        _check(self.lib.pint_group_residual_norm(self._ctxs, self.P, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def get_iterate(self) -> np.ndarray:
        """Global iterate u[l][m][n] gathered from the ranks (rank r holds l = r + P j)."""
        p = self.problem
        N = p.nx * (p.ny if p.dim == 2 else 1)
        out = np.empty((p.L, p.M, N), dtype=np.complex128)
        for s in self.ranks:
            first, stride, count = s.local_steps()
            out[first::stride] = s.get_iterate()
        return out

    def close(self):
        for s in self.ranks:
            s.close()
