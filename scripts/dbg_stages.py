"""Debug: each stage of one iteration (forward / solve / backward) against numpy, any dim."""
import sys
import numpy as np
import paper_2103_12571_b200 as P
import workloads as W
from oracle.collocation import Tableau
from oracle.operators import symbol
from oracle import paralpha as PA


def brev(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


def check(p, alpha=1e-3, seed=1):
    rng = np.random.default_rng(seed)
    u0 = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
    s = P.Solver(p, u0)
    s.set_alpha_schedule([alpha])
    tab = Tableau(p.M)
    lb = int(np.log2(p.L))
    u = np.broadcast_to(u0, (p.L, p.M, p.N)).copy()
    r = PA.residual(p, tab, u, u0)
    x = PA.time_apply(PA.V_inverse(p.L, alpha), r)
    s.debug_stage(0, 0)
    X = s.debug_work(0)
    e0 = 0
    facs = {}
    for pp in range(p.L):
        k = brev(pp, lb)
        dk, S, Si, dkm = s.factors(0, k)
        facs[pp] = (k, dk, S, Si, dkm)
        ref = Si @ x[k]
        e0 = max(e0, np.linalg.norm(X[pp] - ref) / np.linalg.norm(ref))
    s.debug_stage(0, 1)
    X2 = s.debug_work(1)
    kx = np.arange(p.nx)[None, :]
    ky = np.arange(p.ny)[:, None]
    lam = np.broadcast_to(symbol(p, kx, ky), (p.ny, p.nx)).reshape(-1)
    e1 = 0
    for pp in range(p.L):
        k, dk, S, Si, dkm = facs[pp]
        for m in range(p.M):
            ref = np.fft.ifft2((np.fft.fft2(X[pp, m].reshape(p.ny, p.nx)).reshape(-1) / (1 - dkm[m] * p.dT * lam)).reshape(p.ny, p.nx)).reshape(-1)
            e1 = max(e1, np.linalg.norm(X2[pp, m] - ref) / np.linalg.norm(ref))
    s.debug_stage(0, 2)
    ug = s.get_iterate()
    y = np.empty((p.L, p.M, p.N), dtype=np.complex128)
    for pp in range(p.L):
        k, dk, S, Si, dkm = facs[pp]
        rk = dk / (1 + dk)
        SG = S - rk * np.outer(np.ones(p.M), S[p.M - 1])
        y[k] = SG @ X2[pp]
    c = PA.time_apply(PA.V_matrix(p.L, alpha), y)
    e2 = np.linalg.norm(ug - (u + c)) / np.linalg.norm(u + c)
    full = PA.Oracle(p, u0, "fourier").iterate(u, alpha)
    ef = np.linalg.norm(ug - full) / np.linalg.norm(full)
    print(f"{p.name}: fwd {e0:.2e}  solve {e1:.2e}  bwd {e2:.2e}  vs oracle iterate {ef:.2e}", flush=True)
    s.close()


for spec in sys.argv[1:]:
    logn, op = spec.split(":")
    N = 1 << int(logn)
    base = W.CONFIGS[3].replace(name=f"dbg_{spec}", nx=N, M=2, L=4, alpha_mode="fixed", alpha_fixed=1e-3)
    if op == "adv":
        base = base.replace(op="advection", nu=0.0, cx=1.0)
    check(base)
