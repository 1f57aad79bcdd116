"""Debug: 2-D spatial solve stage (node transforms + FFT-diagonal solve) against numpy per slot."""
import sys
import numpy as np
import paper_2103_12571_b200 as P
import workloads as W


def brev(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


def check(p):
    rng = np.random.default_rng(1)
    u0 = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
    s = P.Solver(p, u0)
    print(p.name, s.kernel_names(), flush=True)
    s.set_alpha_schedule([1e-2])
    s.debug_stage(0, 0)
    X = s.debug_work(0)
    s.debug_stage(0, 1)
    X2 = s.debug_work(1)
    from oracle.operators import symbol
    kx = np.arange(p.nx)[None, :]
    ky = np.arange(p.ny)[:, None]
    lam = np.broadcast_to(symbol(p, kx, ky), (p.ny, p.nx))
    lb = int(np.log2(p.L))
    worst = 0
    for pp in range(p.L):
        k = brev(pp, lb)
        dk, S, Si, dkm = s.factors(0, k)
        r = dk / (1 + dk)
        SG = S.copy()
        SG = S - r * np.outer(np.ones(p.M), S[p.M - 1])   # (I - r H_M) S: row m minus r * last row
        x1 = (Si @ X[pp].reshape(p.M, -1)).reshape(p.M, p.ny, p.nx)
        x2 = np.empty_like(x1)
        for m in range(p.M):
            x2[m] = np.fft.ifft2(np.fft.fft2(x1[m]) / (1 - dkm[m] * p.dT * lam))
        y = (SG @ x2.reshape(p.M, -1)).reshape(p.M, -1)
        e = np.linalg.norm(X2[pp] - y) / np.linalg.norm(y)
        worst = max(worst, e)
        em = [np.linalg.norm(X2[pp, m] - y[m]) / np.linalg.norm(y[m]) for m in range(p.M)]
        # also: is the error explained by a missing / wrong node transform?  solve without nodes
        x2n = np.empty_like(x1)
        for m in range(p.M):
            x2n[m] = np.fft.ifft2(np.fft.fft2(X[pp, m].reshape(p.ny, p.nx)) / (1 - dkm[m] * p.dT * lam))
        en = np.linalg.norm(X2[pp] - x2n.reshape(p.M, -1)) / np.linalg.norm(x2n)
        print(f"  slot {pp} k={k} per-m {['%.1e' % v for v in em]} vs no-node {en:.1e}", flush=True)
        if e > 1e-10 and pp < 4:
            d = np.abs(X2[pp] - y).reshape(p.M, p.ny, p.nx)
            idx = np.argwhere(d > 1e-6 * np.abs(y).max())
            print(f"  slot {pp} err {e:.2e}, bad count {len(idx)}, first {idx[:6].tolist()}", flush=True)
    print(f"  worst slot error {worst:.2e}", flush=True)
    s.close()


for c in sys.argv[1:] or ["1024x1024x4"]:
    nx, ny, M = (int(v) for v in c.split("x"))
    check(W.CONFIGS[5].replace(name=f"dbg{c}", nx=nx, ny=ny, M=M, L=4, alpha_mode="fixed", alpha_fixed=1e-2))
