"""Debug: 1-D spatial solve stage (PCR passes) against a numpy FFT solve per line at large N."""
import sys
import numpy as np
import paper_2103_12571_b200 as P
import workloads as W


def brev(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


for logN in [int(a) for a in sys.argv[1:]] or [16, 17, 18, 19, 20]:
    N = 1 << logN
    for op, nu, cx in (("heat", 1e-2, 0.0), ("advection", 0.0, 1.0)):
        p = W.CONFIGS[3].replace(name="dbg", nx=N, M=2, L=4, op=op, nu=nu, cx=cx, alpha_mode="fixed", alpha_fixed=1e-3)
        rng = np.random.default_rng(1)
        u0 = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        s = P.Solver(p, u0)
        s.set_alpha_schedule([1e-3])
        s.debug_stage(0, 0)
        X = s.debug_work(0)
        s.debug_stage(0, 1)
        X2 = s.debug_work(1)
        k = np.arange(N)
        lam = (-4 * nu * N * N * np.sin(np.pi * k / N) ** 2) if op == "heat" else (-1j * cx * N * np.sin(2 * np.pi * k / N))
        worst = 0.0
        for pp in range(p.L):
            kk = brev(pp, 2)
            _, _, _, dkm = s.factors(0, kk)
            for m in range(p.M):
                sh = dkm[m] * p.dT
                ref = np.fft.ifft(np.fft.fft(X[pp, m]) / (1 - sh * lam))
                e = np.linalg.norm(X2[pp, m] - ref) / np.linalg.norm(ref)
                worst = max(worst, e)
                if e > 1e-9:
                    bad = np.nonzero(np.abs(X2[pp, m] - ref) > 1e-6 * np.abs(ref).max())[0]
                    print(f"  N=2^{logN} {op} p={pp} m={m} err={e:.2e} bad idx {bad[:8]} .. count {len(bad)}")
        print(f"N=2^{logN} {op}: worst line error {worst:.2e}", flush=True)
        s.close()
