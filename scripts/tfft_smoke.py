"""Parity of the pipelined time transforms (L >= 128) on 2-D shapes, both forms, vs the oracle."""
import numpy as np
import paper_2103_12571_b200 as P
import workloads as W
from oracle.paralpha import Oracle, relative_l2

cases = [W.CONFIGS[4].replace(name="t512_L128_M3", L=128, nx=64, ny=64),
         W.CONFIGS[5].replace(name="t1024_L256_M2", L=256, nx=128, ny=64, M=2),
         W.CONFIGS[5].replace(name="t512_L512_M1", L=512, nx=64, ny=32, M=1),
         W.CONFIGS[5].replace(name="t1024_L1024_M1", L=1024, nx=32, ny=32, M=1)]
for p in cases:
    rng = np.random.default_rng(3)
    u0 = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
    for form in ("correction", "direct"):
        s = P.Solver(p, u0)
        s.set_form(form)
        s.set_alpha_schedule([1e-2, 5e-2])
        o = Oracle(p, u0, "fourier")
        u = o.initial()
        errs = []
        for k in range(2):
            u = o.iterate(u, [1e-2, 5e-2][k]) if form == "correction" else o.iterate_direct(u, [1e-2, 5e-2][k])
            d = s.iterate(1, want_diff=True)[0]
            errs.append(relative_l2(s.get_iterate(), u))
        print(p.name, form, s.kernel_names()[1], s.kernel_names()[-1], ["%.2e" % e for e in errs], flush=True)
        s.close()
