"""Quick parity + timing of the 2-D pipelined spatial passes on production-plan shapes."""
import time
import numpy as np
import paper_2103_12571_b200 as P
import workloads as W
from oracle.paralpha import Oracle, relative_l2

cases = [
    W.CONFIGS[5].replace(name="p1024_M4_L4", L=4, alpha_mode="fixed", alpha_fixed=1e-2),
    W.CONFIGS[4].replace(name="p512_M3_L4", L=4, alpha_mode="fixed", alpha_fixed=1e-2),
    W.CONFIGS[5].replace(name="p1024x512_M2_L4", ny=512, M=2, L=4, alpha_mode="fixed", alpha_fixed=1e-2),
    W.CONFIGS[5].replace(name="p512x1024_M1_L8", nx=512, M=1, L=8, alpha_mode="fixed", alpha_fixed=1e-2),
]
for p in cases:
    rng = np.random.default_rng(3)
    u0 = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
    s = P.Solver(p, u0)
    print(p.name, s.kernel_names(), flush=True)
    s.set_alpha_schedule([1e-2, 1e-2])
    o = Oracle(p, u0, "fourier")
    u = o.initial()
    for k in range(2):
        u = o.iterate(u, 1e-2)
        s.iterate(1)
        print(f"  iter {k}: rel l2 {relative_l2(s.get_iterate(), u):.3e}", flush=True)
    s.close()
