"""Run one iteration of a case and save/compare the iterate (A/B between two library builds)."""
import sys
import numpy as np
import paper_2103_12571_b200 as P
import workloads as W

name, L, M, Pn, mode = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
p = W.CONFIGS[5].replace(L=L, M=M)
rng = np.random.default_rng(0)
u0 = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
s = P.Group(p, u0, Pn) if Pn > 1 else P.Solver(p, u0)
s.set_alpha_schedule([1e-3])
try:
    s.iterate(1)
    x = s.get_iterate()
except Exception as e:
    print(name, "FAILED", str(e)[:100])
    sys.exit(0)
f = f"/tmp/{name}.npy"
if mode == "save":
    np.save(f, x)
    print(name, "saved", float(np.abs(x).max()))
else:
    y = np.load(f)
    d = np.abs(x - y)
    bad = np.argwhere(d > 1e-9 * np.abs(y).max())
    print(name, "rel", float(np.linalg.norm(x - y) / np.linalg.norm(y)), "bad", len(bad), bad[:5].tolist())
