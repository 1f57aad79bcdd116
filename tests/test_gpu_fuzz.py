"""Randomised GPU parity sweep (seeded): small problems drawn over every operator, dimension,
grid shape, step count, node count, iteration form and the real-data mode, two iterations each
against the oracle.  Complements the hand-picked cases with shapes nobody chose (ragged tiles,
L = 1 / 2, M up to 6, 2-D shapes served by both spatial engines)."""
import numpy as np
import pytest

import workloads as W
from oracle.paralpha import Oracle, relative_l2

pytestmark = pytest.mark.gpu
TOL = 1e-9
OPS = ["heat", "advection", "heat4", "heat6", "upwind1", "upwind3", "upwind5"]


def _cases(n=96, seed=2103):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        dim = int(rng.integers(1, 3))
        op = OPS[int(rng.integers(len(OPS)))]
        nx = int(2 ** rng.integers(3, 7 if dim == 2 else 9))
        ny = int(2 ** rng.integers(2, 7)) if dim == 2 else 1
        L = int(2 ** rng.integers(0, 6))
        M = int(rng.integers(1, 7))
        heat = op.startswith("heat")
        nu = float(rng.uniform(0.05, 1.0)) if heat else 0.0
        cx = 0.0 if heat else float(rng.uniform(-1.0, 1.0))
        cy = 0.0 if heat or dim == 1 else float(rng.uniform(-1.0, 1.0))
        T = float(10 ** rng.uniform(-3, -1))
        alpha = float(10 ** rng.uniform(-4, -2))
        form = "direct" if rng.random() < 0.3 else "correction"
        herm = bool(rng.random() < 0.3)
        p = W.Problem(f"fz{i}_{dim}d_{op}_{nx}x{ny}_L{L}_M{M}_{form}{'_h' if herm else ''}", dim, nx, ny, op,
                      nu, cx, cy, T, L, M, "random", "fixed", alpha, 2)
        out.append((p, form, herm))
    return out


def _max_cond(p, alpha):
    from oracle.collocation import Tableau
    from oracle.paralpha import d_values
    tab = Tableau(p.M)
    worst = 0.0
    for d in d_values(p.L, alpha):
        r = d / (1 + d)
        _, V = np.linalg.eig(tab.Q - r * tab.Dt @ tab.H)
        worst = max(worst, np.linalg.cond(V))
    return worst


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c[0].name)
def test_fuzz_parity(case):
    import paper_2103_12571_b200 as PB
    p, form, herm = case
    u0 = p.u0()
    if herm:
        u0 = np.ascontiguousarray(u0.real.astype(np.complex128))
    s = PB.Solver(p, u0)
    if herm:
        try:
            s.set_hermitian(True)
        except PB.PintError as e:
            s.close()
            # documented requirements (pint.h): 1-D needs N >= 8 and L >= 2; 2-D runs only on the
            # register-engine grids (|log2 nx - log2 ny| <= 1, 4 <= L <= 1024); the rejection must
            # be one of those, then the case is done
            lx, ly, lL = int(np.log2(p.nx)), int(np.log2(p.ny)), int(np.log2(p.L))
            if p.dim == 1:
                supported = p.nx >= 8 and p.L >= 2
            else:
                supported = (2 <= lx <= 12 and 2 <= ly <= 12 and abs(lx - ly) <= 1 and 2 <= lL <= 10
                             and max(p.nx // 16, 1) * p.M <= 256)
            assert e.status == 1 and not supported, str(e)
            return
    if form == "direct":
        s.set_form("direct")
    a = [p.alpha_fixed] * 2
    try:
        s.set_alpha_schedule(a)
    except PB.PintError as e:
        s.close()
        # the guard may only fire where the frequency blocks really are near-defective: check the
        # eigenvector conditioning of Q - r_k D_t H_M independently (numpy) before accepting it
        assert e.status == 3, str(e)
        assert _max_cond(p, a[0]) > 1e6, f"guard fired on a well-conditioned alpha: {e}"
        pytest.skip(f"alpha tables rejected by the documented guard (near-defective): {e}")
    o = Oracle(p, u0, "dense" if p.M * p.N <= 1024 else "fourier")
    u = o.initial()
    for k in range(2):
        u = o.iterate(u, a[k]) if form == "correction" else o.iterate_direct(u, a[k])
        s.iterate(1)
        e = relative_l2(s.get_iterate(), u)
        assert e <= TOL, (k, e)
    s.close()


def _sharded_cases(n=24, seed=12571):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        P = int(rng.choice([2, 4]))
        L = int(2 ** rng.integers(2, 6))
        M = int(rng.integers(1, 5))
        if (L // P) % P or L < P * P or M * P > 32:
            continue
        dim = int(rng.integers(1, 3))
        op = OPS[int(rng.integers(len(OPS)))]
        heat = op.startswith("heat")
        nx = int(2 ** rng.integers(3, 6 if dim == 2 else 8))
        ny = int(2 ** rng.integers(3, 6)) if dim == 2 else 1
        p = W.Problem(f"fzs{len(out)}_P{P}_{dim}d_{op}_{nx}x{ny}_L{L}_M{M}", dim, nx, ny, op,
                      0.5 if heat else 0.0, 0.0 if heat else 0.7, 0.0 if heat or dim == 1 else -0.4,
                      float(10 ** rng.uniform(-3, -1)), L, M, "random", "fixed", 1e-3, 2)
        out.append((p, P))
    return out


@pytest.mark.parametrize("case", _sharded_cases(), ids=lambda c: c[0].name)
def test_fuzz_sharded_parity(case):
    """Time-sharded path (P virtual ranks on one GPU) on random shapes."""
    import paper_2103_12571_b200 as PB
    p, P = case
    u0 = p.u0()
    grp = PB.Group(p, u0, P)
    grp.set_alpha_schedule([p.alpha_fixed] * 2)
    o = Oracle(p, u0, "dense" if p.M * p.N <= 1024 else "fourier")
    u = o.initial()
    for k in range(2):
        u = o.iterate(u, p.alpha_fixed)
        grp.iterate(1)
        e = relative_l2(grp.get_iterate(), u)
        assert e <= TOL, (k, e)
    grp.close()
