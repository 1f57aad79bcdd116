"""GPU parity of the paper's own test problems at their Table 1/2 sizes (SURVEY §8(f)
row 3): heat with centred kappa 2/4/6 and advection u_t + u_x + u_y = 0 with upwind kappa 1..5 on
7-smooth, mostly non-power-of-two grids (N = 300 ... 800), 1-D and 2-D, through the generic-grid
path (generic.cu: mixed-radix Stockham FFT-diagonal solves) — and the upwind kappa = 2, 4 stencils
(reading R16) also on power-of-two grids (PCR factors in 1-D, the register pipeline in 2-D).
Oracle: Fourier tier (any N), relative l2 <= 1e-9 after every iteration."""
import numpy as np
import pytest

import workloads as W
from oracle.paralpha import Oracle, relative_l2

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _run(p, iters=2, alpha=None):
    import paper_2103_12571_b200 as PB
    u0 = p.u0()
    a = [alpha or p.alpha_fixed] * iters
    s = PB.Solver(p, u0)
    names = s.kernel_names()
    s.set_alpha_schedule(a)
    o = Oracle(p, u0, "dense" if p.M * p.N <= 2048 else "fourier")
    u = o.initial()
    errs = []
    for k in range(iters):
        u = o.iterate(u, a[k])
        d = s.iterate(1, want_diff=True)[0]
        errs.append(relative_l2(s.get_iterate(), u))
        assert np.isfinite(d)
    l2, _ = s.residual_norm()
    rl2, _ = o.residual_norms(u)
    s.close()
    assert max(errs) <= TOL, errs
    assert l2 == pytest.approx(rl2, rel=1e-6, abs=1e-9 * np.linalg.norm(u.ravel()))
    return names


@pytest.mark.parametrize("p", W.table_cases(), ids=lambda p: p.name)
def test_table_problem_parity(p):
    names = _run(p)
    pow2 = (p.nx & (p.nx - 1)) == 0 and (p.ny & (p.ny - 1)) == 0
    assert pow2 or "fft_any_kernel<fwd x>" in names, names


GENERIC_EDGES = [
    W.Problem("gen_1d_N6_M2_L4", 1, 6, 1, "heat", 1.0, 0, 0, 0.1, 4, 2, "random", "fixed", 1e-3, 2),
    W.Problem("gen_1d_N105_adv_M3", 1, 105, 1, "advection", 0, -1.0, 0, 0.05, 8, 3, "random", "fixed", 1e-2, 2),
    W.Problem("gen_2d_12x20_heat6_M2", 2, 12, 20, "heat6", 0.5, 0, 0, 0.02, 8, 2, "random", "fixed", 1e-3, 2),
    W.Problem("gen_2d_49x36_upwind4", 2, 49, 36, "upwind4", 0, 0.7, -1.1, 0.01, 16, 2, "random", "fixed", 1e-2, 2),
    W.Problem("gen_2d_14x30_upwind3_M1", 2, 14, 30, "upwind3", 0, 1.0, 0.5, 0.01, 4, 1, "random", "fixed", 1e-2, 2),
    W.Problem("gen_2d_7x5_L1", 2, 7, 5, "heat", 1.0, 0, 0, 0.05, 1, 2, "random", "fixed", 0.3, 2),
]


@pytest.mark.parametrize("p", GENERIC_EDGES, ids=lambda p: p.name)
def test_generic_grid_edges(p):
    """Odd, prime-power and tiny 7-smooth grids, L = 1, both flow signs."""
    _run(p)


@pytest.mark.parametrize("dim", [1, 2])
@pytest.mark.parametrize("op", ["upwind2", "upwind4"])
def test_even_upwind_on_power_of_two_grids(op, dim):
    """kappa = 2, 4 upwind on the power-of-two path: PCR over the host factors (1-D) and the
    residual / pipelined spatial kernels (2-D)."""
    p = W.Problem(f"{op}_{dim}d", dim, 64, 64 if dim == 2 else 1, op, 0, 1.0, 1.0 if dim == 2 else 0.0, 0.005,
                  16, 2, "random", "fixed", 1e-3, 2)
    _run(p)
    _run(p.replace(cx=-1.0, cy=-0.5 if dim == 2 else 0.0))


def test_generic_rejections():
    import paper_2103_12571_b200 as PB
    p = W.table_cases()[0]
    s = PB.Solver(p, p.u0())
    for call in (lambda: s.set_form("direct"), lambda: s.set_hermitian(True)):
        with pytest.raises(PB.PintError) as e:
            call()
        assert e.value.status == 1
    s.close()
    with pytest.raises(PB.PintError):
        PB.Group(p, p.u0(), 2)
