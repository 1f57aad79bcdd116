"""GPU parity for the paper's other spatial discretisations (Tables 1-2; SURVEY §8(f)
row 3; reading R14): centred heat of order 4 / 6 and upwind advection of order 1 / 3 / 5,
in 1-D (PCR on the host-factored tridiagonal factors) and 2-D (FFT diagonal solve with the
operator's symbol; residual stencils with halo up to 3), against the oracle (operators pinned in
tests/test_oracle_operators.py).  Cases: workloads.discretisation_cases()."""
import numpy as np
import pytest

import workloads as W
from oracle.paralpha import Oracle, relative_l2

pytestmark = pytest.mark.gpu
TOL = 1e-9
CASES = W.discretisation_cases()


def _run(p, u0, form="correction", hermitian=False, iters=3, alpha=1e-3):
    import paper_2103_12571_b200 as PB
    s = PB.Solver(p, u0)
    if hermitian:
        s.set_hermitian(True)
    if form != "correction":
        s.set_form(form)
    s.set_alpha_schedule([alpha] * iters)
    o = Oracle(p, u0, "dense" if p.M * p.N <= 1024 else "fourier")
    u = o.initial()
    errs = []
    for k in range(iters):
        u = o.iterate(u, alpha) if form == "correction" else o.iterate_direct(u, alpha)
        s.iterate(1)
        errs.append(relative_l2(s.get_iterate(), u))
    s.close()
    return errs


@pytest.mark.parametrize("p", CASES, ids=lambda p: p.name)
def test_operator_parity(p):
    errs = _run(p, p.u0())
    assert max(errs) <= TOL, errs


@pytest.mark.parametrize("p", W.halo_box_cases(), ids=lambda p: p.name)
def test_residual_halo_boxes(p):
    """residual2d_kernel stages the halo tile of a block that does not wrap the periodic boundary
    as one TMA tensor box and the boundary blocks row by row: 256 x 32 grids hold both kinds, for
    halo widths 1, 2 and 3 (the small operator cases above only have wrapping blocks)."""
    errs = _run(p, p.u0(), iters=2)
    assert max(errs) <= TOL, errs


@pytest.mark.parametrize("name", ["disc_heat6_2d_M3", "disc_upwind5_2d_M3", "disc_upwind3_1d_M2",
                                  "disc_heat6_1d_N16384"])
def test_operator_parity_direct_form(name):
    p = next(c for c in CASES if c.name == name)
    errs = _run(p, p.u0(), form="direct")
    assert max(errs) <= TOL, errs


@pytest.mark.parametrize("name", ["disc_heat6_2d_M3", "disc_upwind5_2d_M3", "disc_heat4_1d_M2",
                                  "disc_upwind5_1d_M3"])
def test_operator_parity_hermitian(name):
    """Real data (real u0; packed time series, L/2 + 1 solved frequencies)."""
    p = next(c for c in CASES if c.name == name)
    u0 = np.ascontiguousarray(p.u0().real.astype(np.complex128))
    errs = _run(p, u0, hermitian=True)
    assert max(errs) <= TOL, errs


def test_paper_heat_problem_converges_to_sequential():
    """The paper's heat test on a small grid with kappa = 6, M = 3 and its forcing:
    Paralpha iterates reach the sequential collocation solution (fixed point)."""
    import paper_2103_12571_b200 as PB
    from oracle.collocation import Tableau
    from oracle.paralpha import forcing_vector, sequential_solution
    p = W.Problem("paper_heat6", 2, 16, 16, "heat6", 1.0, 0, 0, 0.04, 8, 3, "random", "fixed", 1e-4, 6)
    x = np.arange(16) / 16
    mode = (np.sin(2 * np.pi * x)[None, :] * np.sin(2 * np.pi * x)[:, None]).reshape(-1)
    t0 = np.pi                                      # the paper's interval [pi, pi + T]
    v = forcing_vector(p, Tableau(p.M), lambda t: mode * (8 * np.pi ** 2 * np.cos(t0 + t) - np.sin(t0 + t)))
    u0 = (np.sin(t0) * mode).astype(np.complex128)
    s = PB.Solver(p, u0)
    s.set_forcing(v)
    s.set_alpha_schedule([1e-4] * 6)
    s.iterate(6)
    ref = sequential_solution(p, Tableau(p.M), u0, v)
    assert relative_l2(s.get_iterate(), ref) < 1e-10
    s.close()


SHARDED = [("disc_heat6_2d_M3", 2), ("disc_upwind5_2d_M3", 4), ("disc_upwind3_1d_M2", 2),
           ("disc_heat6_1d_N16384", 2)]


@pytest.mark.parametrize("name,P", SHARDED, ids=lambda x: str(x))
def test_operator_parity_sharded(name, P):
    """Wider stencils through the time-sharded path (P virtual ranks on one GPU, loopback group)."""
    import paper_2103_12571_b200 as PB
    p = next(c for c in CASES if c.name == name)
    u0 = p.u0()
    grp = PB.Group(p, u0, P)
    grp.set_alpha_schedule([1e-3] * 3)
    o = Oracle(p, u0, "dense" if p.M * p.N <= 1024 else "fourier")
    u = o.initial()
    for k in range(3):
        u = o.iterate(u, 1e-3)
        grp.iterate(1)
        e = relative_l2(grp.get_iterate(), u)
        assert e <= TOL, (k, e)
    grp.close()


@pytest.mark.parametrize("name", ["disc_heat6_2d_M3", "disc_upwind5_2d_M3", "disc_upwind3_2d_mixed_sign"])
def test_operator_sequential_baseline(name):
    """The GPU sequential Radau IIA baseline with the wider stencils against the oracle's stepping."""
    import paper_2103_12571_b200 as PB
    from oracle.collocation import Tableau
    from oracle.paralpha import sequential_solution
    p = next(c for c in CASES if c.name == name)
    u0 = p.u0()
    s = PB.Solver(p, u0)
    s.sequential()
    ref = sequential_solution(p, Tableau(p.M), u0)
    assert relative_l2(s.get_iterate(), ref) <= 1e-11
    s.close()
