"""Windowed Paralpha (pint_next_window): W windows of L steps, each
solved with the Algorithm 2 driver and started from the previous window's final value, reproduce
sequential collocation stepping over W L steps (oracle)."""
import numpy as np
import pytest

import workloads as W
from oracle.collocation import Tableau
from oracle.paralpha import relative_l2, sequential_solution

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p", [W.reduced(5).replace(name="win_adv2d", L=8, T=0.125),
                               W.reduced(3).replace(name="win_heat1d", L=8, T=0.125, nx=256)],
                         ids=lambda p: p.name)
@pytest.mark.parametrize("hermitian", [False, True], ids=["complex", "hermitian"])
def test_windows_reproduce_sequential_stepping(p, hermitian):
    """hermitian: the real-data mode (real storage of u; the window hand-over goes through the
    real final value)."""
    import paper_2103_12571_b200 as PB
    nwin = 4
    u0 = p.u0()
    s = PB.Solver(p, u0)
    if hermitian:
        s.set_hermitian(True)
    for w in range(nwin):
        r = s.solve(p.m0, 1e-13 * float(np.abs(s.get_final_value()).max() + 1e-300) if w else
                    1e-13 * float(np.abs(u0).max()), 40, p.eps, p.tau)
        assert r["iters"] >= 1
        if w < nwin - 1:
            s.next_window()
    ref = sequential_solution(p.replace(L=p.L * nwin, T=p.T * nwin), Tableau(p.M), u0)
    assert relative_l2(s.get_final_value(), ref[-1, -1]) <= 1e-9
    s.close()
