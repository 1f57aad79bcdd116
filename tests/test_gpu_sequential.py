"""GPU sequential Radau IIA baseline (pint_sequential) against the
oracle's sequential collocation stepping (itself pinned to the converged iteration and to the
single-mode closed form, tests/test_oracle_iteration.py)."""
import numpy as np
import pytest

import workloads as W
from oracle.collocation import Tableau
from oracle.paralpha import relative_l2, sequential_solution

pytestmark = pytest.mark.gpu

CASES = [W.reduced(4), W.reduced(5), W.reduced(5).replace(name="red5_adv2d_32x64_M2_L8", nx=32, ny=64, M=2, L=8)] + [
    p for p in W.edge_cases() if p.dim == 2]
# 1-D: the shifted tridiagonal solves by the PCR kernels (one-pass N <= 4096, two-pass beyond),
# heat and centred advection, and a wider stencil (tridiagonal factors)
CASES_1D = [W.CONFIGS[1], W.CONFIGS[2].replace(L=16), W.reduced(3),
            W.CONFIGS[3].replace(name="seq_heat_N16384_L8", nx=16384, L=8),
            W.CONFIGS[2].replace(name="seq_adv_N8192_M2_L8", nx=8192, M=2, L=8),
            W.CONFIGS[1].replace(name="seq_heat4_N64", op="heat4")] + [
    p for p in W.edge_cases() if p.dim == 1 and p.nx >= 8]


@pytest.mark.parametrize("p", CASES, ids=lambda p: p.name)
def test_sequential_matches_oracle(p):
    import paper_2103_12571_b200 as PB
    u0 = p.u0()
    s = PB.Solver(p, u0)
    s.sequential()
    ref = sequential_solution(p, Tableau(p.M), u0)
    assert relative_l2(s.get_iterate(), ref) <= 1e-11
    s.close()


@pytest.mark.parametrize("p", CASES_1D, ids=lambda p: p.name)
def test_sequential_1d_matches_oracle(p):
    test_sequential_matches_oracle(p)


def test_iteration_converges_to_sequential():
    """The Paralpha iteration's fixed point is the sequential solution: after enough
    iterations the GPU iterate equals the GPU sequential baseline."""
    import paper_2103_12571_b200 as PB
    p = W.reduced(5)
    u0 = p.u0()
    s = PB.Solver(p, u0)
    s.sequential()
    useq = s.get_iterate()
    s.set_initial_value(u0, reset=True)
    r = s.solve(p.m0, 1e-12 * float(np.abs(u0).max()), 30, p.eps, p.tau)
    assert relative_l2(s.get_iterate(), useq) <= 1e-9, r
    s.close()
