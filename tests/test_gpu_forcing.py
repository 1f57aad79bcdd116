"""GPU parity with a forcing term (pint_set_forcing): w = (u0 + v_0, v_1, ...)
through the residual kernels, against the oracle with the same v (pinned in
tests/test_oracle_forcing.py)."""
import numpy as np
import pytest

import workloads as W
from oracle.collocation import Tableau
from oracle.paralpha import Oracle, forcing_vector, relative_l2
from oracle.schedule import adaptive_schedule as oracle_schedule

pytestmark = pytest.mark.gpu
TOL = 1e-9

CASES = [W.CONFIGS[1], W.CONFIGS[2], W.reduced(3), W.reduced(4), W.reduced(5),
         W.CONFIGS[3].replace(name="twopass_N16384_L8", nx=16384, L=8, iters=4),
         # the TMA-staged 1-D forward tile (L M in (512, 1024], L <= 256) and the pipelined PCR passes
         W.CONFIGS[3].replace(name="fwd1d_N256_L256", nx=256, L=256, iters=3),
         W.CONFIGS[3].replace(name="fwd1d_pcr1d_N8192_L256", nx=8192, L=256, iters=2),
         # the 2-D plane passes
         W.CONFIGS[4].replace(name="pipe_512sq_M2_L4", M=2, L=4, iters=3)] + W.edge_cases()


def _alphas(p, u0):
    if p.alpha_mode == "fixed":
        return [p.alpha_fixed] * p.iters
    return list(oracle_schedule(p.L, float(np.abs(u0).max()), p.m0, p.iters, p.eps, p.tau)[0])


@pytest.mark.parametrize("p", CASES, ids=lambda p: p.name)
def test_forcing_parity(p):
    import paper_2103_12571_b200 as PB
    u0 = p.u0()
    rng = np.random.default_rng(11)
    # a smooth forcing b(x, t) = sin(t) * (random field), integrated at the collocation nodes
    field = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
    v = forcing_vector(p, Tableau(p.M), lambda t: np.sin(1 + t) * field)
    a = _alphas(p, u0)
    s = PB.Solver(p, u0)
    s.set_forcing(v)
    s.set_alpha_schedule(a)
    o = Oracle(p, u0, "dense" if p.M * p.N <= 2048 else "fourier", v=v)
    u = o.initial()
    for k in range(min(p.iters, 5)):
        u = o.iterate(u, a[k])
        s.iterate(1)
        e = relative_l2(s.get_iterate(), u)
        assert e <= TOL, (k, e)
    # residual norms (forcing included); compared where they are above the roundoff floor
    # eps ||C|| ||u|| of the stiff cases
    l2, linf = s.residual_norm()
    r2, rinf = o.residual_norms(u)
    floor = 1e-12 * (1 + p.dT * 4 * max(p.nu, abs(p.cx)) * p.nx ** 2) * float(np.linalg.norm(u))
    assert abs(l2 - r2) <= 1e-6 * r2 + floor, (l2, r2, floor)
    s.close()


def test_forcing_rejects_incompatible_modes():
    import paper_2103_12571_b200 as PB
    p = W.reduced(5)
    s = PB.Solver(p, p.u0())
    s.set_forcing(np.ones((p.L, p.M, p.N), dtype=np.complex128))
    with pytest.raises(PB.PintError):
        s.set_form("direct")
    with pytest.raises(PB.PintError):
        s.set_hermitian(True)
    with pytest.raises(PB.PintError):
        s.sequential()
    s.set_forcing(None)
    s.set_form("direct")
    s.close()


def test_w_inf_and_algorithm2_gamma_with_forcing():
    """||w||_inf with a forcing attached is the max over the assembled w = (u0 + v_0, v_1, ...)
    (P:105), and Algorithm 2 takes gamma = L (3 eps + tau) ||w||_inf from it: the
    driver's alphas equal the a-priori schedule of that ||w||_inf."""
    import paper_2103_12571_b200 as PB
    from oracle.paralpha import w_vector
    p = W.reduced(5)
    u0 = p.u0()
    rng = np.random.default_rng(3)
    field = 40.0 * (rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N))   # dominates ||u0||
    v = forcing_vector(p, Tableau(p.M), lambda t: np.cos(t) * field)
    s = PB.Solver(p, u0)
    assert s.w_inf() == pytest.approx(float(np.abs(u0).max()), rel=1e-15)
    s.set_forcing(v)
    want = float(np.abs(w_vector(p, u0, v)).max())
    assert s.w_inf() == pytest.approx(want, rel=1e-14)
    tol = 1e-9 * want
    res = s.solve(p.m0, tol, 6, p.eps, p.tau)
    a_or, m_or = oracle_schedule(p.L, want, p.m0, res["iters"], p.eps, p.tau)
    np.testing.assert_allclose(res["m"], m_or[:res["iters"] + 1], rtol=1e-13)
    s.close()
