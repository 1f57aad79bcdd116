"""GPU parity of the direct form (Alg. 1 as printed, PINT_FORM_DIRECT) against the oracle's
direct-form iteration (itself pinned to a dense C_a solve, tests/test_oracle_iteration.py)."""
import numpy as np
import pytest

import workloads as W
from oracle.paralpha import ModeOracle, Oracle, mode_coefficients, relative_l2
from oracle.schedule import adaptive_schedule as oracle_schedule

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _alphas(p, u0):
    if p.alpha_mode == "fixed":
        return [p.alpha_fixed] * p.iters
    return list(oracle_schedule(p.L, float(np.abs(u0).max()), p.m0, p.iters, p.eps, p.tau)[0])


CASES = [W.CONFIGS[1], W.CONFIGS[2], W.reduced(3), W.reduced(4), W.reduced(5),
         W.CONFIGS[3].replace(name="twopass_N16384_L8", nx=16384, L=8, iters=4)] + W.edge_cases()


@pytest.mark.parametrize("p", CASES, ids=lambda p: p.name)
def test_direct_form_parity(p):
    import paper_2103_12571_b200 as PB
    u0 = p.u0()
    a = _alphas(p, u0)
    s = PB.Solver(p, u0)
    s.set_form("direct")
    s.set_alpha_schedule(a)
    o = Oracle(p, u0, "dense" if p.M * p.N <= 2048 else "fourier")
    u = o.initial()
    for k in range(min(p.iters, 5)):
        un = o.iterate_direct(u, a[k])
        d = s.iterate(1, want_diff=True)[0]
        e = relative_l2(s.get_iterate(), un)
        assert e <= TOL, (k, e)
        ref = float(np.abs(un[-1] - u[-1]).max())
        assert abs(d - ref) <= 1e-4 * ref + 1e-10 * np.abs(un).max()
        u = un
    s.close()


def test_direct_form_full_size_config5_sampled():
    import paper_2103_12571_b200 as PB
    p = W.CONFIGS[5]
    u0 = p.u0()
    a = _alphas(p, u0)
    s = PB.Solver(p, u0)
    s.set_form("direct")
    s.set_alpha_schedule(a)
    rng = np.random.default_rng(5)
    kx = np.concatenate([np.arange(0, 5).repeat(5), rng.integers(0, p.nx, 8)])
    ky = np.concatenate([np.tile(np.arange(0, 5), 5), rng.integers(0, p.ny, 8)])
    mo = ModeOracle(p, mode_coefficients(p, u0, kx, ky), kx, ky)
    uh = mo.initial()
    from test_gpu_parity import _gpu_project
    for k in range(4):
        uh = mo.iterate_direct(uh, a[k])
        s.iterate(1)
        g = _gpu_project(s, p, kx, ky)
        e = float(np.linalg.norm((g - uh).ravel()) / np.linalg.norm(uh.ravel()))
        assert e <= TOL, (k, e)
    s.close()


def test_direct_form_group_needs_one_form():
    """The direct form runs on sharded ranks (tests/test_gpu_sharded.py::test_sharded_direct_form);
    a group whose virtual ranks disagree on the form is refused, not run half-and-half."""
    import paper_2103_12571_b200 as PB
    p = W.CONFIGS[2].replace(L=16)
    grp = PB.Group(p, p.u0(), 2)
    grp.set_alpha_schedule([1e-5])
    grp.ranks[0].set_form("direct")
    with pytest.raises(PB.PintError) as e:
        grp.iterate(1)
    assert e.value.status == 7
    grp.close()


@pytest.mark.parametrize("form", ["correction", "direct"])
@pytest.mark.parametrize("p", [W.reduced(3), W.reduced(5)], ids=lambda p: p.name)
def test_algorithm2_driver(p, form):
    """pint_solve (Algorithm 2): the schedule is the oracle's recurrence, the driver stops
    at the first consecutive-iterate norm <= tol, and the iterate it stops at matches the oracle
    run for the same number of iterations with the same alphas."""
    import paper_2103_12571_b200 as PB
    u0 = p.u0()
    tol = 1e-9 * float(np.abs(u0).max())
    s = PB.Solver(p, u0)
    s.set_form(form)
    r = s.solve(p.m0, tol, 12, p.eps, p.tau)
    n = r["iters"]
    assert 1 <= n <= 12 and r["stop"] in ("consecutive iterates", "m_k <= tol", "max_iter")
    if r["stop"] == "consecutive iterates":
        assert r["diffs"][-1] <= tol and (n == 1 or np.all(r["diffs"][:-1] > tol))
    a_or, m_or = oracle_schedule(p.L, float(np.abs(u0).max()), p.m0, n, p.eps, p.tau)
    np.testing.assert_allclose(r["m"], m_or[:n + 1], rtol=1e-13)
    o = Oracle(p, u0, "dense" if p.M * p.N <= 2048 else "fourier")
    u = o.initial()
    for k in range(n):
        u = o.iterate(u, a_or[k]) if form == "correction" else o.iterate_direct(u, a_or[k])
    assert relative_l2(s.get_iterate(), u) <= TOL
    s.close()
