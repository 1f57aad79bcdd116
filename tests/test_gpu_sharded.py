"""Time-sharded path (P ranks, cyclic steps, four-step time FFT, ring halo) on ONE GPU via the
single-process loopback group: the same kernels and phase sequence as NCCL ranks, with the
halo and all-to-all chunks moved by device copies.  Parity against the CPU oracle per iteration
(gathered global iterate) and against the 1-rank CUDA path."""
import numpy as np
import pytest

import workloads as W
from oracle.paralpha import Oracle, relative_l2
from oracle.schedule import adaptive_schedule as oracle_schedule

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _alphas(p, u0):
    if p.alpha_mode == "fixed":
        return [p.alpha_fixed] * p.iters
    return list(oracle_schedule(p.L, float(np.abs(u0).max()), p.m0, p.iters, p.eps, p.tau)[0])


CASES = [
    (W.CONFIGS[2], 2), (W.CONFIGS[2], 8),
    (W.reduced(3), 2), (W.reduced(3), 4),
    (W.reduced(4), 2), (W.reduced(4), 4),
    (W.reduced(5), 2), (W.reduced(5), 4),
    (W.CONFIGS[3].replace(name="twopass_N16384_L16", nx=16384, L=16, iters=3), 4),
    (W.edge_cases()[4], 2),   # M = 5, L = 16
]


@pytest.mark.parametrize("p,P", CASES, ids=lambda x: getattr(x, "name", str(x)))
def test_sharded_parity(p, P):
    import paper_2103_12571_b200 as PB
    u0 = p.u0()
    a = _alphas(p, u0)
    grp = PB.Group(p, u0, P)
    one = PB.Solver(p, u0)
    grp.set_alpha_schedule(a)
    one.set_alpha_schedule(a)
    o = Oracle(p, u0, "dense" if p.M * p.N <= 2048 else "fourier")
    u = o.initial()
    np.testing.assert_array_equal(grp.get_iterate(), u)
    for k in range(min(p.iters, 4)):
        u = o.iterate(u, a[k])
        d = grp.iterate(1, want_diff=True)[0]
        one.iterate(1)
        ug = grp.get_iterate()
        e = relative_l2(ug, u)
        assert e <= TOL, (k, e)
        # both are within 1e-9 of the oracle; they differ only by the FFT factorisation (roundoff)
        assert relative_l2(ug, one.get_iterate()) <= 1e-10
        assert d >= 0.0 and np.isfinite(d)
    # residual norms: equal up to the roundoff floor eps * ||C|| * ||u|| (the iterates are converged)
    # against the oracle's residual of the group's own iterate: only the rounding of one residual
    # evaluation separates them (a few ulps of u0, u and dT (Q x A) u)
    l2, linf = grp.residual_norm()
    ug = grp.get_iterate()
    rl2, rlinf = o.residual_norms(ug)
    stiff = 1 + p.dT * 4 * max(p.nu, abs(p.cx), abs(getattr(p, "cy", 0.0))) * p.nx ** 2
    assert abs(l2 - rl2) <= 1e-9 * rl2 + 1e-13 * stiff * float(np.linalg.norm(ug.ravel())), (l2, rl2)
    assert abs(linf - rlinf) <= 1e-9 * rlinf + 1e-13 * stiff * float(np.abs(ug).max()), (linf, rlinf)
    grp.close()
    one.close()


def test_sharded_last_step_diff():
    import paper_2103_12571_b200 as PB
    p = W.CONFIGS[2].replace(L=16, iters=3)
    u0 = p.u0()
    a = [1e-5, 1e-3, 1e-2]
    grp = PB.Group(p, u0, 4)
    grp.set_alpha_schedule(a)
    o = Oracle(p, u0)
    u = o.initial()
    for k in range(3):
        un = o.iterate(u, a[k])
        d = grp.iterate(1, want_diff=True)[0]
        # difference of consecutive iterates: cancellation, so compare at the iterate's roundoff scale
        assert d == pytest.approx(float(np.abs(un[-1] - u[-1]).max()), rel=1e-4, abs=1e-10 * np.abs(un).max())
        u = un
    grp.close()


def test_loopback_context_refuses_plain_iterate():
    import paper_2103_12571_b200 as PB
    p = W.CONFIGS[2].replace(L=16)
    grp = PB.Group(p, p.u0(), 2)
    grp.set_alpha_schedule([1e-5])
    with pytest.raises(PB.PintError) as e:
        grp.ranks[0].iterate(1)
    assert e.value.status == 7
    grp.close()


DIRECT = [(W.CONFIGS[2], 4), (W.reduced(3), 2), (W.reduced(4), 4), (W.reduced(5), 2),
          (W.reduced(5).replace(name="red5_L64", L=64, iters=3), 8),
          (W.CONFIGS[3].replace(name="twopass_N16384_L16", nx=16384, L=16, iters=3), 4)]


@pytest.mark.parametrize("p,P", DIRECT, ids=lambda x: getattr(x, "name", str(x)))
def test_sharded_direct_form(p, P):
    """Direct form (Alg. 1 as printed) on P virtual ranks: r0 from the rank holding step L - 1,
    broadcast; the synthesized front in the local slot order; solves; inverse cross-rank DFT and
    the all-to-all back; the overwrite backward.  Against the oracle's direct-form iteration."""
    import paper_2103_12571_b200 as PB
    u0 = p.u0()
    a = _alphas(p, u0)
    grp = PB.Group(p, u0, P)
    grp.set_form("direct")
    grp.set_alpha_schedule(a)
    o = Oracle(p, u0, "dense" if p.M * p.N <= 2048 else "fourier")
    u = o.initial()
    for k in range(min(p.iters, 4)):
        un = o.iterate_direct(u, a[k])
        d = grp.iterate(1, want_diff=True)[0]
        e = relative_l2(grp.get_iterate(), un)
        assert e <= TOL, (k, e)
        ref = float(np.abs(un[-1] - u[-1]).max())
        assert abs(d - ref) <= 1e-4 * ref + 1e-10 * np.abs(un).max()
        u = un
    grp.close()
