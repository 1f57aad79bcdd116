"""Guard paths of the C ABI (include/pint.h error contract): the numeric diagonalisability guard at a
true defective point of Q - r D_t H_M, non-finite inputs and a
diverged (overflowed) iterate reported as PINT_ERR_NUMERIC, and an atomic schedule replacement."""
import mpmath as mp
import numpy as np
import pytest

import workloads as W
from oracle.collocation import Tableau
from oracle.paralpha import Oracle, relative_l2

pytestmark = pytest.mark.gpu

NOT_DIAG, NUMERIC, SCHEDULE = 3, 4, 2


def _defective_alpha_M2_L4():
    """alpha with d_0 = -alpha^{1/4} at the defective point of B(r) = Q - r D_t H_M for M = 2.

    For the Radau IIA M = 2 tableau (Q = [[5/12, -1/12], [3/4, 1/4]], t = (1/3, 1)) the
    characteristic polynomial of B(r) has discriminant r^2 - 2r/3 - 2/9, zero at r* = (1 - sqrt 3)/3;
    with r = d/(1 + d) that is d* = r*/(1 - r*) = -0.19615... (the printed
    forbidden values of Lemma 3.4 carry a sign slip).  Returns the double alpha nearest d*^4 and
    the relative eigenvalue gap there (mpmath, 40 digits)."""
    mp.mp.dps = 40
    rs = (1 - mp.sqrt(3)) / 3
    ds = rs / (1 - rs)
    alpha = float(ds ** 4)
    d = -mp.mpf(alpha) ** mp.mpf(0.25)
    r = d / (1 + d)
    B = mp.matrix([[mp.mpf(5) / 12, -mp.mpf(1) / 12 - r / 3], [mp.mpf(3) / 4, mp.mpf(1) / 4 - r]])
    tr, det = B[0, 0] + B[1, 1], B[0, 0] * B[1, 1] - B[0, 1] * B[1, 0]
    sq = mp.sqrt(tr * tr - 4 * det)
    lmax = max(abs((tr + sq) / 2), abs((tr - sq) / 2))
    return alpha, float(abs(sq) / lmax), float(ds)


def test_defective_point_closed_form():
    """The closed form above is the tableau's: disc(r*) = 0 with the oracle's Q (independent pin)."""
    tab = Tableau(2)
    _, _, ds = _defective_alpha_M2_L4()
    rs = ds / (1 + ds)
    B = tab.Q - rs * tab.Dt @ tab.H
    ev = np.linalg.eigvals(B)
    assert abs(ev[0] - ev[1]) < 1e-6 and ds == pytest.approx(-0.19615242270663188, rel=1e-14)


def test_not_diagonalizable_fires_at_defective_alpha():
    import paper_2103_12571_b200 as P
    p = W.CONFIGS[1]                       # M = 2, L = 4
    alpha, rel_gap, _ = _defective_alpha_M2_L4()
    assert rel_gap < 1e-8                  # inside the documented guard (gap < 1e-8 rho(B))
    s = P.Solver(p, p.u0())
    with pytest.raises(P.PintError) as e:
        s.set_alpha_schedule([alpha])
    assert e.value.status == NOT_DIAG, str(e.value)
    # a nearby, well-conditioned alpha passes and iterates against the oracle
    s.set_alpha_schedule([1.3e-3])
    o = Oracle(p, p.u0())
    s.iterate(1)
    assert relative_l2(s.get_iterate(), o.iterate(o.initial(), 1.3e-3)) <= 1e-9
    s.close()


def test_failed_schedule_keeps_previous_schedule():
    """A rejected entry in the middle of a schedule leaves the old schedule and tables in place."""
    import paper_2103_12571_b200 as P
    p = W.CONFIGS[1]
    alpha_bad, _, _ = _defective_alpha_M2_L4()
    s = P.Solver(p, p.u0())
    s.set_alpha_schedule([1e-4, 1e-4])
    with pytest.raises(P.PintError) as e:
        s.set_alpha_schedule([2e-2, alpha_bad, 3e-2])
    assert e.value.status == NOT_DIAG
    o = Oracle(p, p.u0())
    u = o.initial()
    for _ in range(2):                      # still the old (1e-4, 1e-4) schedule, both entries
        s.iterate(1)
        u = o.iterate(u, 1e-4)
        assert relative_l2(s.get_iterate(), u) <= 1e-9
    with pytest.raises(P.PintError) as e:
        s.iterate(1)
    assert e.value.status == SCHEDULE
    s.close()


@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_non_finite_u0_rejected(bad):
    import paper_2103_12571_b200 as P
    p = W.CONFIGS[1]
    u0 = p.u0().copy()
    u0[3] = bad
    with pytest.raises(P.PintError) as e:
        P.Solver(p, u0)
    assert e.value.status == NUMERIC
    s = P.Solver(p, p.u0())
    with pytest.raises(P.PintError) as e:
        s.set_initial_value(u0)
    assert e.value.status == NUMERIC
    s.close()


@pytest.mark.parametrize("cfg", [1, 5])
def test_overflowed_iterate_reports_numeric(cfg):
    """u0 = 1e308 (finite) overflows the stencil: the iterate turns inf/NaN and both the last-step
    difference (NaN-propagating device max) and the residual norm return PINT_ERR_NUMERIC instead
    of a 'converged' zero."""
    import paper_2103_12571_b200 as P
    p = W.CONFIGS[1] if cfg == 1 else W.reduced(5)
    u0 = np.full(p.N, 1e308, dtype=np.complex128)
    u0[::2] = -1e308
    s = P.Solver(p, u0)
    s.set_alpha_schedule([0.01])
    with pytest.raises(P.PintError) as e:
        s.iterate(1, want_diff=True)
    assert e.value.status == NUMERIC
    with pytest.raises(P.PintError) as e:
        s.residual_norm()
    assert e.value.status == NUMERIC
    s.close()
