"""GPU parity of the real-data fast path (pint_set_hermitian): packed real
time transforms, only the frequencies k <= L/2 solved, y_{L-k} = conj(y_k); 1-D and 2-D, both
forms, against the unchanged complex oracle (the real-data iterate equals the oracle's up to its
roundoff imaginary part)."""
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
         W.CONFIGS[3].replace(name="twopass_N16384_L8", nx=16384, L=8, iters=4)] + [
    p for p in W.edge_cases() if p.N >= 8 and p.L >= 2] + [   # documented: N >= 8, L >= 2 (pint.h)
    W.reduced(5).replace(name="red5_adv2d_32x64_M2_L8", nx=32, ny=64, M=2, L=8)]


@pytest.mark.parametrize("form", ["correction", "direct"])
@pytest.mark.parametrize("p", CASES, ids=lambda p: p.name)
def test_hermitian_parity(p, form):
    import paper_2103_12571_b200 as PB
    u0 = p.u0()
    if np.abs(u0.imag).max() > 0:   # edge cases draw complex u0: the real-data mode takes its real part
        u0 = np.ascontiguousarray(u0.real.astype(np.complex128))
    a = _alphas(p, u0)
    s = PB.Solver(p, u0)
    s.set_form(form)
    s.set_hermitian(True)
    s.set_alpha_schedule(a)
    o = Oracle(p, u0, "dense" if p.M * p.N <= 2048 else "fourier")
    u = o.initial()
    for k in range(min(p.iters, 6)):
        u = o.iterate(u, a[k]) if form == "correction" else o.iterate_direct(u, a[k])
        s.iterate(1)
        ug = s.get_iterate()
        assert relative_l2(ug, u) <= TOL, (k, relative_l2(ug, u))
        assert np.abs(ug.imag).max() <= TOL * np.abs(ug).max()    # real up to (alpha-amplified) roundoff
    s.close()


def test_hermitian_rejects_complex_data():
    import paper_2103_12571_b200 as PB
    p = W.reduced(4)
    u0 = p.u0().astype(np.complex128) * (1 + 0.5j)
    s = PB.Solver(p, u0)
    with pytest.raises(PB.PintError):
        s.set_hermitian(True)
    s.close()


def test_hermitian_full_size_config5_sampled_modes():
    import paper_2103_12571_b200 as PB
    from test_gpu_parity import _gpu_project, _mode_sample
    p = W.CONFIGS[5]
    u0 = p.u0()
    a = _alphas(p, u0)
    s = PB.Solver(p, u0)
    s.set_hermitian(True)
    s.set_alpha_schedule(a)
    kx, ky = _mode_sample(p, 5)
    mo = ModeOracle(p, mode_coefficients(p, u0, kx, ky), kx, ky)
    uh = mo.initial()
    errs = []
    for k in range(4):
        uh = mo.iterate(uh, a[k])
        s.iterate(1)
        g = _gpu_project(s, p, kx, ky)
        errs.append(float(np.linalg.norm((g - uh).ravel()) / np.linalg.norm(uh.ravel())))
    s.close()
    assert max(errs) <= TOL, errs


def test_real_storage_roundtrip():
    """Hermitian mode stores the iterate as real fp64 (first L M N doubles of u_dev): switching on
    converts, get_iterate expands to (re, 0), switching off restores complex128 storage, and the
    iteration continues identically in both storages."""
    import paper_2103_12571_b200 as PB
    p = W.reduced(5)
    u0 = np.ascontiguousarray(p.u0().real.astype(np.complex128))
    a = [1e-3] * 4
    ref = PB.Solver(p, u0)
    ref.set_alpha_schedule(a)
    ref.iterate(2)
    s = PB.Solver(p, u0)
    s.set_alpha_schedule(a)
    s.iterate(1)
    before = s.get_iterate()
    s.set_hermitian(True)
    after = s.get_iterate()
    assert np.array_equal(after.real, before.real) and np.all(after.imag == 0)
    v = s.iterate_view()
    assert v.dtype.is_floating_point and not v.dtype.is_complex and tuple(v.shape) == (p.L, p.M, p.N)
    np.testing.assert_array_equal(v.cpu().numpy(), before.real)
    s.iterate(1)
    assert relative_l2(s.get_iterate(), ref.get_iterate()) < 1e-12
    s.set_hermitian(False)
    np.testing.assert_array_equal(s.iterate_view().cpu().numpy(), s.get_iterate())
    ref.iterate(1)
    s.iterate(1)
    assert relative_l2(s.get_iterate(), ref.get_iterate()) < 1e-12
    s.close()
    ref.close()


# the real-data mode on the pipelined plane passes (grids 512^2 .. 2048^2): packed pairs (y, x),
# (y, x + nx/2), the R pass unpacks X_k row by row, the I pass writes the unit planes
HERM_PIPE = [W.CONFIGS[5].replace(name="hpipe_1024sq_M4_L4", L=4, iters=3),
             W.CONFIGS[4].replace(name="hpipe_512sq_M3_L8", L=8, iters=3),
             W.CONFIGS[5].replace(name="hpipe_1024x512_M2_L4", ny=512, M=2, L=4, iters=3),
             W.CONFIGS[4].replace(name="hpipe_512x1024_M1_L8", ny=1024, M=1, L=8, iters=3),
             W.CONFIGS[5].replace(name="hpipe_2048x1024_heat_M2_L4", nx=2048, op="heat", nu=1e-2, M=2, L=4,
                                  iters=2)]


@pytest.mark.parametrize("form", ["correction", "direct"])
@pytest.mark.parametrize("p", HERM_PIPE, ids=lambda p: p.name)
def test_hermitian_pipe_plans(p, form):
    import paper_2103_12571_b200 as PB
    rng = np.random.default_rng(p.nx + 7 * p.ny + p.M)
    u0 = rng.standard_normal(p.N).astype(np.complex128)   # real data, every spatial mode excited
    s = PB.Solver(p, u0)
    s.set_form(form)
    s.set_hermitian(True)
    assert "cols_pipe_kernel" in " ".join(s.kernel_names()), s.kernel_names()
    a = [1e-3, 2e-2, 0.2][:p.iters]
    s.set_alpha_schedule(a)
    o = Oracle(p, u0, "fourier")
    u = o.initial()
    for k in range(p.iters):
        u = o.iterate(u, a[k]) if form == "correction" else o.iterate_direct(u, a[k])
        s.iterate(1)
        assert relative_l2(s.get_iterate(), u) <= TOL, k
    s.close()
