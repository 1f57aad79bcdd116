"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, per iteration, on the same
seeded inputs.  Bar (north star): relative l2 <= 1e-9 after every iteration."""
import numpy as np
import pytest

import workloads as W
from oracle.paralpha import ModeOracle, Oracle, mode_coefficients, relative_l2
from oracle.schedule import adaptive_schedule as oracle_schedule

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _solver(p, u0):
    import paper_2103_12571_b200 as P
    return P.Solver(p, u0)


def schedules(p, u0, s=None):
    """(oracle alphas, library alphas) — each side computes its own."""
    if p.alpha_mode == "fixed":
        a = [p.alpha_fixed] * p.iters
        return a, a
    w_inf = float(np.abs(u0).max())
    a_or, _ = oracle_schedule(p.L, w_inf, p.m0, p.iters, p.eps, p.tau)
    import paper_2103_12571_b200 as P
    w_lib = s.w_inf() if s is not None else w_inf
    a_lib, _ = P.adaptive_schedule(p.L, w_lib, p.m0, p.iters, p.eps, p.tau)
    np.testing.assert_allclose(a_lib, a_or, rtol=1e-14)
    return list(a_or), list(a_lib)


def run_parity(p, tier="auto", iters=None):
    u0 = p.u0()
    s = _solver(p, u0)
    a_or, a_lib = schedules(p, u0, s)
    s.set_alpha_schedule(a_lib)
    o = Oracle(p, u0, tier)
    u = o.initial()
    np.testing.assert_array_equal(s.get_iterate(), u)
    errs = []
    for k in range(iters or p.iters):
        u = o.iterate(u, a_or[k])
        s.iterate(1)
        ug = s.get_iterate()
        errs.append(relative_l2(ug, u))
    s.close()
    assert max(errs) <= TOL, errs
    return errs


@pytest.mark.parametrize("cfg", [1, 2])
def test_parity_full_size(cfg):
    run_parity(W.CONFIGS[cfg])


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_parity_reduced(cfg):
    run_parity(W.reduced(cfg))


@pytest.mark.parametrize("p", W.edge_cases(), ids=lambda p: p.name)
def test_parity_edge_cases(p):
    run_parity(p, tier="dense")


def test_parity_two_pass_pcr_small():
    """1-D with N > 4096 switches to the two-pass (classes + chunks) PCR; keep the oracle fast."""
    p = W.CONFIGS[3].replace(name="twopass_N16384_L8", nx=16384, L=8, iters=4)
    run_parity(p)


# the pipelined 1-D PCR passes (pcr1d.cu) serve 8192 <= N <= 65536 with classes of 256 points:
# R = N/256 = 32 .. 256 (chunk levels 5 .. 8), heat (symmetric levels) and centred advection
# (antisymmetric level 0), chunk tiles wrapping at both line ends
PIPE1D = [W.CONFIGS[3].replace(name="pcr1d_heat_N8192_L8", nx=8192, L=8, iters=3),
          W.CONFIGS[3].replace(name="pcr1d_heat_N32768_M2_L4", nx=32768, M=2, L=4, iters=3),
          W.CONFIGS[2].replace(name="pcr1d_adv_N16384_L8", nx=16384, L=8, iters=3),
          W.CONFIGS[2].replace(name="pcr1d_adv_N65536_M2_L4", nx=65536, M=2, L=4, iters=2)]


@pytest.mark.parametrize("p", PIPE1D, ids=lambda p: p.name)
def test_parity_pcr1d_pipe(p):
    run_parity(p)


# the TMA-staged 1-D forward tile (fwd1d_tma_kernel) runs where the tile is 4 points wide
# (512 < L M <= 1024, L <= 256): config 3's shape at small N, both operators, M = 3 and 4
FWD1D = [W.CONFIGS[3].replace(name="fwd1d_heat_N256_L256", nx=256, L=256, iters=3),
         W.CONFIGS[2].replace(name="fwd1d_adv_N512_M4_L256", nx=512, M=4, L=256, iters=3),
         W.CONFIGS[3].replace(name="fwd1d_heat_N8192_L256_twopass", nx=8192, L=256, iters=2)]


@pytest.mark.parametrize("p", FWD1D, ids=lambda p: p.name)
def test_parity_fwd1d_tma(p):
    run_parity(p)


def test_last_step_diff_and_residual_norm():
    p = W.CONFIGS[2].replace(L=16, iters=4)
    u0 = p.u0()
    s = _solver(p, u0)
    a = [1e-5, 1e-4, 1e-3, 1e-2]
    s.set_alpha_schedule(a)
    o = Oracle(p, u0)
    u = o.initial()
    for k in range(4):
        un = o.iterate(u, a[k])
        d = s.iterate(1, want_diff=True)[0]
        ref = float(np.abs(un[-1] - u[-1]).max())
        # the difference of two iterates inherits the parity error of each (north star: 1e-9
        # relative to the iterate), so the absolute bound scales with max|u|, not with d
        assert d == pytest.approx(ref, rel=1e-6, abs=2e-9 * float(np.abs(un).max()))
        l2, linf = s.residual_norm()
        # the oracle's residual of the GPU's own iterate: the two norms then differ only by the
        # rounding of one residual evaluation (a few ulps of the terms u0, u and dT (Q x A) u)
        ug = s.get_iterate()
        rl2, rlinf = o.residual_norms(ug)
        stiff = 1 + p.dT * 4 * max(p.nu, abs(p.cx), abs(p.cy)) * p.nx ** 2     # bound on ||I|| + ||dT (Q x A)||
        assert abs(l2 - rl2) <= 1e-9 * rl2 + 1e-13 * stiff * float(np.linalg.norm(ug.ravel())), (l2, rl2)
        assert abs(linf - rlinf) <= 1e-9 * rlinf + 1e-13 * stiff * float(np.abs(ug).max()), (linf, rlinf)
        u = un
    np.testing.assert_allclose(s.get_final_value(), u[-1, -1], rtol=0, atol=1e-10 * np.abs(u).max())


def test_schedule_exhausted_and_bad_alpha():
    import paper_2103_12571_b200 as P
    p = W.CONFIGS[1]
    s = _solver(p, p.u0())
    s.set_alpha_schedule([1e-4])
    s.iterate(1)
    with pytest.raises(P.PintError) as e:
        s.iterate(1)
    assert e.value.status == 2
    with pytest.raises(P.PintError) as e:
        s.set_alpha_schedule([1.5])
    assert e.value.status == 2
    s.iterate(0)  # empty call is a no-op


def test_factor_tables_diagonalise():
    """Host tables: S D S^{-1} = Q - r_k D_t H_M and d_k = -alpha^{1/L} e^{-2 pi i k/L}."""
    from oracle.collocation import Tableau
    p = W.CONFIGS[2].replace(L=16)
    s = _solver(p, p.u0())
    s.set_alpha_schedule([1e-5, 0.3])
    tab = Tableau(p.M)
    for a, al in enumerate([1e-5, 0.3]):
        for k in range(p.L):
            dk, S, Si, dkm = s.factors(a, k)
            assert dk == pytest.approx(-al ** (1 / p.L) * np.exp(-2j * np.pi * k / p.L), abs=1e-15)
            r = dk / (1 + dk)
            B = tab.Q - r * tab.Dt @ tab.H
            np.testing.assert_allclose(S @ np.diag(dkm) @ Si, B, atol=1e-13)
            np.testing.assert_allclose(S @ Si, np.eye(p.M), atol=1e-13)


# ---- full BASELINE sizes: sampled spatial modes (the oracle computes each mode exactly) ----------

def _mode_sample(p, cfg):
    rng = np.random.default_rng(100 + cfg)
    if cfg == 3:
        k = np.arange(1, 17)
        kx = np.concatenate([k, p.nx - k, rng.integers(0, p.nx, 8)])
        ky = np.zeros_like(kx)
    elif cfg == 4:
        ks = W.fourier2d_wavevectors(32)
        pick = rng.choice(len(ks), 48, replace=False)
        kx = np.array([ks[i][0] % p.nx for i in pick] + list(rng.integers(0, p.nx, 8)))
        ky = np.array([ks[i][1] % p.ny for i in pick] + list(rng.integers(0, p.ny, 8)))
    else:
        kx = np.concatenate([np.arange(0, 6).repeat(6), rng.integers(0, p.nx, 12)])
        ky = np.concatenate([np.tile(np.arange(0, 6), 6), rng.integers(0, p.ny, 12)])
    return kx, ky


def _gpu_project(s, p, kx, ky):
    """uhat[l, m, j] = sum_n u[l, m, n] e^{-2 pi i (kx x/nx + ky y/ny)} of the device iterate, via
    torch matmuls on the GPU (test-side measurement only)."""
    import torch
    dev = s.iterate_view().device
    xs = torch.arange(p.nx, device=dev, dtype=torch.int64)
    ys = torch.arange(p.ny, device=dev, dtype=torch.int64)
    kxt = torch.as_tensor(np.asarray(kx), device=dev, dtype=torch.int64)
    kyt = torch.as_tensor(np.asarray(ky), device=dev, dtype=torch.int64)
    ex = torch.exp(-2j * np.pi * ((xs[:, None] * kxt[None, :]) % p.nx).to(torch.float64) / p.nx)  # (nx, K)
    ey = torch.exp(-2j * np.pi * ((ys[:, None] * kyt[None, :]) % p.ny).to(torch.float64) / p.ny)  # (ny, K)
    L, M = p.L, p.M
    out = torch.empty((L * M, len(kx)), dtype=torch.complex128, device=dev)
    U = s.iterate_view().view(L * M, p.ny, p.nx)        # float64 in the Hermitian mode (real storage)
    chunk = max(1, (1 << 27) // (p.N * 4))
    for i in range(0, L * M, chunk):
        a = torch.matmul(U[i:i + chunk].to(torch.complex128), ex)   # (c, ny, K)
        out[i:i + chunk] = (a * ey[None]).sum(1)
    torch.cuda.synchronize()
    return out.view(L, M, len(kx)).cpu().numpy()


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_parity_full_size_sampled_modes(cfg):
    p = W.CONFIGS[cfg]
    u0 = p.u0()
    s = _solver(p, u0)
    a_or, a_lib = schedules(p, u0, s)
    s.set_alpha_schedule(a_lib)
    kx, ky = _mode_sample(p, cfg)
    mo = ModeOracle(p, mode_coefficients(p, u0, kx, ky), kx, ky)
    uh = mo.initial()
    errs = []
    for k in range(p.iters):
        uh = mo.iterate(uh, a_or[k])
        s.iterate(1)
        g = _gpu_project(s, p, kx, ky)
        errs.append(float(np.linalg.norm((g - uh).ravel()) / np.linalg.norm(uh.ravel())))
    s.close()
    assert max(errs) <= TOL, errs


# ---- the pipelined plane passes (rows_pipe / cols_pipe) at production plans -------

PIPE_CASES = [
    W.CONFIGS[5].replace(name="pipe_1024sq_M4_L4", L=4, iters=3),
    W.CONFIGS[4].replace(name="pipe_512sq_M3_L8", L=8, iters=3),
    W.CONFIGS[5].replace(name="pipe_1024x512_M2_L4", ny=512, M=2, L=4, iters=3),
    W.CONFIGS[4].replace(name="pipe_512x1024_M1_L8", ny=1024, M=1, L=8, iters=3),
    W.CONFIGS[5].replace(name="pipe_2048x1024_heat_M2_L4", nx=2048, op="heat", nu=1e-2, M=2, L=4, iters=2),
]


@pytest.mark.parametrize("p", PIPE_CASES, ids=lambda p: p.name)
def test_parity_pipe_plans_random(p):
    """Seeded random complex u0 (every spatial mode excited) through the R / C / I passes; the
    kernel list proves the pipelined passes ran."""
    import paper_2103_12571_b200 as PB
    rng = np.random.default_rng(p.nx + p.ny + p.M)
    u0 = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
    s = PB.Solver(p, u0)
    assert "cols_pipe_kernel" in s.kernel_names(), s.kernel_names()
    a = [1e-3, 2e-2, 0.2][:p.iters]
    s.set_alpha_schedule(a)
    o = Oracle(p, u0, "fourier")
    u = o.initial()
    for k in range(p.iters):
        u = o.iterate(u, a[k])
        s.iterate(1)
        assert relative_l2(s.get_iterate(), u) <= TOL, k
    s.close()


@pytest.mark.parametrize("P", [2, 4])
def test_parity_pipe_plans_sharded(P):
    """Time-sharded loopback ranks on a pipelined plan: the node transforms live in the cross-rank
    DFT kernels and the plane passes run without them (NODE = false instantiations)."""
    import paper_2103_12571_b200 as PB
    p = W.CONFIGS[5].replace(name=f"pipe_sharded_P{P}", L=16, M=2, iters=2)
    rng = np.random.default_rng(P)
    u0 = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
    g = PB.Group(p, u0, P)
    assert "cols_pipe_kernel" in g.ranks[0].kernel_names()
    a = [1e-3, 5e-2]
    g.set_alpha_schedule(a)
    o = Oracle(p, u0, "fourier")
    u = o.initial()
    for k in range(2):
        u = o.iterate(u, a[k])
        g.iterate(1)
        assert relative_l2(g.get_iterate(), u) <= TOL, k
    g.close()


@pytest.mark.parametrize("cfg", [1, 2])
def test_cuda_graph_replay_matches_iterate(cfg):
    """pint_graph_create / pint_graph_launch (launch-bound configs): n captured iterations replayed
    on the current buffers equal n pint_iterate calls with the same (fixed) alpha."""
    import paper_2103_12571_b200 as PB
    import torch
    p = W.CONFIGS[cfg]
    u0 = p.u0()
    a = [p.alpha_fixed] * 8
    s1 = PB.Solver(p, u0, stream=torch.cuda.Stream())
    s2 = PB.Solver(p, u0)
    s1.set_alpha_schedule(a)
    s2.set_alpha_schedule(a)
    h = s1.graph_create(2)              # captures iterations 0, 1 (not executed by the capture)
    np.testing.assert_array_equal(s1.get_iterate(), s2.get_iterate())
    for _ in range(3):
        s1.graph_launch(h)
    s1.stream.synchronize()
    s2.iterate(6)
    np.testing.assert_array_equal(s1.get_iterate(), s2.get_iterate())   # same kernels, same order
    s1.graph_destroy(h)
    with pytest.raises(PB.PintError):
        s1.set_phase_timing(True)       # one rank: no phases
    s1.close()
    s2.close()


@pytest.mark.parametrize("p", PIPE_CASES, ids=lambda p: p.name)
def test_parity_pipe_plans_direct_form(p):
    """Direct form (Alg. 1 as printed) on the pipelined plans: the C pass synthesizes
    sig_q r0hat (no R pass), then the I pass; against the oracle's direct-form iteration."""
    import paper_2103_12571_b200 as PB
    rng = np.random.default_rng(p.nx + 3 * p.ny + p.M)
    u0 = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
    s = PB.Solver(p, u0)
    s.set_form("direct")
    assert "cols_pipe_kernel<synth>" in s.kernel_names(), s.kernel_names()
    a = [1e-3, 2e-2, 0.2][:p.iters]
    s.set_alpha_schedule(a)
    o = Oracle(p, u0, "fourier")
    u = o.initial()
    for k in range(p.iters):
        u = o.iterate_direct(u, a[k])
        s.iterate(1)
        assert relative_l2(s.get_iterate(), u) <= TOL, k
    s.close()


@pytest.mark.parametrize("P", [2, 4])
def test_parity_pipe_plans_sharded_direct_form(P):
    import paper_2103_12571_b200 as PB
    p = W.CONFIGS[5].replace(name=f"pipe_sharded_direct_P{P}", L=16, M=2, iters=2)
    rng = np.random.default_rng(10 + P)
    u0 = rng.standard_normal(p.N) + 1j * rng.standard_normal(p.N)
    g = PB.Group(p, u0, P)
    g.set_form("direct")
    a = [1e-3, 5e-2]
    g.set_alpha_schedule(a)
    o = Oracle(p, u0, "fourier")
    u = o.initial()
    for k in range(2):
        u = o.iterate_direct(u, a[k])
        g.iterate(1)
        assert relative_l2(g.get_iterate(), u) <= TOL, k
    g.close()
