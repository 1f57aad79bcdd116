"""Host-logic checks of the register FFT engine's plan (paper_2103_12571_b200/csrc/fft_reg.cuh),
re-derived here from the rules its header states (no GPU, no library call):

* the pass decomposition N = R0 R1 R2 (B0 = min(4, n), B1 = min(4, n - B0), B2 = rest) with
  per-pass radix-R DFTs on positions beta m_i + j + s_i t and twiddles w_{m_i}^{j bitrev(t)}
  leaves frequency bitrev_n(P) at position P, and the reverse passes (conjugate twiddle, inverse
  radix DFT) return N x  -- checked against numpy's FFT;
* the shared-memory swizzle F is a bijection of every line and makes every quarter-warp access
  of every pass, and (lines of >= 16 points) of the column staging with line stride
  N + max(1, 8/TC), bank-conflict free (16-byte slots, 8 per 128-byte bank row).
"""
import numpy as np
import pytest


def plan(n, maxb=4):
    b0 = min(maxb, n)
    b1 = min(maxb, n - b0)
    return [b for b in (b0, b1, n - b0 - b1) if b > 0]


def bitrev(x, b):
    r = 0
    for i in range(b):
        r |= ((x >> i) & 1) << (b - 1 - i)
    return r


def swizzle(n, p, maxb=4):
    bs = plan(n, maxb)
    h = 0
    if len(bs) >= 2:
        bl = bs[-1]
        h ^= (p >> max(bl, 3)) & (7 if bl >= 3 else (1 << bl) - 1)
    if len(bs) == 3 and bs[2] < 3:
        h ^= ((p >> (n - bs[0])) & ((8 >> bs[2]) - 1)) << bs[2]
    return p ^ h


def passes(n, maxb=4):
    """(b, logm, logs) per pass"""
    out, logm = [], n
    for b in plan(n, maxb):
        out.append((b, logm, logm - b))
        logm -= b
    return out


def positions(n, p, tau, u, maxb=4):
    bs = plan(n, maxb)
    tpl = (1 << n) >> bs[0]
    b, logm, logs = passes(n, maxb)[p]
    g = tau + tpl * u
    return [((g >> logs) << logm) + (g & ((1 << logs) - 1)) + (t << logs) for t in range(1 << b)]


def run_engine(n, x, inverse=False):
    N = 1 << n
    bs = plan(n)
    E = 1 << bs[0]
    tpl = N // E
    a = x.astype(np.complex128).copy()
    order = range(len(bs)) if not inverse else reversed(range(len(bs)))
    for p in order:
        b, logm, logs = passes(n)[p]
        R, s = 1 << b, 1 << logs
        new = a.copy()
        for tau in range(tpl):
            for u in range(E // R):
                g = tau + tpl * u
                j = g & (s - 1)
                P = positions(n, p, tau, u)
                tw = np.exp(-2j * np.pi * j * np.array([bitrev(t, b) for t in range(R)]) / (1 << logm))
                v = a[P]
                if not inverse:
                    X = np.fft.fft(v)
                    new[P] = np.array([X[bitrev(t, b)] for t in range(R)]) * tw
                else:
                    v = v * np.conj(tw)
                    nat = np.array([v[bitrev(t, b)] for t in range(R)])
                    new[P] = np.fft.ifft(nat) * R
        a = new
    return a


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7, 8, 9, 10])
def test_plan_output_is_bit_reversed_dft_and_inverse_restores(n):
    rng = np.random.default_rng(n)
    N = 1 << n
    x = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    y = run_engine(n, x)
    ref = np.fft.fft(x)
    np.testing.assert_allclose(y, ref[[bitrev(P, n) for P in range(N)]], rtol=0, atol=1e-12 * np.abs(ref).max())
    z = run_engine(n, y, inverse=True)
    np.testing.assert_allclose(z / N, x, rtol=0, atol=1e-13 * np.abs(x).max())


def test_plans_have_at_most_three_passes_of_radix_at_most_16():
    for n in range(2, 13):
        bs = plan(n)
        assert sum(bs) == n and len(bs) <= 3 and max(bs) <= 4


@pytest.mark.parametrize("n", list(range(2, 13)))
def test_swizzle_bijective_and_conflict_free(n):
    N = 1 << n
    assert sorted(swizzle(n, p) for p in range(N)) == list(range(N))
    bs = plan(n)
    E = 1 << bs[0]
    tpl = N // E
    for p, (b, _, _) in enumerate(passes(n)):
        R = 1 << b
        for u in range(E // R):
            for t in range(R):
                for t0 in range(0, tpl, 8):          # quarter-warps of one line (16-byte accesses)
                    slots = [swizzle(n, positions(n, p, tau, u)[t]) % 8 for tau in range(t0, min(t0 + 8, tpl))]
                    assert len(set(slots)) == len(slots), (n, p, u, t, t0)
    if N < 16:
        return                                       # tiny lines (tests only): staging conflicts are harmless
    for tc in (1, 2, 4, 8, 16, 32):                  # cp.async column staging, lanes column-fastest
        pad = 1 if tc >= 8 else 8 // tc
        for y0 in range(0, N, max(1, 8 // tc)):
            lanes = [(lane % tc, y0 + lane // tc) for lane in range(8) if y0 + lane // tc < N]
            slots = [(c * (N + pad) + swizzle(n, y)) % 8 for c, y in lanes]
            assert len(set(slots)) == len(slots), (n, tc, y0)
