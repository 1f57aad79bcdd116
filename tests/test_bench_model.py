"""bench.py's algorithmic byte model covers every launch the library can report, in
every mode, and the mode tables stay below the complex correction form's bytes (host logic, no GPU)."""
import importlib.util
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    return b


def _kernel_names():
    names = set()
    csrc = os.path.join(ROOT, "paper_2103_12571_b200", "csrc")
    for f in os.listdir(csrc):
        if f.endswith((".cu", ".cpp")):
            names |= set(re.findall(r'"([a-z0-9_]+_kernel(?:<[^"]*>)?)"', open(os.path.join(csrc, f)).read()))
    return names


def test_every_reported_kernel_has_a_byte_model():
    b = _bench()
    missing = sorted(n for n in _kernel_names() if n not in b.ALGO_BYTES and n not in b.ALGO_BYTES_DIRECT)
    assert not missing, missing


def test_mode_tables_never_exceed_the_complex_correction_bytes():
    b = _bench()
    for tab in (b.ALGO_BYTES_DIRECT, b.ALGO_BYTES_HERM, b.ALGO_BYTES_HERM_DIRECT):
        for n, v in tab.items():
            assert 0 <= v <= b.ALGO_BYTES.get(n, 48), (n, v)
    # real storage halves every pass of the complex correction form
    for n in ("residual2d_kernel", "tfft_fwd_kernel", "rows_pipe_kernel<fwd>", "cols_pipe_kernel",
              "rows_pipe_kernel<inv>", "tfft_bwd_kernel", "bwd_kernel"):
        assert b.ALGO_BYTES_HERM[n] * 2 == b.ALGO_BYTES[n], n
