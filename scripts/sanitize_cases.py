"""One iteration of each product kernel family on tiny shapes, for compute-sanitizer runs
(scripts/gpu_sanitize.sh): 1-D one-pass PCR (config 1), 1-D pipelined PCR (N = 8192), the TMA
forward tile (L = 256, M = 3), the 2-D plane passes (512^2), their Hermitian and direct forms."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_12571_b200 as PB  # noqa: E402
import workloads as W  # noqa: E402

cases = [(W.CONFIGS[1], "correction", False),
         (W.CONFIGS[3].replace(name="san_pcr1d", nx=8192, L=4, M=2), "correction", False),
         (W.CONFIGS[3].replace(name="san_fwd1d", nx=64, L=256, M=3), "correction", False),
         (W.CONFIGS[4].replace(name="san_pipe", L=4, M=2), "correction", False),
         (W.CONFIGS[4].replace(name="san_pipe_h", L=4, M=2), "correction", True),
         (W.CONFIGS[4].replace(name="san_pipe_d", L=4, M=2), "direct", False)]
for p, form, herm in cases:
    u0 = np.ascontiguousarray(p.u0().real.astype(np.complex128))
    s = PB.Solver(p, u0)
    s.set_form(form)
    if herm:
        s.set_hermitian(True)
    s.set_alpha_schedule([1e-3])
    s.iterate(1)
    u = s.get_iterate()
    assert np.isfinite(u).all()
    print(p.name, form, "herm" if herm else "", s.kernel_names(), flush=True)
    s.close()
print("sanitize cases done")
