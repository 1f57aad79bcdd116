"""Builds libpint.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension machinery)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpint.so")
SOURCES = ["kernels.cu", "spatial2d.cu", "pint_abi.cpp", "host_numerics.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
LIBS = ["-lnccl"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def build(verbose: bool = False, force: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "internal.h"), os.path.join(CSRC, "host_numerics.h"), os.path.join(CSRC, "fft_reg.cuh"),
                   os.path.join(CSRC, "device_common.cuh"),
                   os.path.join(ROOT, "include", "pint.h")]
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(d) for d in deps):
        return LIB
    cmd = [NVCC, *FLAGS, "-shared", "-o", LIB, *srcs, "-I", os.path.join(ROOT, "include"), *LIBS]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stdout.write(res.stderr)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force=True)
    print(LIB)
