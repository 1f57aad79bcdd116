"""Builds libpint.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension machinery).
Each translation unit compiles to its own object in parallel; one nvcc call links the library."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libpint.so")
# A/B experiment library (-DPINT_EXPERIMENTS: reads the PINT_* switches of internal.h); never the
# product: bench.py refuses it unless --allow-experiments, and records it
LIB_EXP = os.path.join(HERE, "libpint_exp.so")
SOURCES = ["kernels.cu", "spatial2d.cu", "pcr1d.cu", "generic.cu", "pint_abi.cpp", "host_numerics.cpp"]
HEADERS = ["internal.h", "host_numerics.h", "fft_reg.cuh", "device_common.cuh", "residual.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
LIBS = ["-lnccl"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _compile(src: str, objdir: str, extra: list[str]) -> tuple[str, subprocess.CompletedProcess]:
    obj = os.path.join(objdir, os.path.splitext(os.path.basename(src))[0] + ".o")
    cmd = [NVCC, *FLAGS, *extra, "-c", "-o", obj, src, "-I", os.path.join(ROOT, "include")]
    return obj, subprocess.run(cmd, capture_output=True, text=True)


def build(verbose: bool = False, force: bool = False, experiments: bool = False) -> str:
    lib = LIB_EXP if experiments else LIB
    objdir = OBJ + ("_exp" if experiments else "")
    extra = ["-DPINT_EXPERIMENTS"] if experiments else []
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "pint.h")]
    if not force and os.path.exists(lib) and all(os.path.getmtime(lib) >= os.path.getmtime(d) for d in deps):
        return lib
    os.makedirs(objdir, exist_ok=True)
    log = os.path.join(HERE, "build_exp.log" if experiments else "build.log")
    hdr_time = max(os.path.getmtime(d) for d in deps if d not in srcs)

    def obj_of(src: str) -> str:
        return os.path.join(objdir, os.path.splitext(os.path.basename(src))[0] + ".o")

    def fresh(src: str) -> bool:   # incremental: an object newer than its source and every header
        o = obj_of(src)
        return (not force and os.path.exists(o) and os.path.getmtime(o) >= os.path.getmtime(src)
                and os.path.getmtime(o) >= hdr_time)

    def unit(src: str):
        if fresh(src):
            return obj_of(src), subprocess.CompletedProcess([src, "(up to date)"], 0, "", "")
        return _compile(src, objdir, extra)

    with cf.ThreadPoolExecutor(len(srcs)) as ex:
        results = list(ex.map(unit, srcs))
    text = "".join(" ".join(r.args) + "\n" + r.stdout + r.stderr for _, r in results)
    failed = [r for _, r in results if r.returncode != 0]
    if not failed:
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib,
               *[o for o, _ in results], *LIBS]
        res = subprocess.run(cmd, capture_output=True, text=True)
        text += " ".join(cmd) + "\n" + res.stdout + res.stderr
        if res.returncode != 0:
            failed = [res]
    with open(log, "w") as f:
        f.write(text)
    if failed:
        sys.stderr.write("".join(r.stdout + r.stderr for r in failed))
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stdout.write(text)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True, experiments="--experiments" in sys.argv))
