"""Build libfp8bs.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_2412_19437_b200.build [--verbose]

Flags: -gencode arch=compute_100a,code=sm_100a, -lineinfo for ncu source mapping, IEEE-strict
math (no --use_fast_math; -prec-div=true -ftz=false) because the quantizers are bit-exact
against the oracle, and a static CUDA runtime so the library loads (and its validation paths
run) on machines without a CUDA driver.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libfp8bs.so")
# The same sources built with -DFP8BS_TEST_HOOKS=1: exports fp8bs_internal_* hooks (forced GEMM tile
# variant, debug timestamps) for tests/ and tools/ only; the product library has none of them.
TEST_LIB = os.path.join(PKG, "libfp8bs_testhooks.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-prec-div=true", "-prec-sqrt=true", "-ftz=false", "-fmad=true",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "-cudart", "static",
    "--expt-relaxed-constexpr",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(ROOT, "include", "fp8bs.h")]


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in deps())


def _build_one(lib: str, defines: list[str], verbose: bool) -> list:
    """Start the nvcc compiles of every source for `lib`; returns (lib, objs, procs)."""
    tag = os.path.splitext(os.path.basename(lib))[0]
    objs, procs = [], []
    for src in sources():
        obj = os.path.join(CSRC, f"{os.path.basename(src)}.{tag}.o")
        cmd = [NVCC, *NVCC_FLAGS, *defines, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    return [lib, objs, procs]


def _link(lib: str, objs: list, procs: list, verbose: bool):
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(f"--- {os.path.basename(src)} ({os.path.basename(lib)})\n{out}")
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = lib + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-lpthread", "-ldl", "-lrt"]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)


def build(force: bool = False, verbose: bool = False, test_hooks: bool = True) -> str:
    """Build libfp8bs.so (and, unless test_hooks=False, libfp8bs_testhooks.so) in parallel."""
    jobs = []
    if force or not up_to_date(LIB):
        jobs.append(_build_one(LIB, [], verbose))
    if test_hooks and (force or not up_to_date(TEST_LIB)):
        jobs.append(_build_one(TEST_LIB, ["-DFP8BS_TEST_HOOKS=1"], verbose))
    for lib, objs, procs in jobs:
        _link(lib, objs, procs, verbose)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="--verbose" in sys.argv)
    print(LIB)
