"""Build libkvr.so (the C-ABI replay engine) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libkvr.so")
SOURCES = ["kvr_api.cu", "kvr_pack.cu", "kvr_kernel.cu", "kvr_nextuse.cu", "kvr_batch.cu"]
DEPS = SOURCES + ["kvr_internal.h", "kvr_device.cuh"]

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-fmad=false",            # no fp64 contraction: bit-exact with the oracle's written order
    "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-warn-spills",
    "-shared",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(ROOT, "include", "kvr.h")]
    return any(os.path.getmtime(d) > t for d in deps)


PROF_LIB = os.path.join(PKG, "libkvr_prof.so")


def build(force: bool = False, verbose: bool = False, profile: bool = False) -> str:
    """libkvr.so; with profile=True the phase-profiling variant libkvr_prof.so
    (-DKVR_PHASE_PROFILE, clock64 per replay phase; used by scripts/, never by tests)."""
    lib = PROF_LIB if profile else LIB
    if not force and not stale(lib):
        return lib
    cmd = [nvcc()] + NVCC_FLAGS + ["-I", os.path.join(ROOT, "include"), "-o", lib + ".tmp"]
    if profile:
        cmd.append("-DKVR_PHASE_PROFILE")
    cmd += [os.path.join(CSRC, f) for f in SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


def build_variant(name: str, defines: list[str]) -> str:
    """Experiment build libkvr_<name>.so with extra -D flags (scripts only, via KVR_LIB)."""
    lib = os.path.join(PKG, f"libkvr_{name}.so")
    cmd = [nvcc()] + NVCC_FLAGS + ["-I", os.path.join(ROOT, "include"), "-o", lib + ".tmp"]
    cmd += [f"-D{d}" for d in defines] + [os.path.join(CSRC, f) for f in SOURCES]
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv, profile="--profile" in sys.argv))
