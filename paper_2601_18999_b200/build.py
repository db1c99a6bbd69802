"""Build libkvr.so (the C-ABI replay engine) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import hashlib
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


def source_hash() -> str:
    """SHA-256 prefix over the compiled sources, the header and the nvcc flags; compiled
    into the library as kvr_build_id() (build provenance)."""
    h = hashlib.sha256()
    for path in [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(ROOT, "include", "kvr.h")]:
        h.update(os.path.basename(path).encode())
        with open(path, "rb") as f:
            h.update(f.read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()[:16]


_MARK = b"KVR_BUILD_ID="


def embedded_hash(lib: str) -> str:
    """The source hash a built library carries (read from the file, not loaded)."""
    try:
        with open(lib, "rb") as f:
            data = f.read()
    except OSError:
        return ""
    i = data.find(_MARK)
    return data[i + len(_MARK): i + len(_MARK) + 16].decode(errors="replace") if i >= 0 else ""


def stale(lib: str = LIB) -> bool:
    """True unless `lib` was compiled from exactly the current sources and flags."""
    return embedded_hash(lib) != source_hash()


PROF_LIB = os.path.join(PKG, "libkvr_prof.so")


def build(force: bool = False, verbose: bool = False, profile: bool = False) -> str:
    """libkvr.so; with profile=True the phase-profiling variant libkvr_prof.so
    (-DKVR_PHASE_PROFILE, clock64 per replay phase; used by scripts/, never by tests)."""
    lib = PROF_LIB if profile else LIB
    if not force and not stale(lib):
        return lib
    cmd = [nvcc()] + NVCC_FLAGS + ["-I", os.path.join(ROOT, "include"), "-o", lib + ".tmp",
                                   f"-DKVR_BUILD_ID=\"{source_hash()}\""]
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
    cmd = [nvcc()] + NVCC_FLAGS + ["-I", os.path.join(ROOT, "include"), "-o", lib + ".tmp",
                                   f"-DKVR_BUILD_ID=\"{source_hash()}\""]
    cmd += [f"-D{d}" for d in defines] + [os.path.join(CSRC, f) for f in SOURCES]
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv, profile="--profile" in sys.argv))
