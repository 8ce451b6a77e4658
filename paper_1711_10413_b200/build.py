"""In-tree build of the sm_100a library (``_build/libompds_b200.so``).

``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo`` over
``csrc/ompds_kernels.cu`` (device runtime + generic-mode kernels + C-ABI
launchers) and ``csrc/ompds_host.cpp`` (layout builder, occupancy, trap
strings).  nvcc cross-compiles without a GPU, so this runs in the CPU
container; the .so travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libompds_b200.so")
SOURCES = [os.path.join(CSRC, "ompds_kernels.cu"), os.path.join(CSRC, "ompds_team.cu"),
           os.path.join(CSRC, "ompds_probe.cu"), os.path.join(CSRC, "ompds_host.cpp"),
           os.path.join(CSRC, "ompds_manifest.cpp")]
HEADERS = [os.path.join(CSRC, "ompds_device.cuh"), os.path.join(CSRC, "ompds_generic.cuh"),
           os.path.join(os.path.dirname(HERE), "include", "ompds.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def sources_sha256() -> str:
    """Hash of the device/host sources the library is built from: stamps
    measurements (ncu traffic captures) with the build they were taken on."""
    import hashlib
    h = hashlib.sha256()
    for f in SOURCES + HEADERS:
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


EXAMPLE_SRCS = [os.path.join(os.path.dirname(HERE), "examples", f)
                for f in ("reduction_region.cu", "nested_region.cu")]
EXAMPLE_LIB = os.path.join(OUT_DIR, "libompds_example.so")


def build_example(force: bool = False) -> str:
    """examples/reduction_region.cu: a user-defined region program compiled
    against the runtime headers and linked to libompds_b200.so."""
    if not force and os.path.exists(EXAMPLE_LIB) and all(
            os.path.getmtime(f) <= os.path.getmtime(EXAMPLE_LIB)
            for f in EXAMPLE_SRCS + [LIB] + HEADERS):
        return EXAMPLE_LIB
    cmd = [nvcc()] + NVCC_FLAGS + ["-I", CSRC, "-o", EXAMPLE_LIB + ".tmp"] + EXAMPLE_SRCS + [
                                   "-L", OUT_DIR, "-lompds_b200", "-Xlinker", "-rpath,$ORIGIN"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode}) building {EXAMPLE_LIB}")
    os.replace(EXAMPLE_LIB + ".tmp", EXAMPLE_LIB)
    return EXAMPLE_LIB


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        build_example()
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = LIB + ".tmp"
    cmd = [nvcc()] + NVCC_FLAGS + ["-o", tmp] + SOURCES
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    with open(os.path.join(OUT_DIR, "ptxas.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + log)
    if res.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed ({res.returncode}) building {LIB}")
    if verbose:
        sys.stderr.write(log)
    os.replace(tmp, LIB)
    build_example(force=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
