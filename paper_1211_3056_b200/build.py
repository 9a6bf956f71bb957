"""Build the sm_100a shared library in-tree (nvcc cross-compiles without a GPU).

    python -m paper_1211_3056_b200.build

produces paper_1211_3056_b200/_lib/libhrb200.so, the C-ABI of
include/hrb200.h.  The library is git-ignored but travels with the repo
snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libhrb200.so")
PEAK_LIB = os.path.join(LIBDIR, "libhrbpeak.so")  # INT-pipe microbenchmark (roofline denominator)
SOURCES = [os.path.join(CSRC, "hrb200.cu")]
PEAK_SOURCES = [os.path.join(CSRC, "intpeak.cu")]
HOST_LIB = os.path.join(LIBDIR, "libhrbhost.so")  # native host polygen + confirmation (no CUDA)
HOST_SOURCES = [os.path.join(CSRC, "host", "hrb_host.cpp")]
HOST_HEADERS = [os.path.join(CSRC, "host", f) for f in ("bign.h", "mpexp.h", "decide.h", "polygen.h")] + [
    os.path.join(ROOT, "include", "hrb_host.h")]
HOST_FLAGS = ["-O3", "-std=c++17", "-fopenmp", "-fPIC", "-shared", "-Wall", "-Wextra", "-Wno-unused-parameter",
              "-Wno-maybe-uninitialized"]
HEADERS = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cuh", ".h"))] + [
    os.path.join(CSRC, "host", f) for f in ("bign.h", "mpexp.h", "decide.h", "polygen.h")] + [
    os.path.join(ROOT, "include", f) for f in ("hrb200.h", "hrb_host.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libhrb200.so")


def source_hash(sources: list) -> str:
    """Content hash of a library's sources, headers and flags (mtimes do not
    survive copies of the tree, e.g. the snapshot sent to a GPU box)."""
    import hashlib

    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for p in sorted(sources + HEADERS):
        with open(p, "rb") as fh:
            h.update(os.path.basename(p).encode() + b"\0" + fh.read())
    return h.hexdigest()[:32]


def _stale(lib: str, sources: list) -> bool:
    if not os.path.exists(lib) or not os.path.exists(lib + ".srchash"):
        return True
    with open(lib + ".srchash") as fh:
        return fh.read().strip() != source_hash(sources)


def _compile(lib: str, sources: list, verbose: bool) -> None:
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = lib + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, "-o", tmp, *sources]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"nvcc failed ({proc.returncode}): {' '.join(cmd)}")
    if verbose:
        sys.stderr.write(proc.stderr)
    os.replace(tmp, lib)
    with open(lib + ".srchash.tmp", "w") as fh:
        fh.write(source_hash(sources))
    os.replace(lib + ".srchash.tmp", lib + ".srchash")


def cxx() -> str:
    """The first C++ compiler that links -fopenmp (some images put a g++
    without libgomp first in $CXX / on PATH)."""
    for cand in (os.environ.get("CXX"), "/usr/bin/g++", shutil.which("g++")):
        if not cand or not os.path.exists(cand):
            continue
        probe = subprocess.run([cand, "-fopenmp", "-x", "c++", "-", "-o", os.devnull], input="int main(){return 0;}",
                               capture_output=True, text=True)
        if probe.returncode == 0:
            return cand
    raise RuntimeError("no g++ with OpenMP found: needed for the native host library libhrbhost.so")


def _host_hash() -> str:
    import hashlib

    h = hashlib.sha256(" ".join(HOST_FLAGS).encode())
    for p in sorted(HOST_SOURCES + HOST_HEADERS):
        with open(p, "rb") as fh:
            h.update(os.path.basename(p).encode() + b"\0" + fh.read())
    return h.hexdigest()[:32]


def build_host(force: bool = False, verbose: bool = False) -> str:
    """Compile libhrbhost.so (g++ -O3 -fopenmp) if missing or stale."""
    stamp = HOST_LIB + ".srchash"
    want = _host_hash()
    if not force and os.path.exists(HOST_LIB) and os.path.exists(stamp) and open(stamp).read().strip() == want:
        return HOST_LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = HOST_LIB + ".tmp"
    cmd = [cxx(), *HOST_FLAGS, "-o", tmp, *HOST_SOURCES]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"g++ failed ({proc.returncode}): {' '.join(cmd)}")
    if verbose:
        sys.stderr.write(proc.stderr)
    os.replace(tmp, HOST_LIB)
    with open(stamp + ".tmp", "w") as fh:
        fh.write(want)
    os.replace(stamp + ".tmp", stamp)
    return HOST_LIB


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libhrb200.so (and the INT-peak probe libhrbpeak.so) for
    sm_100a, and the native host library, if missing or stale; return the
    main library's path."""
    if force or _stale(LIB, SOURCES):
        _compile(LIB, SOURCES, verbose)
    if force or _stale(PEAK_LIB, PEAK_SOURCES):
        _compile(PEAK_LIB, PEAK_SOURCES, verbose)
    build_host(force, verbose)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
