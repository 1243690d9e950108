"""Build the sm_100a extension libcbgx.so (and the C++ drop-in libcbg_b200.so).

nvcc cross-compiles for sm_100a without a GPU, so this runs on the CPU
container as well as on the B200 box. Objects are compiled in parallel and
only rebuilt when a source or header changed.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libcbgx.so")
DROPIN_LIB = os.path.join(PKG, "libcbg_b200.so")
CLI_BIN = os.path.join(PKG, "cbgmres")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# Host code: no FMA contraction, so host-side arithmetic (Givens) rounds
# exactly like the reference build (no -march, src/CMakeLists.txt).
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-ffp-contract=off",
                  "-I" + INCLUDE, "-I" + CSRC, "--expt-relaxed-constexpr"]
# Development only: extra -D geometry flags for A/B builds (e.g.
# CBGX_NVFLAGS_EXTRA="-DFUSED_WARPS=12 -DFUSED_STEPS=5").
NVFLAGS += os.environ.get("CBGX_NVFLAGS_EXTRA", "").split()


def _headers_digest() -> str:
    h = hashlib.sha256()
    for f in sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                    glob.glob(os.path.join(INCLUDE, "*.h")) + glob.glob(os.path.join(INCLUDE, "cbg", "*.hpp"))):
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(NVFLAGS).encode())
    return h.hexdigest()[:16]


def _compile(src: str, obj: str) -> None:
    cmd = [NVCC] + NVFLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(src)}:\n{r.stderr}")


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    digest = _headers_digest()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = []
    objs = []
    for src in srcs:
        obj = os.path.join(BUILD, os.path.basename(src) + "." + digest + ".o")
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < os.path.getmtime(src):
            jobs.append((src, obj))
    for stale in glob.glob(os.path.join(BUILD, "*.o")):
        if stale not in objs:
            os.remove(stale)
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            list(ex.map(lambda a: _compile(*a), jobs))
    if force or jobs or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-ldl", "-lpthread", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stderr)
    _build_dropin(force)
    if verbose:
        print("built", LIB)
    return LIB


def _build_dropin(force: bool) -> None:
    """C++ drop-in for the reference's cbg:: API over the C-ABI."""
    srcs = sorted(glob.glob(os.path.join(CSRC, "dropin", "*.cpp")))
    if not srcs:
        return
    deps = srcs + glob.glob(os.path.join(INCLUDE, "cbg", "*.hpp")) + [os.path.join(INCLUDE, "cbgx.h"), LIB]
    if not force and os.path.exists(DROPIN_LIB) and all(os.path.getmtime(d) <= os.path.getmtime(DROPIN_LIB) for d in deps):
        return
    cmd = ["g++", "-std=gnu++20", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-I" + INCLUDE,
           "-o", DROPIN_LIB] + srcs + ["-L" + PKG, "-lcbgx", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("drop-in build failed:\n" + r.stderr)
    _build_cli(True)


def _build_cli(force: bool) -> None:
    """The `cbgmres` tool (the reference's tools/cbgmres_main.cpp) over libcbg_b200.so."""
    src = os.path.join(CSRC, "tools", "cbgmres.cpp")
    if not os.path.exists(src):
        return
    if not force and os.path.exists(CLI_BIN) and os.path.getmtime(CLI_BIN) >= max(
            os.path.getmtime(src), os.path.getmtime(DROPIN_LIB)):
        return
    cmd = ["g++", "-std=gnu++20", "-O2", "-I" + INCLUDE, "-o", CLI_BIN, src,
           "-L" + PKG, "-lcbg_b200", "-lcbgx", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("cbgmres build failed:\n" + r.stderr)


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
