"""Build the native library libdgds_b200.so in-tree (sm_100a only).

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 over csrc/*.cu + the
host C++ (server.cpp, host_query.cpp, replica.cpp, wire.cpp) -> paper_2511_14617_b200/libdgds_b200.so.
The bench/test trace generator is a separate host library (tools/workload, build_workload).
The built .so is git-ignored but travels to the GPU box with the snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdgds_b200.so")
SOURCES = ["kernels.cu", "peer.cu", "server.cpp", "host_query.cpp", "replica.cpp", "wire.cpp", "cluster.cpp", "px_driver.cpp"]
# the trace generator of the bench / tests: a separate host-only tools library
WORKLOAD_SRC = os.path.join(HERE, "..", "tools", "workload", "workload_gen.cpp")
WORKLOAD_LIB = os.path.join(HERE, "..", "tools", "workload", "libdgds_workload.so")


def build_workload(force: bool = False) -> str:
    if force or not os.path.exists(WORKLOAD_LIB) or os.path.getmtime(WORKLOAD_SRC) > os.path.getmtime(WORKLOAD_LIB):
        subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-o", WORKLOAD_LIB, WORKLOAD_SRC], check=True)
    return WORKLOAD_LIB
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


# Test-only variants: the same sources with a compile-time switch, loaded when the environment
# names them (DGDS_LIB_VARIANT, see _lib.py). "hash10" truncates the stored content hash to 10
# bits, so content probes collide constantly and every exact-key fallback and long probe run in
# K1 / K2 is exercised by the parity tests. "checked" adds device bounds checks (DGDS_CHECK in
# trie.cuh) that flag any index outside its arena (compute-sanitizer is unavailable on the pool).
VARIANTS = {"hash10": ["-DDGDS_TEST_HASH_BITS=10"], "checked": ["-DDGDS_CHECKED"]}


def lib_path(variant: str | None = None) -> str:
    return LIB if not variant else os.path.join(HERE, "libdgds_b200_%s.so" % variant)


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "dgds_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, variant: str | None = None) -> str:
    build_workload(force)
    lib = lib_path(variant)
    if not force and not _stale(lib):
        return lib
    objs = []
    common = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3"] + ARCH
    common += VARIANTS[variant] if variant else []
    outdir = os.path.join(HERE, "_build" + ("_" + variant if variant else ""))
    os.makedirs(outdir, exist_ok=True)
    for src in SOURCES:
        obj = os.path.join(outdir, os.path.splitext(src)[0] + ".o")
        # host sources include the device layout header, so everything goes through nvcc as CUDA
        cmd = [nvcc()] + common + ["-x", "cu", "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = lib + ".tmp"
    subprocess.run([nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    for v in VARIANTS:
        if "--variants" in sys.argv:
            print(build(force="--force" in sys.argv, variant=v))
