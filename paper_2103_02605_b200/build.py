"""Build libfcirc.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo).

Each translation unit is compiled to an object in parallel (the two field executors dominate the
build time), then linked into one shared library.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
OBJ_DIR = os.path.join(LIB_DIR, "obj")
LIB = os.path.join(LIB_DIR, "libfcirc.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
SOURCES = ["matvec_gold.cu", "matvec_u32.cu", "matvec_u32m.cu", "matvec_m31.cu", "api.cu", "plan.cpp", "probe.cu"]
HEADERS = ["modarith.cuh", "fcirc_kernels.cuh", "matvec_impl.cuh", "apps.cuh", "plan.h", "runtime.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    paths = [os.path.join(CSRC, d) for d in SOURCES + HEADERS] + [os.path.join(INCLUDE, "fcirc.h")]
    return any(os.path.getmtime(p) > t for p in paths if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, extra_flags=()) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OBJ_DIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")

    def compile_one(src):
        obj = os.path.join(OBJ_DIR, src.rsplit(".", 1)[0] + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *extra_flags, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        return obj

    hdr_t = max(os.path.getmtime(p) for p in [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "fcirc.h")]
                if os.path.exists(p))

    def obj_of(src):
        return os.path.join(OBJ_DIR, src.rsplit(".", 1)[0] + ".o")

    def stale_obj(src):   # object older than its source or any shared header (or extra flags given)
        o = obj_of(src)
        return force or extra_flags or not os.path.exists(o) or \
            os.path.getmtime(o) < max(os.path.getmtime(os.path.join(CSRC, src)), hdr_t)

    todo = [src for src in SOURCES if stale_obj(src)]
    with cf.ThreadPoolExecutor(max_workers=max(1, len(todo))) as ex:
        list(ex.map(compile_one, todo))
    objs = [obj_of(src) for src in SOURCES]
    cmd = [nvcc, *ARCH, "-shared", *objs, "-o", LIB + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
