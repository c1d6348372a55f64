"""Build libtn.so (the CUDA path) in-tree with nvcc for sm_100a.

`python paper_1801_09449_b200/build.py [--force]` (run it by path: importing the
package needs the library) or `__graft_entry__.build()`.  Object files go
to paper_1801_09449_b200/build/ and are rebuilt when a source or header is
newer; the shared library is linked next to this file so it travels with the
repo snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libtn.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-Wall", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include")]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, extra):
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if _stale(obj, [src] + _headers()):
        cmd = [NVCC] + ARCH + FLAGS + extra + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if r.stderr.strip() and os.environ.get("TN_BUILD_VERBOSE"):
            print(r.stderr, file=sys.stderr)
    return obj


def build_library(force: bool = False, extra=None, lib_path: str = None, obj_dir: str = None) -> str:
    global OBJ, LIB
    if obj_dir:
        OBJ = obj_dir
    if lib_path:
        LIB = lib_path
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if force:
        for o in glob.glob(os.path.join(OBJ, "*.o")):
            os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, extra or []), srcs))
    if force or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "shared", "-o", tmp] + objs + ["-lnccl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    if "--trace" in sys.argv:   # profiling build: per-role wait counters (TN_TRACE), libtn_trace.so
        print(build_library(force="--force" in sys.argv, extra=["-DTN_TRACE"],
                            lib_path=os.path.join(HERE, "libtn_trace.so"), obj_dir=os.path.join(HERE, "build_trace")))
    elif "--ab" in sys.argv:     # measurement A/B switches read from the environment (TN_AB), libtn_ab.so
        print(build_library(force="--force" in sys.argv, extra=["-DTN_AB"],
                            lib_path=os.path.join(HERE, "libtn_ab.so"), obj_dir=os.path.join(HERE, "build_ab")))
    elif "--check" in sys.argv:  # device bounds checks (TN_CHECK), libtn_check.so
        print(build_library(force="--force" in sys.argv, extra=["-DTN_CHECK"],
                            lib_path=os.path.join(HERE, "libtn_check.so"), obj_dir=os.path.join(HERE, "build_check")))
    else:
        print(build_library(force="--force" in sys.argv))
