"""Builds the in-tree native library paper_2411_16680_b200/liblvsg.so.

CUDA sources are compiled for sm_100a only (`-gencode arch=compute_100a,
code=sm_100a`), with -lineinfo so ncu's source page maps back to them; host
C++ with g++. nvcc cross-compiles without a GPU. Objects are cached under
build/ by source + header mtimes.
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
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "liblvsg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC",
                  "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
                  "-I", os.path.join(ROOT, "include")]
CXXFLAGS = ["-O2", "-std=c++20", "-fPIC", "-Wall", "-I", os.path.join(ROOT, "include"),
            "-I", "/usr/local/cuda/include"]


def _deps_mtime() -> float:
    hdrs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    hdrs.append(os.path.join(ROOT, "include", "lvsg.h"))
    return max(os.path.getmtime(h) for h in hdrs)


def _compile(src: str, hdr_mtime: float, verbose: bool) -> str:
    base = os.path.splitext(os.path.basename(src))[0]
    ext = os.path.splitext(src)[1]
    obj = os.path.join(OBJ, base + (".cu.o" if ext == ".cu" else ".o"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return obj
    if ext == ".cu":
        cmd = [NVCC] + NVFLAGS + ["-c", src, "-o", obj]
    else:
        cmd = ["g++"] + CXXFLAGS + ["-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"compile failed: {src}")
    if verbose and (r.stderr.strip()):
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    hm = _deps_mtime()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, hm, verbose), srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lrt", "-ldl",
                                                              "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
