"""In-tree build of the native library paper_1707_09683_b200/_lib/liblhmm_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a for every CUDA translation unit
(the kernels are sm_100a-only: DPX, cp.async.bulk), compiled in parallel and
linked into one shared library with an extern "C" surface
(include/lhmm_b200.h).  Incremental: a unit is rebuilt when it or a header
is newer than its object.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "liblhmm_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fopenmp",
          "-I" + os.path.join(ROOT, "include")]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) + \
        glob.glob(os.path.join(CSRC, "*.inc")) + \
        [os.path.join(ROOT, "include", "lhmm_b200.h"), os.path.join(CSRC, "gen", "registry.inc")]


def _stale(src, obj, hdr_mtime):
    if not os.path.exists(obj):
        return True
    m = os.path.getmtime(obj)
    return os.path.getmtime(src) > m or hdr_mtime > m


def _compile(src, obj, verbose):
    cmd = [NVCC] + ARCH + COMMON + ["-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC] + COMMON + ["-x", "cu", "-c", src, "-o", obj] + ARCH
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr.strip():
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose=False, jobs=None, defines=(), tag=""):
    """Build the library; `defines`/`tag` produce experimental side builds
    (_build<tag>/, _lib<tag>/) used only by tuning sweeps."""
    global BUILD, LIBDIR, LIB, COMMON
    if tag:
        BUILD = os.path.join(PKG, "_build" + tag)
        LIBDIR = os.path.join(PKG, "_lib" + tag)
        LIB = os.path.join(LIBDIR, "liblhmm_b200.so")
    COMMON = COMMON + [f"-D{d}" for d in defines]
    sys.path.insert(0, CSRC)
    try:
        import gen_instances
        gen_instances.main()
    finally:
        sys.path.pop(0)
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")) +
                  glob.glob(os.path.join(CSRC, "gen", "*.cu")))
    hdr_mtime = max(os.path.getmtime(h) for h in _headers() if os.path.exists(h))
    todo, objs = [], []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if _stale(s, o, hdr_mtime):
            todo.append((s, o))
    if todo:
        with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 8) as ex:
            list(ex.map(lambda so: _compile(so[0], so[1], verbose), todo))
    if todo or not os.path.exists(LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-Xcompiler", "-fPIC,-fopenmp", "-o", LIB] + objs + \
            ["-lgomp", "-lz"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if not tag:
        build_examples()
    return LIB


def build_examples():
    """Plain-C programs against the C ABI only (examples/*.c -> examples/bin/)."""
    src_dir = os.path.join(ROOT, "examples")
    out_dir = os.path.join(src_dir, "bin")
    os.makedirs(out_dir, exist_ok=True)
    for src in sorted(glob.glob(os.path.join(src_dir, "*.c"))):
        exe = os.path.join(out_dir, os.path.splitext(os.path.basename(src))[0])
        if os.path.exists(exe) and os.path.getmtime(exe) > max(os.path.getmtime(src),
                                                              os.path.getmtime(LIB)):
            continue
        cmd = ["gcc", "-O2", "-Wall", "-std=c11", "-I" + os.path.join(ROOT, "include"), src,
               "-o", exe, "-L" + LIBDIR, "-llhmm_b200",
               "-Wl,-rpath,$ORIGIN/../../paper_1707_09683_b200/_lib"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"example build failed: {' '.join(cmd)}\n{r.stderr}")


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("-v", action="store_true")
    ap.add_argument("-D", action="append", default=[])
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    print(build(verbose=a.v, defines=a.D, tag=a.tag))
