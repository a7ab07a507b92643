"""Build libsptrsv.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

Each .cu is compiled to an object in parallel (the translation units share no
device symbols), then linked into one shared library.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libsptrsv.so")
OBJDIR = os.path.join(LIBDIR, "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "177"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(INCLUDE, "sptrsv.h")])


def source_digest() -> str:
    """sha256 over the nvcc flags and the sources (paths relative to the repo,
    contents): identifies a build independently of file times (the -lineinfo
    tables embed source mtimes, so the library bytes differ between builds of
    the same sources).  profiles/ncu_traffic.json entries are keyed by it."""
    import hashlib
    h = hashlib.sha256()
    h.update(" ".join(NVCC_FLAGS + ARCH).encode())
    for src in sources():
        h.update(os.path.relpath(src, ROOT).encode() + b"\0")
        with open(src, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _compile(cu: str, headers_mtime: float, force: bool, verbose: bool) -> str:
    obj = os.path.join(OBJDIR, os.path.basename(cu)[:-3] + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(cu), headers_mtime):
        return obj
    tmp = obj + ".tmp.o"          # a fixed name (nvcc records the output path)
    cmd = [nvcc(), *NVCC_FLAGS, "-I" + INCLUDE, "-I" + CSRC, "-c", "-o", tmp, cu]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, obj)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    srcs = sources()
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(s) for s in srcs):
        return LIB
    cu = [s for s in srcs if s.endswith(".cu")]
    hdr = max(os.path.getmtime(s) for s in srcs if not s.endswith(".cu"))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(cu))) as ex:
        objs = list(ex.map(lambda c: _compile(c, hdr, force, verbose), cu))
    tmp = LIB + ".tmp.so"
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    # the host objects name nvcc's per-process temporary files (tmpxft_<pid>_...)
    # in their local symbol table (not needed: ctypes binds the dynamic symbols).
    # The library bytes still depend on the sources' mtimes (-lineinfo);
    # source_digest() identifies a build
    try:
        subprocess.check_call(["strip", "--strip-unneeded", tmp])
    except (OSError, subprocess.CalledProcessError):
        pass
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
