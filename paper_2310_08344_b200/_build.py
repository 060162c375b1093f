"""Build liblexint_b200.so in-tree with nvcc for sm_100a (no JIT cache).

Sources: csrc/*.cu (kernels) and csrc/*.cpp (host runtime, C ABI); headers
csrc/*.h and include/lexint.h.  Objects go to build/, the shared object to
paper_2310_08344_b200/liblexint_b200.so (git-ignored, travels with gpurun).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "liblexint_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    """torch's bundled NCCL 2.28 (nvidia-nccl wheel): headers + libnccl.so.2."""
    try:
        import nvidia
        bases = [os.path.join(p, "nccl") for p in nvidia.__path__]
    except Exception:
        return None
    for base in bases:
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    return None


def _flags():
    f = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    # build-time extras (the bounds-checked debug build of tools/debug_bounds.sh: -DLX_DEBUG_BOUNDS)
    f += [x for x in os.environ.get("NVCC_EXTRA", "").split() if x]
    nccl = _nccl_dir()
    if nccl:
        f += ["-I", nccl[0], "-DLX_HAVE_NCCL=1"]
    return f


def _deps():
    return (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
            glob.glob(os.path.join(ROOT, "include", "*.h")))


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    hdr_mtime = max([os.path.getmtime(h) for h in _deps()] + [0])
    src_mtime = max([os.path.getmtime(x) for x in srcs] + [hdr_mtime, os.path.getmtime(__file__)])
    flags = _flags()
    # objects compiled with other flags (e.g. an NVCC_EXTRA variant build) are stale: rebuild everything
    stamp = os.path.join(BUILD, "flags.txt")
    key = " ".join(ARCH + flags)
    if os.path.exists(stamp) and open(stamp).read() != key:
        force = True
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= src_mtime:
        return LIB   # up to date (objects may be absent, e.g. on a gpurun box)
    objs = []
    cmds = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr_mtime):
            cmd = [NVCC] + ARCH + flags + ["-c", s, "-o", o]
            if s.endswith(".cu") and verbose:
                cmd += ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            cmds.append(cmd)
    # translation units compile in parallel (the Leja kernel files dominate the build time)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(subprocess.check_call, c) for c in cmds]:
            f.result()
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        link = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB + ".tmp"] + objs
        nccl = _nccl_dir()
        if nccl:
            link += ["-L", nccl[1], "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nccl[1]]
        if verbose:
            print(" ".join(link), file=sys.stderr)
        subprocess.check_call(link)
        os.replace(LIB + ".tmp", LIB)
    with open(stamp, "w") as fh:
        fh.write(key)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
