"""Build libmdhp.so (sm_100a) in-tree with nvcc.  No JIT cache: the .so travels with the repo."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libmdhp.so")
LIB_DEBUG = os.path.join(LIBDIR, "libmdhp_debug.so")   # -DMDHP_DEBUG: device bounds asserts
SOURCES = ["abi.cu", "pack.cu", "fit.cu", "exact.cu", "seq.cu", "dense.cu", "features.cu"]
HEADERS = ["common.cuh", "eval.cuh"]
CC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC"]
LINK_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xlinker", "--no-undefined"]


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(os.path.dirname(HERE), "include", "mdhp.h")]
    os.makedirs(LIBDIR, exist_ok=True)
    out = LIB_DEBUG if debug else LIB
    if force or _stale(out, deps):
        # one object per source, compiled in parallel, then one link
        from concurrent.futures import ThreadPoolExecutor
        objdir = os.path.join(LIBDIR, "obj")
        os.makedirs(objdir, exist_ok=True)
        tag = ".dbg" if debug else ""
        objs = [os.path.join(objdir, os.path.basename(s)[:-3] + tag + ".o") for s in srcs]

        def cc(src, obj):
            cmd = ["nvcc", *CC_FLAGS, *(["-DMDHP_DEBUG"] if debug else []),
                   *(["-Xptxas=-v"] if verbose else []), "-c", "-o", obj, src]
            return cmd, subprocess.run(cmd, capture_output=True, text=True)

        with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 1)) as ex:
            for cmd, r in ex.map(lambda a: cc(*a), zip(srcs, objs)):
                if r.returncode != 0:
                    raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
                if verbose:
                    print(r.stderr)
        cmd = ["nvcc", *LINK_FLAGS, "-o", out, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=False))
