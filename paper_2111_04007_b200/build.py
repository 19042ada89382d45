"""Build libvpipe.so in-tree: every CUDA source for sm_100a + the C++ control
plane. Invoked by ``__graft_entry__.build()`` and by ``python
paper_2111_04007_b200/build.py`` (loaded by path: the package itself needs the
built library to import). Incremental by mtime (objects under
``paper_2111_04007_b200/_build/``)."""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
# VP_BUILD_TAG builds an alternative library (e.g. with VP_EXTRA_NVCC=-DVP_BWD_TRACE
# for the clock64 timelines) beside the product one; load it with VP_LIB_PATH
_TAG = os.environ.get("VP_BUILD_TAG", "")
OBJ = os.path.join(PKG, "_build" + (f"_{_TAG}" if _TAG else ""))
LIB = os.path.join(PKG, f"libvpipe{'_' + _TAG if _TAG else ''}.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{INC}", f"-I{CSRC}"]
CU_FLAGS = ARCH + COMMON + ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-v"] + \
    os.environ.get("VP_EXTRA_NVCC", "").split()


def _deps(src):
    heads = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    return [src, os.path.join(INC, "vpipe.h")] + heads


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src):
    base = os.path.splitext(os.path.basename(src))[0]
    obj = os.path.join(OBJ, base + ".o")
    if not _stale(obj, _deps(src)):
        return obj, None
    if src.endswith(".cu"):
        cmd = [NVCC] + CU_FLAGS + ["-c", src, "-o", obj]
    else:
        cmd = [NVCC] + COMMON + ["-x", "c++", "-c", src, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    log = os.path.join(OBJ, base + ".ptxas.log")
    with open(log, "w") as f:
        f.write(p.stdout + p.stderr)
    return obj, log


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, srcs))
    objs = [o for o, _ in results]
    if _stale(LIB, objs) or any(log for _, log in results):
        tmp = LIB + ".tmp"
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lpthread", "-ldl", "-lrt"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
        os.replace(tmp, LIB)
    if verbose:
        for _, log in results:
            if log:
                print(open(log).read())
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
