"""Build libevict.so (the C-ABI hot-path library) in-tree for sm_100a.

Each translation unit under csrc/ compiles in parallel with nvcc
(-gencode arch=compute_100a,code=sm_100a -lineinfo), then one link step makes
``paper_2605_00342_b200/libevict.so``.  Rebuilds only when a source is newer
than the library.
"""
from __future__ import annotations

import glob
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libevict.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
              f"-I{INCLUDE}", f"-I{CSRC}"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(
        os.path.join(CSRC, "*.h")) + [os.path.join(INCLUDE, "evict.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def _includes(path, seen=None):
    """Local headers a translation unit pulls in (transitively, quoted includes only)."""
    seen = set() if seen is None else seen
    with open(path) as f:
        for line in f:
            m = re.match(r'\s*#\s*include\s+"([^"]+)"', line)
            if not m:
                continue
            for d in (os.path.dirname(path), CSRC, INCLUDE):
                h = os.path.join(d, m.group(1))
                if os.path.exists(h) and h not in seen:
                    seen.add(h)
                    _includes(h, seen)
                    break
    return seen


def _obj(src):
    return os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))


def _obj_stale(src):
    obj = _obj(src)
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src, *_includes(src)])


def _compile(src):
    os.makedirs(OBJ, exist_ok=True)
    obj = _obj(src)
    if not FORCE[0] and not _obj_stale(src):
        return obj
    log = obj.replace(".o", ".ptxas.log")
    cmd = ["nvcc", *ARCH, *NVCC_FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    return obj


FORCE = [False]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    FORCE[0] = force
    srcs = sources()
    with ThreadPoolExecutor(max(1, min(len(srcs), os.cpu_count() or 4))) as ex:
        objs = list(ex.map(_compile, srcs))
    cmd = ["nvcc", *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-lcuda"]
    subprocess.check_call(cmd)
    if verbose:
        print(f"built {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
