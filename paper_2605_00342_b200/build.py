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


VARIANT = [None, []]   # (name, extra -D flags): kernel A/B builds into build_<name>/, libevict_<name>.so


def _objdir():
    return OBJ if VARIANT[0] is None else OBJ + "_" + VARIANT[0]


def _lib():
    return LIB if VARIANT[0] is None else LIB.replace("libevict.so", f"libevict_{VARIANT[0]}.so")


def _obj(src):
    return os.path.join(_objdir(), os.path.basename(src).replace(".cu", ".o"))


def _obj_stale(src):
    obj = _obj(src)
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src, *_includes(src)])


def _compile(src):
    os.makedirs(_objdir(), exist_ok=True)
    obj = _obj(src)
    if not FORCE[0] and not _obj_stale(src):
        return obj
    log = obj.replace(".o", ".ptxas.log")
    cmd = ["nvcc", *ARCH, *NVCC_FLAGS, *VARIANT[1], "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    return obj


FORCE = [False]


def build(force: bool = False, verbose: bool = False) -> str:
    if VARIANT[0] is None and not force and not stale():
        return LIB
    FORCE[0] = force
    srcs = sources()
    with ThreadPoolExecutor(max(1, min(len(srcs), os.cpu_count() or 4))) as ex:
        objs = list(ex.map(_compile, srcs))
    cmd = ["nvcc", *ARCH, "-shared", "-o", _lib(), *objs, "-lcudart", "-lcuda"]
    subprocess.check_call(cmd)
    if verbose:
        print(f"built {_lib()}", file=sys.stderr)
    return _lib()


if __name__ == "__main__":
    if "--variant" in sys.argv:
        VARIANT[0] = sys.argv[sys.argv.index("--variant") + 1]
        VARIANT[1] = [a for a in sys.argv if a.startswith("-D")]
    build(force="--force" in sys.argv, verbose=True)
