"""The C-ABI library loads and exports every symbol include/evict.h declares (CPU only)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "evict.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(evict_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    fns = declared_functions()
    for f in ("evict_select", "evict_build_verify_tree", "evict_expert_union",
              "evict_router_union", "evict_select_build_union", "evict_batch_stats"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    import paper_2605_00342_b200 as ev
    from paper_2605_00342_b200 import build
    build.build()
    lib = ctypes.CDLL(ev.LIB_PATH)
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    assert lib.evict_abi_version() == 8
    lib.evict_workspace_bytes.restype = ctypes.c_size_t
    assert lib.evict_workspace_bytes(64) == 8 * (1 + 64)   # serving batches: one state word per tree
    assert lib.evict_workspace_bytes(4096) == 8 * (1 + 1024)   # above 2048: one per 4-tree warp tile


def test_library_targets_sm100a_only():
    import subprocess
    from paper_2605_00342_b200 import build
    lib = build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2605_00342_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower() or f == "__init__.py" and \
                    "import oracle" not in txt, f
