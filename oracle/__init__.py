"""CPU oracle for the EVICT hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The
product path (``paper_2605_00342_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``evict_oracle.c`` (plain C, one tree at a
time, following PAPER.md step by step); this module only marshals numpy
arrays through ctypes and fans trees out over host threads.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "evict_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

TREE_BAD_SIZE = 0x01
TREE_BAD_PARENT = 0x02
TREE_BAD_PROB = 0x04
TREE_BAD_COST = 0x08
TREE_BAD_EXPERT = 0x10
TREE_BAD_KEEP = 0x20
TIE_REL = 1e-5


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
               "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _P(t):
    return ctypes.POINTER(t)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            i32, u32, f32, f64, u64, i64, u16 = (ctypes.c_int32, ctypes.c_uint32, ctypes.c_float,
                                                ctypes.c_double, ctypes.c_uint64, ctypes.c_int64,
                                                ctypes.c_uint16)
            vp = ctypes.c_void_p
            L.oracle_select_batch.argtypes = [ctypes.c_int] * 3 + [vp] * 4 + [ctypes.c_int] + [vp] * 11
            L.oracle_select_batch.restype = None
            L.oracle_select_batch_policy.argtypes = ([ctypes.c_int] * 3 + [vp] * 4 + [ctypes.c_int] * 2 +
                                                     [ctypes.c_double, ctypes.c_int] + [vp] * 11)
            L.oracle_select_batch_policy.restype = None
            L.oracle_union_curve_batch.argtypes = ([ctypes.c_int] * 3 + [vp] * 3 + [ctypes.c_int] * 4 +
                                                   [vp] * 3)
            L.oracle_union_curve_batch.restype = None
            L.oracle_profile_cost.argtypes = ([ctypes.c_int] * 3 + [vp] * 3 + [ctypes.c_double] * 3 + [vp])
            L.oracle_profile_cost.restype = None
            L.oracle_build_batch.argtypes = [ctypes.c_int] * 2 + [vp] * 11
            L.oracle_build_batch.restype = None
            L.oracle_union_batch.argtypes = [ctypes.c_int] * 3 + [vp] * 3 + [ctypes.c_int] * 4 + [vp] * 4
            L.oracle_union_batch.restype = None
            L.oracle_router_topk.argtypes = [ctypes.c_int, vp, vp, ctypes.c_int, ctypes.c_int, vp, vp]
            L.oracle_router_topk.restype = ctypes.c_int
            L.oracle_router_union_batch.argtypes = [ctypes.c_int] * 4 + [vp] * 2 + [ctypes.c_int] * 4 + [vp] * 6
            L.oracle_router_union_batch.restype = None
            L.oracle_batch_stats.argtypes = [ctypes.c_int] * 3 + [vp] * 8
            L.oracle_batch_stats.restype = None
            _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


def _ranges(B, threads):
    threads = max(1, min(threads, B))
    step = (B + threads - 1) // threads
    return [(s, min(B, s + step)) for s in range(0, B, step)]


POLICIES = {"cost": 0, "coverage": 1, "fixed": 2}


def select(parent, q, cost, n_nodes=None, cost_stride=0, threads=1, policy=None):
    """A1–A5 for a [B][N] batch.  Returns a dict of numpy arrays.
    policy: None / ("cost",) — Eq. 10; ("coverage", rho) — smallest k with S_k/S_K ≥ rho
    (PAPER.md:290-291); ("fixed", k) — k* = min(k, n_b)."""
    kind, rho, kfix = 0, 0.0, 0
    if policy is not None:
        kind = POLICIES[policy[0]]
        if kind == 1:
            rho = float(np.float32(policy[1]))   # the GPU receives ρ as fp32
        elif kind == 2:
            kfix = int(policy[1])
    parent = _c(parent, np.int32)
    q = _c(q, np.float32)
    cost = _c(cost, np.float32)
    B, N = parent.shape
    W = (N + 63) // 64
    n_nodes = _c(n_nodes, np.int32)
    out = dict(score=np.zeros((B, N), np.float32), depth=np.zeros((B, N), np.int32),
               order=np.zeros((B, N), np.int32), S=np.zeros((B, N), np.float64),
               R=np.zeros((B, N), np.float64), k_star=np.zeros(B, np.int32),
               e_hat=np.zeros(B, np.float64), utility=np.zeros(B, np.float64),
               keep_bits=np.zeros((B, W), np.uint64), tie_bits=np.zeros((B, W), np.uint64),
               status=np.zeros(B, np.uint32))
    L = lib()

    def run(r):
        L.oracle_select_batch_policy(r[0], r[1], N, _ptr(n_nodes), _ptr(parent), _ptr(q), _ptr(cost),
                              cost_stride, kind, rho, kfix,
                              _ptr(out["score"]), _ptr(out["depth"]),
                              _ptr(out["order"]), _ptr(out["S"]), _ptr(out["R"]),
                              _ptr(out["k_star"]), _ptr(out["e_hat"]), _ptr(out["utility"]),
                              _ptr(out["keep_bits"]), _ptr(out["tie_bits"]), _ptr(out["status"]))

    _fan(run, B, threads)
    return out


def _fan(fn, B, threads):
    rs = _ranges(B, threads)
    if len(rs) == 1:
        fn(rs[0])
    else:
        with ThreadPoolExecutor(len(rs)) as ex:
            list(ex.map(fn, rs))


def build_verify_tree(parent, keep_bits, n_nodes=None, pos_offset=None):
    """A6 (packed verify layout).  Returns a dict of numpy arrays."""
    parent = _c(parent, np.int32)
    keep_bits = _c(keep_bits, np.uint64)
    B, N = parent.shape
    W = (N + 63) // 64
    cap = B * N
    out = dict(verify_offsets=np.zeros(B + 1, np.int32), kept_index=np.full(cap, -1, np.int32),
               retrieve_index=np.full(cap, -1, np.int32), positions=np.full(cap, -1, np.int32),
               next_token=np.full(cap, -1, np.int32), next_sibling=np.full(cap, -1, np.int32),
               tree_mask=np.zeros((cap, W), np.uint64), status=np.zeros(B, np.uint32))
    lib().oracle_build_batch(B, N, _ptr(_c(n_nodes, np.int32)), _ptr(parent), _ptr(keep_bits),
                             _ptr(_c(pos_offset, np.int32)), _ptr(out["verify_offsets"]),
                             _ptr(out["kept_index"]), _ptr(out["retrieve_index"]),
                             _ptr(out["positions"]), _ptr(out["next_token"]),
                             _ptr(out["next_sibling"]), _ptr(out["tree_mask"]), _ptr(out["status"]))
    return out


def expert_union(keep_bits, ids, num_experts, n_nodes=None, threads=1):
    """A7: ids is [B][N][L][K] uint8 or int32."""
    keep_bits = _c(keep_bits, np.uint64)
    ids = np.ascontiguousarray(ids)
    assert ids.dtype in (np.uint8, np.int32)
    B, N, Lyr, K = ids.shape
    E = num_experts
    EW = (E + 63) // 64
    out = dict(union_count=np.zeros((B, Lyr), np.int32), union_total=np.zeros(B, np.int32),
               union_bits=np.zeros((B, Lyr, EW), np.uint64), status=np.zeros(B, np.uint32))
    n_nodes = _c(n_nodes, np.int32)
    L = lib()

    def run(r):
        L.oracle_union_batch(r[0], r[1], N, _ptr(n_nodes), _ptr(keep_bits), _ptr(ids),
                             ids.dtype.itemsize, Lyr, K, E, _ptr(out["union_count"]),
                             _ptr(out["union_total"]), _ptr(out["union_bits"]), _ptr(out["status"]))

    _fan(run, B, threads)
    return out


def union_curve(order, ids, num_experts, n_nodes=None, threads=1, per_layer=True):
    """NEXT-1: prefix-union curve along the ranking.  order [B][N] (evict_select's order row),
    ids [B][N][L][K] uint8/int32.  Returns curve [B][N], curve_layer [B][N][L], status."""
    order = _c(order, np.int32)
    ids = np.ascontiguousarray(ids)
    assert ids.dtype in (np.uint8, np.int32)
    B, N, Lyr, K = ids.shape
    out = dict(curve=np.zeros((B, N), np.int32), status=np.zeros(B, np.uint32))
    if per_layer:
        out["curve_layer"] = np.zeros((B, N, Lyr), np.int32)
    n_nodes = _c(n_nodes, np.int32)
    L = lib()

    def run(r):
        L.oracle_union_curve_batch(r[0], r[1], N, _ptr(n_nodes), _ptr(order), _ptr(ids),
                                   ids.dtype.itemsize, Lyr, K, num_experts, _ptr(out["curve"]),
                                   _ptr(out.get("curve_layer")), _ptr(out["status"]))

    _fan(run, B, threads)
    return out


def profile_cost(curve, num_layers, n_nodes=None, status=None, c0=10.47, c_union=0.0915, c_tok=0.15):
    """Offline C(k) from measured curves (fp64): Ū(k) = mean curve(k)/L over trees with n_b ≥ k."""
    curve = _c(curve, np.int32)
    B, N = curve.shape
    n_nodes = _c(n_nodes, np.int32)
    status = _c(status, np.uint32)
    cost = np.zeros(N, np.float64)
    lib().oracle_profile_cost(B, N, num_layers, _ptr(n_nodes), _ptr(curve), _ptr(status), c0, c_union,
                              c_tok, _ptr(cost))
    return cost


def router_topk(h_bits, wg_bits, K):
    """Eq. 4 top-K of one hidden row (bf16 bits [d]) against Wg bits [E][d]."""
    h_bits = _c(h_bits, np.uint16)
    wg_bits = _c(wg_bits, np.uint16)
    E, d = wg_bits.shape
    ids = np.zeros(K, np.int32)
    logits = np.zeros(E, np.float64)
    nt = lib().oracle_router_topk(d, _ptr(h_bits), _ptr(wg_bits), E, K, _ptr(ids), _ptr(logits))
    return ids, logits, bool(nt)


def router_union(keep_bits, h_bits, wg_bits, K, n_nodes=None, threads=1):
    """A8 → A7: h_bits [L][B*N][d] bf16 bits, wg_bits [L][E][d] bf16 bits."""
    keep_bits = _c(keep_bits, np.uint64)
    h_bits = _c(h_bits, np.uint16)
    wg_bits = _c(wg_bits, np.uint16)
    B, W = keep_bits.shape
    Lyr, BN, d = h_bits.shape
    N = BN // B
    E = wg_bits.shape[1]
    EW = (E + 63) // 64
    out = dict(union_count=np.zeros((B, Lyr), np.int32), union_total=np.zeros(B, np.int32),
               union_bits=np.zeros((B, Lyr, EW), np.uint64), near_tie=np.zeros((B, Lyr), np.int32))
    n_nodes = _c(n_nodes, np.int32)
    L = lib()

    def run(r):
        L.oracle_router_union_batch(r[0], r[1], B, N, _ptr(n_nodes), _ptr(keep_bits), Lyr, E, K, d,
                                    _ptr(h_bits), _ptr(wg_bits), _ptr(out["union_count"]),
                                    _ptr(out["union_total"]), _ptr(out["union_bits"]),
                                    _ptr(out["near_tie"]))

    _fan(run, B, threads)
    return out


def batch_stats(N, num_layers, k_star, e_hat, utility, union_count, status, n_nodes=None):
    """A9 stats vector (layout documented in evict_oracle.c)."""
    B = len(k_star)
    stats = np.zeros(6 + N + num_layers, np.int64)
    dstats = np.zeros(2, np.float64)
    lib().oracle_batch_stats(B, N, num_layers, _ptr(_c(n_nodes, np.int32)), _ptr(_c(k_star, np.int32)),
                             _ptr(_c(e_hat, np.float64)), _ptr(_c(utility, np.float64)),
                             _ptr(_c(union_count, np.int32)), _ptr(_c(status, np.uint32)),
                             _ptr(stats), _ptr(dstats))
    return stats, dstats
