"""Seeded synthetic workload generator shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic (see ``evict_gen.h`` for the recipe and
DESIGN.md §4).  Host entry points return numpy arrays (inputs of oracle parity
tests); ``*_cuda`` entry points fill torch CUDA tensors (bench inputs).  The
two builds are bit-identical by construction (integer ops and correctly
rounded fp64 ops only), checked by tests/test_gen.py on the GPU.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_HDR = os.path.join(_HERE, "evict_gen.h")
_HOST_SRC = os.path.join(_HERE, "gen_host.c")
_HOST_LIB = os.path.join(_HERE, "libevictgen_host.so")
_CUDA_SRC = os.path.join(_HERE, "gen_cuda.cu")
_CUDA_LIB = os.path.join(_HERE, "libevictgen_cuda.so")
NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

_lock = threading.Lock()
_host = None
_cuda = None

# BASELINE.json configs; tree shapes and model shapes
CONFIGS = {
    "toy": dict(B=1, N=8, L=2, E=8, K=2, d=64),
    "c2": dict(B=1, N=60, steps=6, topk=10, L=48, E=128, K=8, d=2048, seed=2),
    "c3": dict(B=16, N=60, steps=6, topk=10, L=94, E=128, K=8, d=4096, seed=3),
    "c4": dict(B=64, N=128, steps=8, topk=10, L=48, E=128, K=8, d=2048, seed=4),
    "c4_60": dict(B=64, N=60, steps=6, topk=10, L=48, E=128, K=8, d=2048, seed=4),
    "c5": dict(B=1_000_000, N=60, steps=6, topk=10, L=48, E=128, K=8, d=2048, seed=5),
    "paper": dict(B=1, N=32, steps=4, topk=8, L=48, E=128, K=8, d=2048, seed=7),
    # Ling-flash-2.0 (256 experts, top-8; 32 MoE layers, hidden 4096) — NEXT-4 shape
    "ling": dict(B=1, N=60, steps=6, topk=10, L=32, E=256, K=8, d=4096, seed=6),
}
M_LO, M_HI = 1, 16          # per-tree difficulty exponent range (evict_gen.h)
SIGMA_Q4 = 9                # round(4 * sigma_b), sigma_b = 2.25

# The hand-written toy tree (dyadic values, BASELINE config 0)
TOY_PARENT = np.array([-1, 0, 0, 1, 1, 2, 3, 4], np.int32)
TOY_Q = np.array([1, .75, .125, .5, .25, .5, .5, .5], np.float32)
TOY_COST = np.array([1.0, 1.25, 1.5, 1.75, 2.0, 2.25, 2.5, 2.75], np.float32)
TOY_ROUTING = np.array([
    [[0, 1], [4, 5]], [[0, 2], [4, 6]], [[5, 6], [0, 1]], [[1, 2], [5, 6]],
    [[3, 0], [7, 4]], [[7, 6], [2, 3]], [[2, 4], [6, 5]], [[1, 3], [0, 7]],
], np.uint8)  # [node][layer][K]


def _build_host(force=False):
    if force or not os.path.exists(_HOST_LIB) or os.path.getmtime(_HOST_LIB) < max(
            os.path.getmtime(_HOST_SRC), os.path.getmtime(_HDR)):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-shared", "-fPIC", "-o", _HOST_LIB, _HOST_SRC])
    return _HOST_LIB


def _build_cuda(force=False):
    if force or not os.path.exists(_CUDA_LIB) or os.path.getmtime(_CUDA_LIB) < max(
            os.path.getmtime(_CUDA_SRC), os.path.getmtime(_HDR)):
        subprocess.check_call(["nvcc", *NVCC_ARCH, "-O3", "-lineinfo", "-fmad=false",
                               "-Xcompiler", "-fPIC", "-shared", "-o", _CUDA_LIB, _CUDA_SRC])
    return _CUDA_LIB


def build(force=False):
    _build_host(force)
    _build_cuda(force)


def host_lib():
    global _host
    with _lock:
        if _host is None:
            _build_host()
            L = ctypes.CDLL(_HOST_LIB)
            u64, i = ctypes.c_uint64, ctypes.c_int
            vp = ctypes.c_void_p
            L.gen_trees_host.argtypes = [u64, u64, i, i, i, i, i, i, vp, vp, vp]
            L.gen_routing_host.argtypes = [u64, u64, i, i, i, i, i, i, i, vp]
            L.gen_hidden_host.argtypes = [u64, u64, i, i, i, i, i, vp]
            L.gen_wgate_host.argtypes = [u64, i, i, i, i, i, vp]
            _host = L
    return _host


def cuda_lib():
    global _cuda
    with _lock:
        if _cuda is None:
            _build_cuda()
            L = ctypes.CDLL(_CUDA_LIB)
            u64, i = ctypes.c_uint64, ctypes.c_int
            vp = ctypes.c_void_p
            L.gen_tree_scratch_bytes.restype = ctypes.c_size_t
            L.gen_trees_cuda.argtypes = [u64, u64, i, i, i, i, i, i, vp, vp, vp, vp, i, vp]
            L.gen_routing_cuda.argtypes = [u64, u64, i, i, i, i, i, i, i, vp, vp]
            L.gen_hidden_cuda.argtypes = [u64, u64, i, i, i, i, i, vp, vp]
            L.gen_wgate_cuda.argtypes = [u64, i, i, i, i, i, vp, vp]
            L.gen_ids_to_mask_cuda.argtypes = [vp, ctypes.c_size_t, i, i, vp, vp]
            L.gen_ids_to_mask_cuda.restype = ctypes.c_int
            for f in ("gen_trees_cuda", "gen_routing_cuda", "gen_hidden_cuda", "gen_wgate_cuda"):
                getattr(L, f).restype = ctypes.c_int
            _cuda = L
    return _cuda


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


GEN_MAX_TOPK, GEN_MAX_POOL = 16, 1024   # evict_gen.h


def check_tree_shape(steps, topk):
    """The generator's candidate pool (topk + (steps − 1)·topk² candidates) lives in fixed scratch
    arrays (evict_gen.h GEN_MAX_POOL): reject shapes that would overflow them."""
    if not (1 <= topk <= GEN_MAX_TOPK) or steps < 1 or topk + (steps - 1) * topk * topk > GEN_MAX_POOL:
        raise ValueError(f"draft-tree shape steps={steps} topk={topk} exceeds the generator's pool "
                         f"({GEN_MAX_POOL} candidates, topk <= {GEN_MAX_TOPK})")


def _fan(fn, B, threads):
    threads = max(1, min(threads, B))
    step = (B + threads - 1) // threads
    rs = [(s, min(B, s + step)) for s in range(0, B, step)]
    if len(rs) == 1:
        fn(*rs[0])
    else:
        with ThreadPoolExecutor(len(rs)) as ex:
            list(ex.map(lambda r: fn(*r), rs))


# ---------------------------------------------------------------- host side
def trees(seed, B, N, steps, topk, tree_base=0, m_lo=M_LO, m_hi=M_HI, threads=8):
    """EAGLE-style draft trees: (parent int32 [B][N], q float32 [B][N], n_nodes int32 [B])."""
    check_tree_shape(steps, topk)
    parent = np.empty((B, N), np.int32)
    q = np.empty((B, N), np.float32)
    n = np.empty(B, np.int32)
    L = host_lib()

    def run(lo, hi):
        L.gen_trees_host(seed, tree_base + lo, hi - lo, steps, topk, N, m_lo, m_hi,
                         _p(parent[lo:hi]), _p(q[lo:hi]), _p(n[lo:hi]))

    _fan(run, B, threads)
    return parent, q, n


def routing(seed, B, N, L, E, K, tree_base=0, sigma_q4=SIGMA_Q4, dtype=np.uint8, threads=8):
    """Routing top-K ids [B][N][L][K] (uint8 or int32)."""
    dtype = np.dtype(dtype)
    out = np.empty((B, N, L, K), dtype)
    lib = host_lib()

    def run(lo, hi):
        lib.gen_routing_host(seed, tree_base + lo, hi - lo, N, L, E, K, sigma_q4, dtype.itemsize,
                             _p(out[lo:hi]))

    _fan(run, B, threads)
    return out


def hidden(seed, B, N, L, d, mode=0, tree_base=0):
    """Per-layer hidden states, bf16 bits [L][B*N][d] (uint16)."""
    out = np.empty((L, B * N, d), np.uint16)
    host_lib().gen_hidden_host(seed, tree_base, B, N, L, d, mode, _p(out))
    return out


def wgate(seed, L, E, d, mode=0, scale_log2=0):
    """Router weights W_g, bf16 bits [L][E][d] (uint16)."""
    out = np.empty((L, E, d), np.uint16)
    host_lib().gen_wgate_host(seed, L, E, d, mode, scale_log2, _p(out))
    return out


def ids_to_mask(ids, E):
    """One-hot routing masks [B][N][L][ceil(E/64)] uint64 from ids (input re-encoding)."""
    EW = (E + 63) // 64
    B, N, L, K = ids.shape
    m = np.zeros((B, N, L, EW), np.uint64)
    idx = ids.astype(np.int64)
    for j in range(K):
        e = idx[..., j]
        for w in range(EW):
            sel = (e // 64) == w
            m[..., w] |= np.where(sel, np.left_shift(np.uint64(1), (e % 64).astype(np.uint64)),
                                  np.uint64(0))
    return m


def cost_table(N, E=128, K=8, c0=10.47, c_union=0.0915, c_tok=0.15):
    """Default profiled-cost stand-in C(k), k=1..N (ms):
    C(k) = c0 + c_union * U(k) + c_tok * k with U(k) = E (1 - (1 - K/E)^k)."""
    k = np.arange(1, N + 1, dtype=np.float64)
    U = E * (1.0 - (1.0 - K / E) ** k)
    return (c0 + c_union * U + c_tok * k).astype(np.float32)


# ---------------------------------------------------------------- device side
def _tp(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def trees_cuda(seed, B, N, steps, topk, tree_base=0, m_lo=M_LO, m_hi=M_HI, device="cuda"):
    import torch
    check_tree_shape(steps, topk)
    L = cuda_lib()
    parent = torch.empty((B, N), dtype=torch.int32, device=device)
    q = torch.empty((B, N), dtype=torch.float32, device=device)
    n = torch.empty(B, dtype=torch.int32, device=device)
    nscratch = min(B, 148 * 512)
    scratch = torch.empty(nscratch * L.gen_tree_scratch_bytes(), dtype=torch.uint8, device=device)
    rc = L.gen_trees_cuda(seed, tree_base, B, steps, topk, N, m_lo, m_hi, _tp(parent), _tp(q),
                          _tp(n), _tp(scratch), nscratch, _stream())
    assert rc == 0, rc
    torch.cuda.current_stream().synchronize()
    del scratch
    return parent, q, n


def routing_cuda(seed, B, N, L, E, K, tree_base=0, sigma_q4=SIGMA_Q4, dtype="uint8",
                 device="cuda", out=None):
    import torch
    tdt = torch.uint8 if dtype == "uint8" else torch.int32
    if out is None:
        out = torch.empty((B, N, L, K), dtype=tdt, device=device)
    rc = cuda_lib().gen_routing_cuda(seed, tree_base, B, N, L, E, K, sigma_q4,
                                     1 if tdt == torch.uint8 else 4, _tp(out), _stream())
    assert rc == 0, rc
    return out


def hidden_cuda(seed, B, N, L, d, mode=0, tree_base=0, device="cuda"):
    import torch
    out = torch.empty((L, B * N, d), dtype=torch.bfloat16, device=device)
    rc = cuda_lib().gen_hidden_cuda(seed, tree_base, B, N, L, d, mode, _tp(out), _stream())
    assert rc == 0, rc
    return out


def wgate_cuda(seed, L, E, d, mode=0, scale_log2=0, device="cuda"):
    import torch
    out = torch.empty((L, E, d), dtype=torch.bfloat16, device=device)
    rc = cuda_lib().gen_wgate_cuda(seed, L, E, d, mode, scale_log2, _tp(out), _stream())
    assert rc == 0, rc
    return out


def ids_to_mask_cuda(ids, E):
    """Device re-encoding of uint8 ids [B][N][L][K] into one-hot masks [B][N][L][EW] (int64)."""
    import torch
    B, N, L, K = ids.shape
    EW = (E + 63) // 64
    out = torch.empty((B, N, L, EW), dtype=torch.int64, device=ids.device)
    rc = cuda_lib().gen_ids_to_mask_cuda(_tp(ids), B * N * L, K, EW, _tp(out), _stream())
    assert rc == 0, rc
    return out
