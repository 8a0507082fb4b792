"""B200-native EVICT hot path (arxiv 2605.00342): thin Python binding over libevict.so.

Argument marshalling only — every step of the path runs in the CUDA kernels
behind the C ABI declared in ``include/evict.h``.  Tensors are torch CUDA
tensors (torch supplies device memory and streams); results come back as
torch CUDA tensors.  There is no CPU fallback: if ``libevict.so`` is missing or
the device is not sm_100 the calls raise.

Functions mirror the C ABI names:
  evict_select, evict_build_verify_tree, evict_expert_union,
  evict_select_build_union, evict_router_union, evict_batch_stats.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libevict.so")
# kernel A/B experiments only: EVICT_LIB_VARIANT=x loads libevict_x.so (built by
# `python -m paper_2605_00342_b200.build --variant x -D...`); the product build is libevict.so
if os.environ.get("EVICT_LIB_VARIANT"):
    LIB_PATH = os.path.join(PKG, f"libevict_{os.environ['EVICT_LIB_VARIANT']}.so")

EVICT_OK, EVICT_ERR_INVALID_ARG, EVICT_ERR_UNSUPPORTED, EVICT_ERR_CUDA = 0, 1, 2, 3
TREE_BAD_SIZE, TREE_BAD_PARENT, TREE_BAD_PROB = 0x01, 0x02, 0x04
TREE_BAD_COST, TREE_BAD_EXPERT, TREE_BAD_KEEP = 0x08, 0x10, 0x20
ID_U8, ID_I32, ID_MASK = 1, 4, 8
MAX_NODES = 128


class EvictError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: status {code} ({_status_string(code)})")
        self.code = code


class _Trees(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("max_nodes", ctypes.c_int32),
                ("n_nodes", ctypes.c_void_p), ("parent", ctypes.c_void_p), ("q", ctypes.c_void_p)]


class _Routing(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("num_experts", ctypes.c_int32),
                ("top_k", ctypes.c_int32), ("id_format", ctypes.c_int32), ("ids", ctypes.c_void_p)]


class _Policy(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("rho", ctypes.c_float), ("k_fixed", ctypes.c_int32)]


POLICY_KINDS = {"cost": 0, "coverage": 1, "fixed": 2}


def _policy(policy):
    """None / ("cost",) → NULL (Eq. 10); ("coverage", rho); ("fixed", k)."""
    if policy is None or policy[0] == "cost":
        return None
    kind = POLICY_KINDS[policy[0]]
    return _Policy(kind, float(policy[1]) if kind == 1 else 0.0, int(policy[1]) if kind == 2 else 0)


def _pp(pol):
    return ctypes.byref(pol) if pol is not None else None


class _Router(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("num_experts", ctypes.c_int32),
                ("top_k", ctypes.c_int32), ("hidden_dim", ctypes.c_int32),
                ("hidden", ctypes.c_void_p), ("w_gate", ctypes.c_void_p), ("max_rows", ctypes.c_int32)]


_OUT_FIELDS = ["k_star", "e_hat", "utility", "keep_bits", "order", "prefix_sums", "pos_offset",
               "verify_offsets", "kept_index", "retrieve_index", "positions", "next_token",
               "next_sibling", "tree_mask", "union_count", "union_total", "union_bits",
               "expert_hist", "status", "stats", "dstats"]


class _FusedOut(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in _OUT_FIELDS]


_lock = threading.Lock()
_lib = None


def lib():
    """Load libevict.so (raises if it was not built — there is no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(LIB_PATH)
            vp, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
            L.evict_select.argtypes = [vp, vp, i32] + [vp] * 8
            L.evict_build_verify_tree.argtypes = [vp] * 12 + [sz, vp]
            L.evict_expert_union.argtypes = [vp] * 9
            L.evict_select_build_union.argtypes = [vp, vp, i32, vp, vp, vp, sz, vp]
            L.evict_select_policy.argtypes = [vp, vp, i32, vp] + [vp] * 8
            L.evict_union_curve.argtypes = [vp] * 7
            L.evict_profile_workspace_bytes.argtypes = [i32]
            L.evict_profile_workspace_bytes.restype = sz
            L.evict_profile_cost.argtypes = ([i32] * 3 + [vp] * 3 + [ctypes.c_float] * 3 + [vp, vp, sz, vp])
            L.evict_select_build_union_policy.argtypes = [vp, vp, i32, vp, vp, vp, vp, sz, vp]
            L.evict_router_union.argtypes = [vp] * 9
            L.evict_verify_sample.argtypes = [vp, vp, i32, ctypes.c_int64, i32] + [vp] * 7
            L.evict_dispatch_create.argtypes = [i32, vp, vp, vp, vp, vp, vp]
            L.evict_build_draft_tree.argtypes = [i32] * 4 + [vp] * 7
            L.evict_dispatch_launch.argtypes = [vp, vp]
            L.evict_dispatch_destroy.argtypes = [vp]
            L.evict_dispatch_destroy.restype = None
            L.evict_batch_stats.argtypes = [i32, i32, i32] + [vp] * 9
            L.evict_workspace_bytes.argtypes = [i32]
            L.evict_workspace_bytes.restype = sz
            L.evict_status_string.argtypes = [ctypes.c_int]
            L.evict_status_string.restype = ctypes.c_char_p
            for f in ("evict_select", "evict_build_verify_tree", "evict_expert_union",
                      "evict_select_build_union", "evict_router_union", "evict_batch_stats",
                      "evict_select_policy", "evict_select_build_union_policy", "evict_union_curve",
                      "evict_profile_cost", "evict_verify_sample", "evict_dispatch_create",
                      "evict_dispatch_launch", "evict_build_draft_tree"):
                getattr(L, f).restype = ctypes.c_int
            _lib = L
    return _lib


def _status_string(code):
    try:
        return lib().evict_status_string(code).decode()
    except Exception:  # pragma: no cover
        return "?"


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _check(rc, what):
    if rc != EVICT_OK:
        raise EvictError(rc, what)


def _trees(parent, q, n_nodes):
    assert parent.is_cuda and parent.dtype == torch.int32 and parent.is_contiguous()
    assert q.is_cuda and q.dtype == torch.float32 and q.is_contiguous() and q.shape == parent.shape
    if n_nodes is not None:
        assert n_nodes.dtype == torch.int32 and n_nodes.is_contiguous()
    B, N = parent.shape
    return _Trees(B, N, _p(n_nodes), _p(parent), _p(q))


def _dev(t):
    return t.device


def workspace_bytes(batch):
    return int(lib().evict_workspace_bytes(batch))


def new_workspace(batch, device):
    return torch.empty(workspace_bytes(batch) // 8, dtype=torch.int64, device=device)


# ----------------------------------------------------------------- select (A1–A5)
def evict_select(parent, q, cost, n_nodes=None, cost_stride=0, with_order=False, policy=None,
                 stream=None):
    B, N = parent.shape
    dev = _dev(parent)
    W = (N + 63) // 64
    out = dict(k_star=torch.empty(B, dtype=torch.int32, device=dev),
               e_hat=torch.empty(B, dtype=torch.float32, device=dev),
               utility=torch.empty(B, dtype=torch.float32, device=dev),
               keep_bits=torch.empty((B, W), dtype=torch.int64, device=dev),
               status=torch.empty(B, dtype=torch.int32, device=dev))
    if with_order:
        out["order"] = torch.empty((B, N), dtype=torch.int32, device=dev)
        out["prefix_sums"] = torch.empty((B, N), dtype=torch.float32, device=dev)
    tr = _trees(parent, q, n_nodes)
    pol = _policy(policy)
    rc = lib().evict_select_policy(ctypes.byref(tr), _p(cost), cost_stride, _pp(pol), _p(out["k_star"]),
                                   _p(out["e_hat"]), _p(out["utility"]), _p(out["keep_bits"]),
                                   _p(out.get("order")), _p(out.get("prefix_sums")), _p(out["status"]),
                                   _stream(stream))
    _check(rc, "evict_select_policy")
    return out


# ----------------------------------------------------------------- build (A6)
def evict_build_verify_tree(parent, keep_bits, n_nodes=None, pos_offset=None, q=None,
                            workspace=None, stream=None):
    B, N = parent.shape
    dev = _dev(parent)
    W = (N + 63) // 64
    cap = B * N
    if q is None:
        q = torch.zeros_like(parent, dtype=torch.float32)
    out = dict(verify_offsets=torch.empty(B + 1, dtype=torch.int32, device=dev),
               kept_index=torch.full((cap,), -1, dtype=torch.int32, device=dev),
               retrieve_index=torch.full((cap,), -1, dtype=torch.int32, device=dev),
               positions=torch.full((cap,), -1, dtype=torch.int32, device=dev),
               next_token=torch.full((cap,), -1, dtype=torch.int32, device=dev),
               next_sibling=torch.full((cap,), -1, dtype=torch.int32, device=dev),
               tree_mask=torch.zeros((cap, W), dtype=torch.int64, device=dev),
               status=torch.empty(B, dtype=torch.int32, device=dev))
    if workspace is None:
        workspace = new_workspace(B, dev)
    tr = _trees(parent, q, n_nodes)
    rc = lib().evict_build_verify_tree(
        ctypes.byref(tr), _p(keep_bits), _p(pos_offset), _p(out["verify_offsets"]),
        _p(out["kept_index"]), _p(out["retrieve_index"]), _p(out["positions"]),
        _p(out["next_token"]), _p(out["next_sibling"]), _p(out["tree_mask"]), _p(out["status"]),
        _p(workspace), workspace.numel() * 8, _stream(stream))
    _check(rc, "evict_build_verify_tree")
    return out


# ----------------------------------------------------------------- union (A7)
def _routing(ids, num_experts, id_format=None):
    if id_format is None:
        id_format = {torch.uint8: ID_U8, torch.int32: ID_I32, torch.int64: ID_MASK}[ids.dtype]
    # device memory, or page-locked host memory mapped into the device address space (UVA): the
    # union then reads only the kept rows over PCIe (zero-copy)
    assert (ids.is_cuda or ids.is_pinned()) and ids.is_contiguous()
    L = ids.shape[2]
    K = ids.shape[3] if id_format != ID_MASK else 0
    return _Routing(L, num_experts, K, id_format, _p(ids))


def evict_expert_union(keep_bits, ids, num_experts, n_nodes=None, max_nodes=None,
                       with_bits=True, expert_hist=None, stream=None):
    """ids: [B][N][L][K] uint8/int32 top-K ids, or [B][N][L][EW] int64 one-hot masks."""
    B, N, L = ids.shape[:3]
    dev = ids.device
    E = num_experts
    EW = (E + 63) // 64
    out = dict(union_count=torch.empty((B, L), dtype=torch.int32, device=dev),
               union_total=torch.empty(B, dtype=torch.int32, device=dev),
               status=torch.empty(B, dtype=torch.int32, device=dev))
    if with_bits:
        out["union_bits"] = torch.empty((B, L, EW), dtype=torch.int64, device=dev)
    tr = _Trees(B, N, _p(n_nodes), None, None)
    rt = _routing(ids, E)
    rc = lib().evict_expert_union(ctypes.byref(tr), _p(keep_bits), ctypes.byref(rt),
                                  _p(out["union_count"]), _p(out["union_total"]),
                                  _p(out.get("union_bits")), _p(expert_hist), _p(out["status"]),
                                  _stream(stream))
    _check(rc, "evict_expert_union")
    return out


# ----------------------------------------------------------------- fused (A1–A7)
class FusedBuffers:
    """Pre-allocated outputs of evict_select_build_union for a fixed batch shape."""

    def __init__(self, B, N, L, E, device, full=True, with_bits=False, with_order=False, with_stats=False):
        W = (N + 63) // 64
        EW = (E + 63) // 64
        cap = B * N
        d = device
        self.t = dict(k_star=torch.empty(B, dtype=torch.int32, device=d),
                      e_hat=torch.empty(B, dtype=torch.float32, device=d),
                      utility=torch.empty(B, dtype=torch.float32, device=d),
                      keep_bits=torch.empty((B, W), dtype=torch.int64, device=d),
                      verify_offsets=torch.empty(B + 1, dtype=torch.int32, device=d),
                      union_count=torch.empty((B, L), dtype=torch.int32, device=d),
                      union_total=torch.empty(B, dtype=torch.int32, device=d),
                      status=torch.empty(B, dtype=torch.int32, device=d))
        if full:
            for f in ("kept_index", "retrieve_index", "positions", "next_token", "next_sibling"):
                self.t[f] = torch.empty(cap, dtype=torch.int32, device=d)
            self.t["tree_mask"] = torch.empty((cap, W), dtype=torch.int64, device=d)
        if with_bits:
            self.t["union_bits"] = torch.empty((B, L, EW), dtype=torch.int64, device=d)
        if with_order:
            self.t["order"] = torch.empty((B, N), dtype=torch.int32, device=d)
            self.t["prefix_sums"] = torch.empty((B, N), dtype=torch.float32, device=d)
        if with_stats:   # A9 over the call's outputs (evict_batch_stats layout), ABI 8
            self.t["stats"] = torch.empty(6 + N + L, dtype=torch.int64, device=d)
            self.t["dstats"] = torch.empty(2, dtype=torch.float64, device=d)
        self.workspace = new_workspace(B, d)

    def struct(self, pos_offset=None):
        vals = {f: _p(self.t.get(f)) for f in _OUT_FIELDS}
        vals["pos_offset"] = _p(pos_offset)
        return _FusedOut(**vals)


def evict_select_build_union(parent, q, cost, ids, num_experts, n_nodes=None, cost_stride=0,
                             pos_offset=None, buffers=None, policy=None, stream=None, **buf_kw):
    B, N = parent.shape
    L = ids.shape[2]
    if buffers is None:
        buffers = FusedBuffers(B, N, L, num_experts, parent.device, **buf_kw)
    tr = _trees(parent, q, n_nodes)
    rt = _routing(ids, num_experts)
    o = buffers.struct(pos_offset)
    pol = _policy(policy)
    rc = lib().evict_select_build_union_policy(ctypes.byref(tr), _p(cost), cost_stride, _pp(pol),
                                               ctypes.byref(rt), ctypes.byref(o), _p(buffers.workspace),
                                               buffers.workspace.numel() * 8, _stream(stream))
    _check(rc, "evict_select_build_union_policy")
    return buffers.t


class FusedCall:
    """A pre-marshalled evict_select_build_union call (for CUDA-graph capture and timing loops)."""

    def __init__(self, parent, q, cost, ids, num_experts, n_nodes=None, cost_stride=0,
                 pos_offset=None, buffers=None, policy=None, **buf_kw):
        B, N = parent.shape
        L = ids.shape[2]
        self.keep = (parent, q, cost, ids, n_nodes, pos_offset)
        self.buffers = buffers or FusedBuffers(B, N, L, num_experts, parent.device, **buf_kw)
        self.tr = _trees(parent, q, n_nodes)
        self.rt = _routing(ids, num_experts)
        self.o = self.buffers.struct(pos_offset)
        self.cost = _p(cost)
        self.cs = cost_stride
        self.ws = _p(self.buffers.workspace)
        self.wsb = self.buffers.workspace.numel() * 8
        self.pol = _policy(policy)
        self.fn = lib().evict_select_build_union_policy

    def __call__(self, stream=None):
        rc = self.fn(ctypes.byref(self.tr), self.cost, self.cs, _pp(self.pol), ctypes.byref(self.rt),
                     ctypes.byref(self.o), self.ws, self.wsb, _stream(stream))
        if rc:
            raise EvictError(rc, "evict_select_build_union")
        return self.buffers.t


# ----------------------------------------------------------------- NEXT-1: union curve + profiler
def evict_union_curve(order, ids, num_experts, n_nodes=None, per_layer=False, stream=None):
    """Prefix-union curve along the ranking `order` ([B][N], evict_select's order row)."""
    B, N = order.shape
    L = ids.shape[2]
    dev = order.device
    out = dict(curve=torch.empty((B, N), dtype=torch.int32, device=dev),
               status=torch.empty(B, dtype=torch.int32, device=dev))
    if per_layer:
        out["curve_layer"] = torch.empty((B, N, L), dtype=torch.int32, device=dev)
    tr = _Trees(B, N, _p(n_nodes), None, None)
    rt = _routing(ids, num_experts)
    rc = lib().evict_union_curve(ctypes.byref(tr), _p(order), ctypes.byref(rt), _p(out["curve"]),
                                 _p(out.get("curve_layer")), _p(out["status"]), _stream(stream))
    _check(rc, "evict_union_curve")
    return out


def evict_profile_cost(curve, num_layers, n_nodes=None, status=None, c0=10.47, c_union=0.0915, c_tok=0.15,
                       stream=None):
    """Offline C(k) (fp32 [N]) from measured curves; a valid evict_select cost table."""
    B, N = curve.shape
    cost = torch.empty(N, dtype=torch.float32, device=curve.device)
    ws = torch.empty((lib().evict_profile_workspace_bytes(N) + 7) // 8, dtype=torch.int64, device=curve.device)
    rc = lib().evict_profile_cost(B, N, num_layers, _p(n_nodes), _p(curve), _p(status), c0, c_union, c_tok,
                                  _p(cost), _p(ws), ws.numel() * 8, _stream(stream))
    _check(rc, "evict_profile_cost")
    return cost


# ----------------------------------------------------------------- verify sampling (NEXT-3)
VERIFY_SAMPLE, VERIFY_GREEDY, VERIFY_EXACT = 0, 1, 0x10
TREE_BAD_TOKEN = 0x40


class _VerifyBatch(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("max_nodes", ctypes.c_int32), ("verify_offsets", ctypes.c_void_p),
                ("next_token", ctypes.c_void_p), ("next_sibling", ctypes.c_void_p),
                ("retrieve_index", ctypes.c_void_p), ("tokens", ctypes.c_void_p)]


def evict_verify_sample(verify_offsets, next_token, next_sibling, retrieve_index, tokens, probs,
                        u_accept=None, u_bonus=None, greedy=False, vocab=None, exact=False, stream=None, out=None):
    """Eq. 3 tree sampling (or greedy T = 0) on the packed verify tree.
    tokens: int32 [B][N] node-indexed draft tokens; probs: fp32 [T][stride] target rows;
    u_accept: uint32-as-int32 [B][N]; u_bonus: [B].  exact: force the fixed-point bonus path.
    Returns dict of CUDA tensors."""
    B, N = tokens.shape
    for t in (verify_offsets, next_token, next_sibling, retrieve_index, tokens):
        assert t.is_cuda and t.dtype == torch.int32 and t.is_contiguous()
    assert probs.dtype == torch.float32 and probs.dim() == 2 and probs.stride(1) == 1
    V = probs.shape[1] if vocab is None else int(vocab)
    dev = tokens.device
    if out is None:
        out = dict(accept_len=torch.empty(B, dtype=torch.int32, device=dev),
                   accepted_slots=torch.empty((B, N), dtype=torch.int32, device=dev),
                   bonus_token=torch.empty(B, dtype=torch.int32, device=dev),
                   status=torch.empty(B, dtype=torch.int32, device=dev))
    vb = _VerifyBatch(B, N, _p(verify_offsets), _p(next_token), _p(next_sibling), _p(retrieve_index), _p(tokens))
    rc = lib().evict_verify_sample(ctypes.byref(vb), _p(probs), V, probs.stride(0),
                                   (VERIFY_GREEDY if greedy else VERIFY_SAMPLE) | (VERIFY_EXACT if exact else 0),
                                   _p(u_accept), _p(u_bonus),
                                   _p(out["accept_len"]), _p(out["accepted_slots"]), _p(out["bonus_token"]),
                                   _p(out["status"]), _stream(stream))
    _check(rc, "evict_verify_sample")
    return out


# ----------------------------------------------------------------- draft-tree builder (NEXT-4, P2)
def evict_build_draft_tree(child_tokens, child_probs, max_nodes, out=None, stream=None):
    """child_tokens int32 / child_probs fp32 CUDA [B][steps][topk][topk] → dict(parent, q, tokens
    [B][max_nodes], n_nodes [B], status [B]) — a ready evict_trees_t batch."""
    B, S, K1, K2 = child_tokens.shape
    assert K1 == K2 and child_probs.shape == child_tokens.shape
    assert child_tokens.dtype == torch.int32 and child_probs.dtype == torch.float32
    assert child_tokens.is_contiguous() and child_probs.is_contiguous()
    dev = child_tokens.device
    N = int(max_nodes)
    if out is None:
        out = dict(parent=torch.empty((B, N), dtype=torch.int32, device=dev),
                   q=torch.empty((B, N), dtype=torch.float32, device=dev),
                   tokens=torch.empty((B, N), dtype=torch.int32, device=dev),
                   n_nodes=torch.empty(B, dtype=torch.int32, device=dev),
                   status=torch.empty(B, dtype=torch.int32, device=dev))
    rc = lib().evict_build_draft_tree(B, S, K1, N, _p(child_tokens), _p(child_probs), _p(out["parent"]),
                                      _p(out["q"]), _p(out["tokens"]), _p(out["n_nodes"]), _p(out["status"]),
                                      _stream(stream))
    _check(rc, "evict_build_draft_tree")
    return out


# ----------------------------------------------------------------- verify-graph dispatch (NEXT-4)
class VerifyDispatch:
    """One CUDA graph: [pre] → device-side choice of the verify graph → SWITCH over the bodies.

    lengths: ascending verification lengths, one per body; bodies: torch.cuda.CUDAGraph objects
    captured with keep_graph=True (their cudaGraph_t is cloned); pre: optional CUDAGraph run first;
    rows: int32 CUDA tensor whose first element is the step's verify row count at launch
    (e.g. verify_offsets[B:]); chosen: int32 CUDA tensor [1] receiving the body index (or -1)."""

    def __init__(self, lengths, bodies, rows, chosen=None, pre=None):
        assert len(lengths) == len(bodies) >= 1
        n = len(lengths)
        self._lens = (ctypes.c_int32 * n)(*[int(x) for x in lengths])
        self._bodies = (ctypes.c_void_p * n)(*[int(b.raw_cuda_graph()) for b in bodies])
        self._keep = (rows, chosen, bodies, pre)
        self._h = ctypes.c_void_p()
        rc = lib().evict_dispatch_create(n, self._lens, self._bodies,
                                         ctypes.c_void_p(int(pre.raw_cuda_graph())) if pre is not None else None,
                                         _p(rows), _p(chosen), ctypes.byref(self._h))
        _check(rc, "evict_dispatch_create")

    def launch(self, stream=None):
        _check(lib().evict_dispatch_launch(self._h, _stream(stream)), "evict_dispatch_launch")

    def close(self):
        if self._h:
            lib().evict_dispatch_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass


# ----------------------------------------------------------------- router (A8 → A7)
def evict_router_union(verify_offsets, retrieve_index, hidden, w_gate, top_k, batch, max_nodes,
                       with_topk=False, max_rows=0, stream=None):
    """hidden: bf16 [L][B*N][d]; w_gate: bf16 [L][E][d]; rows from evict_build_verify_tree."""
    L, BN, d = hidden.shape
    E = w_gate.shape[1]
    dev = hidden.device
    EW = (E + 63) // 64
    out = dict(union_count=torch.empty((batch, L), dtype=torch.int32, device=dev),
               union_total=torch.empty(batch, dtype=torch.int32, device=dev),
               union_bits=torch.empty((batch, L, EW), dtype=torch.int64, device=dev))
    if with_topk:
        out["topk_ids"] = torch.full((L, BN, top_k), -1, dtype=torch.int32, device=dev)
    tr = _Trees(batch, max_nodes, None, None, None)
    rt = _Router(L, E, top_k, d, _p(hidden), _p(w_gate), int(max_rows))
    rc = lib().evict_router_union(ctypes.byref(tr), _p(verify_offsets), _p(retrieve_index),
                                  ctypes.byref(rt), _p(out["union_count"]), _p(out["union_total"]),
                                  _p(out["union_bits"]), _p(out.get("topk_ids")), _stream(stream))
    _check(rc, "evict_router_union")
    return out


class RouterCall:
    """A pre-marshalled evict_router_union call with pre-allocated outputs (timing loops, graphs)."""

    def __init__(self, verify_offsets, retrieve_index, hidden, w_gate, top_k, batch, max_nodes,
                 with_topk=False, max_rows=0):
        L, BN, d = hidden.shape
        E = w_gate.shape[1]
        dev = hidden.device
        EW = (E + 63) // 64
        self.keep = (verify_offsets, retrieve_index, hidden, w_gate)
        self.t = dict(union_count=torch.empty((batch, L), dtype=torch.int32, device=dev),
                      union_total=torch.empty(batch, dtype=torch.int32, device=dev),
                      union_bits=torch.empty((batch, L, EW), dtype=torch.int64, device=dev))
        if with_topk:
            self.t["topk_ids"] = torch.full((L, BN, top_k), -1, dtype=torch.int32, device=dev)
        self.tr = _Trees(batch, max_nodes, None, None, None)
        self.rt = _Router(L, E, top_k, d, _p(hidden), _p(w_gate), int(max_rows))
        self.args = (_p(verify_offsets), _p(retrieve_index))
        self.fn = lib().evict_router_union

    def __call__(self, stream=None):
        rc = self.fn(ctypes.byref(self.tr), self.args[0], self.args[1], ctypes.byref(self.rt),
                     _p(self.t["union_count"]), _p(self.t["union_total"]), _p(self.t["union_bits"]),
                     _p(self.t.get("topk_ids")), _stream(stream))
        if rc:
            raise EvictError(rc, "evict_router_union")
        return self.t


# ----------------------------------------------------------------- stats (A9)
def evict_batch_stats(k_star, e_hat, utility, union_count, status, max_nodes, n_nodes=None,
                      stream=None):
    B = k_star.shape[0]
    L = 0 if union_count is None else union_count.shape[1]
    dev = k_star.device
    stats = torch.empty(6 + max_nodes + L, dtype=torch.int64, device=dev)
    dstats = torch.empty(2, dtype=torch.float64, device=dev)
    rc = lib().evict_batch_stats(B, max_nodes, L, _p(n_nodes), _p(k_star), _p(e_hat),
                                 _p(utility), _p(union_count), _p(status), _p(stats), _p(dstats),
                                 _stream(stream))
    _check(rc, "evict_batch_stats")
    return stats, dstats
