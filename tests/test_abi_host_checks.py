"""Host-side argument checks of the newer entry points (CPU only: every error below is detected
before any device access, and a well-formed call on a machine without an sm_100 device returns
EVICT_ERR_UNSUPPORTED instead of launching)."""
import ctypes

import pytest

INVALID, UNSUPPORTED = 1, 2


@pytest.fixture(scope="module")
def lib():
    import paper_2605_00342_b200 as ev
    from paper_2605_00342_b200 import build
    build.build()
    return ev.lib()


class VB(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("max_nodes", ctypes.c_int32), ("verify_offsets", ctypes.c_void_p),
                ("next_token", ctypes.c_void_p), ("next_sibling", ctypes.c_void_p),
                ("retrieve_index", ctypes.c_void_p), ("tokens", ctypes.c_void_p)]


FAKE = 0x10000   # a 16-byte-aligned non-null "device" address (never dereferenced on these paths)


def _verify(lib, vb, vocab=1000, stride=1000, mode=0, probs=FAKE, ua=FAKE, ub=FAKE):
    p = ctypes.c_void_p
    return lib.evict_verify_sample(ctypes.byref(vb) if vb is not None else None, p(probs), vocab, stride, mode,
                                   p(ua), p(ub), p(FAKE), p(FAKE), p(FAKE), None, None)


def test_verify_sample_checks(lib):
    vb = VB(4, 60, FAKE, FAKE, FAKE, FAKE, FAKE)
    assert _verify(lib, None) == INVALID
    assert _verify(lib, VB(0, 60, FAKE, FAKE, FAKE, FAKE, FAKE)) == INVALID      # batch
    assert _verify(lib, VB(4, 129, FAKE, FAKE, FAKE, FAKE, FAKE)) == INVALID     # N > 128
    assert _verify(lib, VB(4, 60, 0, FAKE, FAKE, FAKE, FAKE)) == INVALID         # null offsets
    assert _verify(lib, vb, vocab=0) == INVALID
    assert _verify(lib, vb, vocab=262145, stride=262148) == INVALID              # > EVICT_MAX_VOCAB
    assert _verify(lib, vb, stride=999) == INVALID                               # stride < vocab
    assert _verify(lib, vb, vocab=998, stride=998 + 1) == INVALID                # stride % 4
    assert _verify(lib, vb, probs=FAKE + 4) == INVALID                           # 16-byte alignment
    assert _verify(lib, vb, mode=2) == INVALID                                   # unknown mode bit
    assert _verify(lib, vb, ua=0) == INVALID                                     # sampling needs uniforms
    assert _verify(lib, vb, mode=1, ua=0, ub=0) == UNSUPPORTED                   # greedy: no uniforms, no GPU
    assert _verify(lib, vb, mode=0x10) == UNSUPPORTED                            # forced-exact sampling


def _draft(lib, B=4, steps=6, topk=10, N=60, ptr=FAKE):
    p = ctypes.c_void_p
    return lib.evict_build_draft_tree(B, steps, topk, N, p(ptr), p(FAKE), p(FAKE), p(FAKE), p(FAKE), p(FAKE),
                                      None, None)


def test_draft_tree_checks(lib):
    assert _draft(lib, B=0) == INVALID
    assert _draft(lib, steps=0) == INVALID
    assert _draft(lib, steps=17) == INVALID
    assert _draft(lib, topk=0) == INVALID
    assert _draft(lib, topk=17) == INVALID
    assert _draft(lib, N=129) == INVALID
    assert _draft(lib, steps=10, topk=16) == INVALID          # pool 1 + 16 + 9·256 > 2048
    assert _draft(lib, ptr=0) == INVALID
    assert _draft(lib) == UNSUPPORTED                         # well-formed, no sm_100 device here


def test_dispatch_checks(lib):
    p = ctypes.c_void_p
    out = p()
    lens = (ctypes.c_int32 * 3)(8, 16, 32)
    bodies = (p * 3)(FAKE, FAKE, FAKE)
    assert lib.evict_dispatch_create(0, lens, bodies, None, p(FAKE), None, ctypes.byref(out)) == INVALID
    assert lib.evict_dispatch_create(33, lens, bodies, None, p(FAKE), None, ctypes.byref(out)) == INVALID
    bad = (ctypes.c_int32 * 3)(8, 8, 32)
    assert lib.evict_dispatch_create(3, bad, bodies, None, p(FAKE), None, ctypes.byref(out)) == INVALID
    assert lib.evict_dispatch_create(3, lens, (p * 3)(FAKE, 0, FAKE), None, p(FAKE), None,
                                     ctypes.byref(out)) == INVALID
    assert lib.evict_dispatch_create(3, lens, bodies, None, None, None, ctypes.byref(out)) == INVALID
    assert lib.evict_dispatch_create(3, lens, bodies, None, p(FAKE), None, None) == INVALID
    assert lib.evict_dispatch_launch(None, None) == INVALID
    lib.evict_dispatch_destroy(None)                           # a no-op on NULL
    assert lib.evict_dispatch_create(3, lens, bodies, None, p(FAKE), None, ctypes.byref(out)) == UNSUPPORTED
    assert not out.value


def _profile(lib, c0=10.47, cu=0.0915, ct=0.15, N=60):
    p = ctypes.c_void_p
    ws = lib.evict_profile_workspace_bytes(N)
    return lib.evict_profile_cost(8, N, 48, None, p(FAKE), None, c0, cu, ct, p(FAKE), p(FAKE), ws, None)


def test_profile_cost_checks(lib):
    """Coefficients that could give cost[k] <= 0 or overflow fp32 are rejected on the host (the
    result must always be a valid evict_select cost table)."""
    assert _profile(lib, c0=0.0) == INVALID
    assert _profile(lib, c0=-1.0) == INVALID
    assert _profile(lib, cu=-0.5) == INVALID
    assert _profile(lib, ct=-0.1) == INVALID
    assert _profile(lib, c0=float("nan")) == INVALID
    assert _profile(lib, cu=3.0e38) == INVALID                # 256 * c_union overflows fp32
    assert _profile(lib, c0=1e-30, cu=0.0, ct=0.0) == UNSUPPORTED   # valid, no sm_100 device here
    assert _profile(lib) == UNSUPPORTED


def test_router_checks(lib):
    """evict_router_union: E > 256 is UNSUPPORTED, a well-formed E < 128 call (the C1 toy shape)
    reaches the device check (no sm_100 device here)."""
    p = ctypes.c_void_p

    class Trees(ctypes.Structure):
        _fields_ = [("batch", ctypes.c_int32), ("max_nodes", ctypes.c_int32), ("n_nodes", p),
                    ("parent", p), ("q", p)]

    class Router(ctypes.Structure):
        _fields_ = [("num_layers", ctypes.c_int32), ("num_experts", ctypes.c_int32), ("top_k", ctypes.c_int32),
                    ("hidden_dim", ctypes.c_int32), ("hidden", p), ("w_gate", p), ("max_rows", ctypes.c_int32)]

    tr = Trees(1, 8, None, None, None)

    def call(E, K=2, d=64):
        rt = Router(2, E, K, d, FAKE, FAKE, 0)
        return lib.evict_router_union(ctypes.byref(tr), p(FAKE), p(FAKE), ctypes.byref(rt), p(FAKE), None,
                                      p(FAKE), None, None)

    assert call(320) == UNSUPPORTED
    assert call(8, K=9) == INVALID                            # K > E
    assert call(8, d=96) == INVALID                           # d % 64
    assert call(8) == UNSUPPORTED                             # C1 toy shape: supported, no device here
