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
