"""Request sharding on one GPU: the C5 set split as the bench splits it
over G ranks ([⌊rM/G⌋, ⌊(r+1)M/G⌋), each shard generated from (seed, tree id)) and run shard by
shard must give per-tree outputs that concatenate bit-identically to the single-shard run, and
A9 statistics that sum to the single-shard statistics (integers exact)."""
import numpy as np
import pytest

import gen

pytestmark = pytest.mark.gpu


def _run(ev, torch, base, M, N=60, L=48, E=128, K=8):
    P, Q, n = gen.trees_cuda(5, M, N, 6, 10, tree_base=base)
    ids = gen.routing_cuda(5, M, N, L, E, K, tree_base=base)
    cost = torch.from_numpy(gen.cost_table(N)).cuda()
    call = ev.FusedCall(P, Q, cost, ids, E, n_nodes=n)
    out = {k: v.clone() for k, v in call().items()}
    st, dst = ev.evict_batch_stats(out["k_star"], out["e_hat"], out["utility"], out["union_count"],
                                   out["status"], N, n_nodes=n)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}, st.cpu().numpy(), dst.cpu().numpy()


@pytest.mark.parametrize("G", [2, 3, 8])
def test_shards_concatenate_to_the_single_run(G):
    import torch
    import paper_2605_00342_b200 as ev
    from paper_2605_00342_b200.dist import shard
    M = 100_003
    full, st, dst = _run(ev, torch, 0, M)
    parts, sts, dsts = [], [], []
    for r in range(G):
        lo, m = shard(r, G, 0, total=M)
        o, s, d = _run(ev, torch, lo, m)
        parts.append(o)
        sts.append(s)
        dsts.append(d)
    for key in ("k_star", "e_hat", "utility", "keep_bits", "union_count", "union_total", "status"):
        cat = np.concatenate([p[key] for p in parts])
        assert cat.shape == full[key].shape and (cat.view(np.uint8) == full[key].view(np.uint8)).all(), key
    # packed verify rows: shard r's rows are the full run's rows [off, off + T_r) with the offsets
    # shifted by off = full verify_offsets[lo], and retrieve_index (b·N + node) by lo·N
    N = full["keep_bits"].shape[0] and 60
    for r, p in enumerate(parts):
        lo, m = shard(r, G, 0, total=M)
        off = int(full["verify_offsets"][lo])
        assert (p["verify_offsets"][:m + 1] + off == full["verify_offsets"][lo:lo + m + 1]).all()
        T = int(p["verify_offsets"][m])
        for key in ("kept_index", "positions", "next_token", "next_sibling"):
            assert (p[key][:T] == full[key][off:off + T]).all(), key
        assert (p["retrieve_index"][:T] + lo * N == full["retrieve_index"][off:off + T]).all()
        assert (p["tree_mask"][:T] == full["tree_mask"][off:off + T]).all()
    assert (np.sum(sts, axis=0) == st).all()               # the all-reduce(SUM) of the shards
    assert np.allclose(np.sum(dsts, axis=0), dst, rtol=1e-9)
