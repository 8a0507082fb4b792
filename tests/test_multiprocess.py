"""Multi-rank plumbing on CPU with a world-size-2 gloo group (the NCCL path's host logic)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import gen
    import oracle
    from paper_2605_00342_b200.dist import allreduce_stats, max_over_ranks, shard
    M, N, L, E, K = 300, 60, 6, 128, 8
    base, m = shard(rank, world, M)
    P, Q, n = gen.trees(5, m, N, 6, 10, tree_base=base)
    ids = gen.routing(5, m, N, L, E, K, tree_base=base)
    o = oracle.select(P, Q, gen.cost_table(N), n_nodes=n)
    u = oracle.expert_union(o["keep_bits"], ids, E, n_nodes=n)
    st, d = oracle.batch_stats(N, L, o["k_star"], o["e_hat"], o["utility"], u["union_count"],
                               o["status"], n_nodes=n)
    st_t, d_t = torch.from_numpy(st.copy()), torch.from_numpy(d.copy())
    allreduce_stats(st_t, d_t)
    t = max_over_ranks(torch.tensor([float(rank + 1)]))
    q.put((rank, st_t.numpy(), d_t.numpy(), float(t[0])))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_stats_equal_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import gen
    import oracle
    M, N, L, E, K = 300, 60, 6, 128, 8
    P, Q, n = gen.trees(5, M * world, N, 6, 10)
    ids = gen.routing(5, M * world, N, L, E, K)
    o = oracle.select(P, Q, gen.cost_table(N), n_nodes=n)
    u = oracle.expert_union(o["keep_bits"], ids, E, n_nodes=n)
    st, d = oracle.batch_stats(N, L, o["k_star"], o["e_hat"], o["utility"], u["union_count"],
                               o["status"], n_nodes=n)
    for rank, s, dd, t in res:
        assert (s == st).all()                          # integers: exact
        assert np.allclose(dd, d, rtol=1e-12)
        assert t == world                               # max over ranks


def test_shard_ranges():
    from paper_2605_00342_b200.dist import shard
    assert shard(3, 8, 1000) == (3000, 1000)
    parts = [shard(r, 3, 0, total=10) for r in range(3)]
    assert parts == [(0, 3), (3, 3), (6, 4)]


@pytest.mark.parametrize("scaling,trees,world", [("strong", 1000, 2), ("strong", 1_000_001, 3), ("weak", 777, 2)])
def test_bench_launcher_world2_gloo(scaling, trees, world):
    """`bench.py --gpus N` with no torchrun environment spawns N ranks itself (torch.distributed.run
    on 127.0.0.1); the dry run takes each rank's shard and runs the step's collectives on gloo.
    The shards must tile the tree ids exactly once (strong: [0, trees); weak: trees per rank)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(world), "--dry-run",
                        "--trees", str(trees), "--scaling", scaling], capture_output=True, text=True,
                       timeout=240, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout            # rank 0 alone prints the line
    out = json.loads(lines[0])
    assert out["n_gpus"] == world and out["backend"] == "gloo"
    total = trees if scaling == "strong" else trees * world
    shards = out["shards"]
    assert shards[0][0] == 0 and all(a + m == b for (a, m), (b, _) in zip(shards, shards[1:]))
    assert sum(m for _, m in shards) == total == out["trees"]
    assert max(m for _, m in shards) - min(m for _, m in shards) <= (1 if scaling == "strong" else 0)
    assert out["id_sum"] == total * (total - 1) // 2          # every id once (all-reduced)
    assert out["id_sq_sum"] == (total - 1) * total * (2 * total - 1) // 6
