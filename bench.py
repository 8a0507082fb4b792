#!/usr/bin/env python
"""EVICT hot-path benchmark (BASELINE.json metric: trees/s and µs per batch-64 selection;
expert-union HBM GB/s vs B200 peak at 1/2/4/8 GPUs).

Workload (BASELINE.json configs[4], "c5"): the set of 1,000,000 synthetic EAGLE-3-shaped draft
trees of 60 nodes (steps 6, topk 10) with Qwen3-30B-A3B-shaped routing (48 layers × 128 experts,
top-8, uint8 ids: 23 GB), sharded by request over the N ranks (rank r: tree ids
[⌊rM/N⌋, ⌊(r+1)M/N⌋), generated on its GPU from (seed, tree id), device-resident).  One step =
one pass of the whole hot path over the rank's shard: the fused select → verify-tree build →
expert-union launch (A1–A7), the batch statistics kernel (A9) and, for N > 1, the NCCL
all-reduce of those statistics.  The headline splits the fixed 1M-tree set ("scaling":
"strong"); for N > 1 a weak-scaling sweep (1M trees per rank) is reported beside it.

`python bench.py --gpus N` without a torchrun environment re-executes itself under
torch.distributed.run with N local ranks (one per GPU, NCCL over NVLink).

Timing: W warm-up steps, then K steps between a barrier + synchronize on both sides, timed
with CUDA events on the launching stream, max over ranks.  Inputs (23 GB/rank) are far larger
than the 126 MB L2, so no flush is needed between steps.

`--impl reference` times the CPU oracle (oracle/, the reference arm of this tier) on the host
cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("trees/s and µs per batch-64 selection; expert-union HBM GB/s vs B200 peak at "
          "1/2/4/8 GPUs")
SEED = 5
N_NODES, STEPS, TOPK = 60, 6, 10
L_LAYERS, N_EXPERTS, TOP_K = 48, 128, 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--trees", type=int, default=1_000_000,
                    help="total trees (strong scaling: split over the ranks)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: --trees in total; weak: --trees per rank")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU check of the launcher, sharding and all-reduce (gloo, no kernels)")
    ap.add_argument("--id-format", default="u8", choices=["u8", "i32", "mask"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-extras", action="store_true", help="skip latency / variant sub-benchmarks")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def hbm_peak():
    p = peaks()
    if "hbm_gbs" in p:
        return float(p["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
_SAMPLER = r"""
import sys, time
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
        nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
print("ready", flush=True)
while True:
    t = time.time()
    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
    print(f"{t:.6f},{sm},{mx}," + ",".join("1" if r & b else "0" for b in bits), flush=True)
    time.sleep(0.001)
"""


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region by a separate NVML process
    (no GIL sharing with the launching thread) polling every ~1 ms; only samples whose host
    timestamp falls inside [region start, region end] are kept.  nvidia-smi -lms 100 is the
    fallback when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.kind = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER, str(self.gpu)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            if self.proc.stdout.readline().strip() == "ready":
                self.kind = "nvml"
                return
            self.proc.kill()
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.kind = "smi"
        except Exception:
            self.proc = None

    def region(self, on):
        """Mark the timed region by host wall clock."""
        if on:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        rows = []
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            try:
                if self.kind == "nvml" and len(f) == 7:
                    t = float(f[0])
                    if self.t0 is not None and self.t1 is not None and not (self.t0 <= t <= self.t1):
                        continue
                    rows.append((float(f[1]), float(f[2]), ["Active" if x == "1" else "" for x in f[3:7]]))
                elif self.kind == "smi" and len(f) >= 8:
                    rows.append((float(f[0]), float(f[1]), f[4:8]))
            except ValueError:
                continue
        if not rows:
            return None
        sm = sorted(r[0] for r in rows)
        reasons = sorted({self.NAMES[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows),
                "source": "nvml process ~1 ms, timed region only" if self.kind == "nvml" else "nvidia-smi 100 ms"}


# ------------------------------------------------------------------ algorithmic bytes
def algorithmic_bytes(n_sum, k_sum, trees, id_bytes, W=1, L=L_LAYERS, K=TOP_K, EW=2,
                      id_format="u8"):
    """SURVEY.md §8(d) per-unit figures × units:
    select  in 8n (parent+q), out 12 + 8W (k*, e_hat, utility, keep) + 4 (status)
    build   out k*(20 + 8W) + 4 (verify_offsets)
    union   in k*·L·K·s_id (ids) or k*·L·EW·8 (masks), out 4L + 4 (counts, total)."""
    row = L * K * id_bytes if id_format != "mask" else L * EW * 8
    sel = 8 * n_sum + trees * (12 + 8 * W + 4)
    bld = k_sum * (20 + 8 * W) + trees * 4
    uni = k_sum * row + trees * (4 * L + 4)
    return sel + bld + uni, dict(select=sel, build=bld, union=uni)


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    import numpy as np

    import gen
    import oracle
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    # pilot to size a bounded sample (~cpu_seconds of oracle work per step)
    pilot = 2000
    P, Q, n = gen.trees(SEED, pilot, N_NODES, STEPS, TOPK)
    ids = gen.routing(SEED, pilot, N_NODES, L_LAYERS, N_EXPERTS, TOP_K)
    cost = gen.cost_table(N_NODES)
    t0 = time.perf_counter()
    o = oracle.select(P, Q, cost, n_nodes=n, threads=threads)
    oracle.build_verify_tree(P, o["keep_bits"], n_nodes=n)
    oracle.expert_union(o["keep_bits"], ids, N_EXPERTS, n_nodes=n, threads=threads)
    per_tree = (time.perf_counter() - t0) / pilot
    budget = args.cpu_seconds / max(1, args.steps + args.warmup)
    S = int(min(200_000, max(2000, budget / per_tree)))
    P, Q, n = gen.trees(SEED, S, N_NODES, STEPS, TOPK, threads=threads)
    ids = gen.routing(SEED, S, N_NODES, L_LAYERS, N_EXPERTS, TOP_K, threads=threads)

    def step():
        o = oracle.select(P, Q, cost, n_nodes=n, threads=threads)
        oracle.build_verify_tree(P, o["keep_bits"], n_nodes=n)
        oracle.expert_union(o["keep_bits"], ids, N_EXPERTS, n_nodes=n, threads=threads)
        return o

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / max(1, args.steps)
    v = S / dt
    sample = (f"first {S} trees of the c5 workload (seed {SEED}), oracle select+build+union "
              f"per step, {threads} host threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "trees/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": config_dict(args, world, S),
        "cpu_baseline": {"value": v, "unit": "trees/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": v, "unit": "trees/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, world, trees=None, total=None):
    return {"workload": "c5: EAGLE-3-shaped 60-node draft trees (steps 6, topk 10), "
                        "Qwen3-30B-A3B-shaped routing 48 layers x 128 experts top-8",
            "trees_total": total if total is not None else (
                args.trees if args.scaling == "strong" else args.trees * world),
            "trees_per_rank": trees or (args.trees if args.scaling == "weak" else
                                        -(-args.trees // world)), "max_nodes": N_NODES, "layers": L_LAYERS,
            "experts": N_EXPERTS, "top_k": TOP_K, "id_format": args.id_format,
            "cost_table": "C(k)=10.47+0.0915*U(k)+0.15k ms (DESIGN.md §4)",
            "l2": "inputs >= 23 GB per rank >> 126 MB L2; no flush needed",
            "parallelism": f"dp{world} (trees sharded by request, NCCL all-reduce of stats)"}


# ------------------------------------------------------------------ native arm
def cpu_baseline(args, k_star_mean, gpu_out=None, base=0):
    import numpy as np

    import gen
    import oracle
    from oracle.parity import compare_select, compare_union, downstream_keep
    threads = os.cpu_count() or 1
    cost = gen.cost_table(N_NODES)
    pilot = 2000
    P, Q, n = gen.trees(SEED, pilot, N_NODES, STEPS, TOPK, tree_base=base, threads=threads)
    ids = gen.routing(SEED, pilot, N_NODES, L_LAYERS, N_EXPERTS, TOP_K, tree_base=base, threads=threads)
    t0 = time.perf_counter()
    o = oracle.select(P, Q, cost, n_nodes=n, threads=threads)
    oracle.build_verify_tree(P, o["keep_bits"], n_nodes=n)
    oracle.expert_union(o["keep_bits"], ids, N_EXPERTS, n_nodes=n, threads=threads)
    per = (time.perf_counter() - t0) / pilot
    S = int(min(400_000, max(pilot, args.cpu_seconds / per)))
    P, Q, n = gen.trees(SEED, S, N_NODES, STEPS, TOPK, tree_base=base, threads=threads)
    ids = gen.routing(SEED, S, N_NODES, L_LAYERS, N_EXPERTS, TOP_K, tree_base=base, threads=threads)
    t0 = time.perf_counter()
    o = oracle.select(P, Q, cost, n_nodes=n, threads=threads)
    oracle.build_verify_tree(P, o["keep_bits"], n_nodes=n)
    ou = oracle.expert_union(o["keep_bits"], ids, N_EXPERTS, n_nodes=n, threads=threads)
    dt = time.perf_counter() - t0
    # parity of the GPU's outputs for the same trees (the bench's exact launch; SURVEY §5 counts)
    parity = None
    if gpu_out is not None:
        m = min(S, len(gpu_out["k_star"]))
        osub = {k: v[:m] for k, v in o.items()}
        res, msgs = compare_select(osub, {k: gpu_out[k][:m] for k in ("k_star", "e_hat", "utility",
                                                                      "keep_bits", "status")}, n_nodes=n[:m])
        keep = downstream_keep(osub, {"k_star": gpu_out["k_star"][:m]})
        ou2 = ou if (keep == o["keep_bits"][:m]).all() and m == S else oracle.expert_union(
            keep, ids[:m], N_EXPERTS, n_nodes=n[:m], threads=threads)
        um = compare_union({k: v[:m] for k, v in ou2.items()},
                           {k: gpu_out[k][:m] for k in ("union_count", "union_total")})
        parity = dict(res, trees=m, union_mismatch=len(um), first_mismatch=(msgs + um)[:1],
                      rule="k*/keep bit-exact, e_hat/utility 1e-5 rel, ties per the oracle near-tie set; "
                           "union counts bit-exact")
    per_config = {}
    for name in ("toy", "c2", "c3", "c4"):
        per_config[name] = _oracle_config_ms(gen, oracle, name, threads)
    # one-thread rate on the first 20,000 of the same trees (both are reported)
    S1 = min(S, 20_000)
    t0 = time.perf_counter()
    o1 = oracle.select(P[:S1], Q[:S1], cost, n_nodes=n[:S1], threads=1)
    oracle.build_verify_tree(P[:S1], o1["keep_bits"], n_nodes=n[:S1])
    oracle.expert_union(o1["keep_bits"], ids[:S1], N_EXPERTS, n_nodes=n[:S1], threads=1)
    dt1 = time.perf_counter() - t0
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
    except OSError:
        pass
    return {"value": S / dt, "unit": "trees/s", "cores": threads, "kind": "oracle",
            "one_thread_value": S1 / dt1, "cpu_model": model, "parity": parity,
            "per_config_ms_per_batch": per_config,
            "sample": f"first {S} trees of rank 0's c5 shard (seed {SEED}); oracle select+build+"
                      f"union (C, fp64 sums) on {threads} host threads (one_thread_value: first {S1} "
                      f"on 1 thread); generation excluded"}


def _oracle_config_ms(gen, oracle, name, threads):
    """Oracle select+build+union ms per batch of a BASELINE config (C1 toy / C2 / C3 / C4),
    median of 5."""
    import numpy as np
    c = gen.CONFIGS[name]
    if name == "toy":
        P, Q, n = gen.TOY_PARENT[None], gen.TOY_Q[None], np.array([8], np.int32)
        cost = gen.TOY_COST
        ids = gen.TOY_ROUTING[None]
        E = c["E"]
    else:
        P, Q, n = gen.trees(c["seed"], c["B"], c["N"], c["steps"], c["topk"])
        cost = gen.cost_table(c["N"])
        ids = gen.routing(c["seed"], c["B"], c["N"], c["L"], c["E"], c["K"])
        E = c["E"]
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        o = oracle.select(P, Q, cost, n_nodes=n, threads=threads)
        oracle.build_verify_tree(P, o["keep_bits"], n_nodes=n)
        oracle.expert_union(o["keep_bits"], ids, E, n_nodes=n, threads=threads)
        ts.append((time.perf_counter() - t0) * 1e3)
    return {"B": int(P.shape[0]), "N": int(P.shape[1]), "ms": float(np.median(ts))}


def latency(ev, torch, gen, B=64, N=60, steps=6, topk=10, seed=4, replays=2000):
    """µs per batch-B selection (select only, and fused select+build+union), CUDA-graph replay.
    B = 64 is the north_star latency point; B = 1 the paper's serving setting."""
    import numpy as np
    P, Q, n = gen.trees(seed, B, N, steps, topk)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    tP, tQ, tn, tc = cu(P), cu(Q), cu(n), cu(gen.cost_table(N))
    ids = gen.routing_cuda(seed, B, N, L_LAYERS, N_EXPERTS, TOP_K)
    out = {}
    s = torch.cuda.Stream()
    for name in ("select", "fused"):
        if name == "select":
            bufs = ev.evict_select(tP, tQ, tc, n_nodes=tn)   # allocate once

            def call(st):
                tr = ev._trees(tP, tQ, tn)
                return ev.lib().evict_select(ev.ctypes.byref(tr), ev._p(tc), 0, ev._p(bufs["k_star"]),
                                             ev._p(bufs["e_hat"]), ev._p(bufs["utility"]),
                                             ev._p(bufs["keep_bits"]), None, None,
                                             ev._p(bufs["status"]), ev._stream(st))
        else:
            fc = ev.FusedCall(tP, tQ, tc, ids, N_EXPERTS, n_nodes=tn)

            def call(st):
                fc(st)
                return 0
        with torch.cuda.stream(s):
            for _ in range(3):
                assert call(s) == 0
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            call(s)
        with torch.cuda.stream(s):
            for _ in range(50):
                g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(replays):
                g.replay()
            e1.record(s)
        e1.synchronize()
        out[f"{name}_b{B}_n{N}_us"] = e0.elapsed_time(e1) * 1e3 / replays
        # per-replay device times (SURVEY §8(d) latency): p50 / p99 over 1000 replays
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(1000)]
        with torch.cuda.stream(s):
            for a, b in evs:
                a.record(s)
                g.replay()
                b.record(s)
        s.synchronize()
        t = np.sort([a.elapsed_time(b) * 1e3 for a, b in evs])
        out[f"{name}_b{B}_n{N}_p50_us"] = float(t[len(t) // 2])
        out[f"{name}_b{B}_n{N}_p99_us"] = float(t[int(len(t) * 0.99)])
    return out


def time_fused(ev, torch, call, stream, reps):
    """Mean device time of `call` (a FusedCall) over reps launches, CUDA events on `stream`."""
    for _ in range(3):
        call(stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        call(stream)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def ling_variant(ev, gen, torch, P, Q, n, cost, M, stream, reps):
    """NEXT-4 model shape: the same trees with Ling-flash-2.0-shaped routing (256 experts top-8,
    PAPER.md:557; 32 MoE layers), u8 ids [M][60][32][8] (15.4 KB per tree), fused
    select → build → union with 4-word expert sets."""
    L, E = 32, 256
    ids = gen.routing_cuda(6, M, P.shape[1], L, E, TOP_K)
    call = ev.FusedCall(P, Q, cost, ids, E, n_nodes=n)
    ms = time_fused(ev, torch, call, stream, reps)
    k_sum = int(call.buffers.t["k_star"].sum())
    n_sum = int(n.sum())
    abytes, parts = algorithmic_bytes(n_sum, k_sum, M, 1, L=L, EW=4)
    peak, _ = hbm_peak()
    ach = abytes / (ms / 1e3) / 1e9
    um = float(call.buffers.t["union_total"].double().mean()) / L
    del call, ids
    torch.cuda.empty_cache()
    return {"model": "Ling-flash-2.0-shaped (L 32, E 256, top-8)", "id_format": "u8", "value": M / (ms / 1e3),
            "unit": "trees/s", "kernel_ms": ms, "k_sum": k_sum, "union_mean_per_layer": um,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "algorithmic_bytes_per_launch": abytes}}


def mask_variant(ev, gen, torch, P, Q, n, cost, ids8, M, stream, reps):
    """Same trees with routing re-encoded as one-hot expert masks (16 B per node-layer):
    the union becomes a pure OR stream."""
    masks = gen.ids_to_mask_cuda(ids8, N_EXPERTS)
    call = ev.FusedCall(P, Q, cost, masks, N_EXPERTS, n_nodes=n)
    ms = time_fused(ev, torch, call, stream, reps)
    k_sum = int(call.buffers.t["k_star"].sum())
    n_sum = int(n.sum())
    abytes, parts = algorithmic_bytes(n_sum, k_sum, M, 8, id_format="mask")
    peak, _ = hbm_peak()
    ach = abytes / (ms / 1e3) / 1e9
    del call, masks
    torch.cuda.empty_cache()
    return {"id_format": "mask", "value": M / (ms / 1e3), "unit": "trees/s", "kernel_ms": ms,
            "k_sum": k_sum, "n_sum": n_sum,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "algorithmic_bytes_per_launch": abytes}}


def policy_variants(ev, torch, P, Q, n, cost, ids8, M, stream, reps):
    """NEXT-2: the same C5 sweep (select + build + union, u8 routing) cut by the score-coverage
    rule (rho = 1 is EAGLE-3) and by a fixed k: throughput, mean k* and the
    HBM roofline of each (the union reads k*·384 B per tree, so the cut moves the bytes)."""
    out = {}
    peak, _ = hbm_peak()
    for name, pol in (("coverage_0.7", ("coverage", 0.7)), ("coverage_0.4", ("coverage", 0.4)),
                      ("eagle3_rho_1", ("coverage", 1.0)), ("fixed_8", ("fixed", 8))):
        call = ev.FusedCall(P, Q, cost, ids8, N_EXPERTS, n_nodes=n, policy=pol)
        ms = time_fused(ev, torch, call, stream, reps)
        k_sum = int(call.buffers.t["k_star"].sum())
        abytes, _ = algorithmic_bytes(int(n.sum()), k_sum, M, 1, id_format="u8")
        ach = abytes / (ms / 1e3) / 1e9
        out[name] = {"value": M / (ms / 1e3), "unit": "trees/s", "kernel_ms": ms, "mean_k": k_sum / M,
                     "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                                  "frac": ach / peak}}
        del call
    torch.cuda.empty_cache()
    return out


def union_curve_bench(ev, torch, P, Q, n, cost, ids8, M, stream, reps=3):
    """NEXT-1 on the C5 sweep: the prefix-union curve of every tree along its ranking reads
    every node's routing (N·L·K = 23 KB per tree, not k*·384 B), plus the order row in and the
    curve out (4N B each): the roofline is HBM."""
    sel = ev.evict_select(P, Q, cost, n_nodes=n, with_order=True)
    order = sel["order"]
    del sel["prefix_sums"]
    for _ in range(2):
        ev.evict_union_curve(order, ids8, N_EXPERTS, n_nodes=n, stream=stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        g = ev.evict_union_curve(order, ids8, N_EXPERTS, n_nodes=n, stream=stream)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    Nn = order.shape[1]
    byt = float(n.sum()) * L_LAYERS * TOP_K + M * Nn * 4 * 2 + M * 4
    peak, _ = hbm_peak()
    ach = byt / (ms / 1e3) / 1e9
    res = {"value": M / (ms / 1e3), "unit": "trees/s", "kernel_ms": ms,
           "mean_curve_at_n": float(g["curve"].max(dim=1).values.float().mean()),
           "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                        "algorithmic_bytes_per_launch": byt}}
    del order, g
    torch.cuda.empty_cache()
    return res


def verify_bench(ev, gen, torch, stream):
    """NEXT-3: Eq. 3 tree sampling (and greedy T = 0) on the verify side, Qwen3 vocabulary
    V = 151936.  Trees: the C2 generator (60 nodes), keep = Eq. 10 (evict_select), packed
    verify tree from evict_build_verify_tree, target rows from gen/verify.py (64 distinct
    trees; the 1024-tree batch repeats them 16× in HBM so every tree reads its own rows).
    Algorithmic bytes per tree: sampling = the bonus row (4V) + k gathers + uniforms/links;
    greedy = accept_len rows (4V each).  Batch 1024 moves ≥ 620 MB ≫ L2; the batch-64
    latency flushes L2 (256 MB write) before every timed launch."""
    import numpy as np
    from gen import verify as gv
    V = gv.QWEN3_VOCAB
    B0, Nn, rep = 64, 60, 16
    P, Q, n = gen.trees(21, B0, Nn, 6, 10)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    sel = ev.evict_select(cu(P), cu(Q), cu(gen.cost_table(Nn)), n_nodes=cu(n))
    vt = ev.evict_build_verify_tree(cu(P), sel["keep_bits"], n_nodes=cu(n))
    off = vt["verify_offsets"].cpu().numpy()
    T0 = int(off[-1])
    kept = vt["kept_index"][:T0].cpu().numpy()
    tok = gv.draft_tokens(21, P, V, n_nodes=n)
    rows = cu(gv.target_rows(21, P, Q, tok, np.repeat(np.arange(B0), np.diff(off)), kept, V, n_nodes=n))
    ua, ub = gv.uniforms(21, B0 * rep, Nn)
    B = B0 * rep
    # 16 copies of the batch: offsets shift by T0 per copy, retrieve_index by B0·N per copy
    offs = np.concatenate([off[:-1] + r * T0 for r in range(rep)] + [[rep * T0]]).astype(np.int32)
    nt = vt["next_token"][:T0].repeat(rep)
    ns = vt["next_sibling"][:T0].repeat(rep)
    ri = torch.cat([vt["retrieve_index"][:T0] + r * B0 * Nn for r in range(rep)])
    probs = rows.repeat(rep, 1)
    tokb = cu(np.tile(tok, (rep, 1)))
    args = (cu(offs), nt.contiguous(), ns.contiguous(), ri.contiguous(), tokb, probs)
    uA, uB = cu(ua.view(np.int32)), cu(ub.view(np.int32))
    peak, _ = hbm_peak()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {"vocab": V, "trees": B, "rows": rep * T0, "probs_bytes": int(probs.numel() * 4)}
    for mode in ("sample", "greedy"):
        greedy = mode == "greedy"
        call = lambda: ev.evict_verify_sample(*args, u_accept=uA, u_bonus=uB, greedy=greedy,  # noqa: E731
                                              stream=stream)
        for _ in range(3):
            g = call()
        reps = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            g = call()
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        alen = g["accept_len"].double()
        assert int((g["status"] != 0).sum()) == 0
        rows_read = float(B) if not greedy else float(alen.sum())
        k_sum = float(np.diff(offs).sum())
        byt = rows_read * V * 4 + k_sum * 4 * 5 + B * (Nn * 4 + 4 * 4 + 8)
        ach = byt / (ms / 1e3) / 1e9
        # batch-64 latency, cold L2, through the first 64 trees
        a64 = (args[0][:B0 + 1].contiguous(), *args[1:4], tokb[:B0].contiguous(), probs)
        lat = []
        for _ in range(10):
            flush.fill_(1)
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            ev.evict_verify_sample(*a64, u_accept=uA[:B0], u_bonus=uB[:B0], greedy=greedy, stream=stream)
            f1.record(stream)
            f1.synchronize()
            lat.append(f0.elapsed_time(f1) * 1e3)
        res[mode] = {"value": B / (ms / 1e3), "unit": "trees/s", "kernel_ms": ms,
                     "mean_accept_len": float(alen.mean()),
                     "b64_cold_us": float(np.median(lat)),
                     "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                                  "frac": ach / peak, "algorithmic_bytes_per_launch": byt}}
    del probs, rows, flush
    torch.cuda.empty_cache()
    return res


def dispatch_bench(ev, gen, torch):
    """NEXT-4: one decoding step's selection → verify hand-off.  device: ONE graph launch
    [captured fused EVICT step on a batch of 64 C2 trees] → k_dispatch → SWITCH over 10 verify
    bodies (each a stand-in memset).  host (the paper's dispatch): replay the
    captured EVICT step, read verify_offsets[B] to the host (sync), replay the chosen body.
    µs per step, wall clock over 200 steps after warm-up, stream-synchronised at the end."""
    import time
    import numpy as np
    B, N, L, E, K = 64, 60, 48, 128, 8
    P, Q, n = gen.trees(2, B, N, 6, 10)
    ids = gen.routing(2, B, N, L, E, K)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    s = torch.cuda.Stream()
    lengths = [64, 128, 256, 384, 512, 640, 768, 1024, 2048, 3840]
    marker = torch.zeros(1, dtype=torch.int32, device="cuda")
    chosen = torch.zeros(1, dtype=torch.int32, device="cuda")

    def cap(fn):
        g = torch.cuda.CUDAGraph(keep_graph=True)
        with torch.cuda.graph(g, stream=s):
            fn()
        g.instantiate()
        return g

    with torch.cuda.stream(s):
        call = ev.FusedCall(cu(P), cu(Q), cu(gen.cost_table(N)), cu(ids), E, n_nodes=cu(n))
        call(s)
        pre = cap(lambda: call(s))
        rows = call.buffers.t["verify_offsets"][B:]
        bodies = [cap(lambda i=i: marker.fill_(i)) for i in range(len(lengths))]
    d = ev.VerifyDispatch(lengths, bodies, rows, chosen, pre=pre)
    R = 200
    for _ in range(20):
        d.launch(s)
    s.synchronize()
    t0 = time.perf_counter()
    for _ in range(R):
        d.launch(s)
    s.synchronize()
    dev_us = (time.perf_counter() - t0) / R * 1e6
    with torch.cuda.stream(s):
        for _ in range(20):
            pre.replay()
            T = int(rows.item())
            bodies[next(i for i, x in enumerate(lengths) if x >= T)].replay()
        s.synchronize()
        t0 = time.perf_counter()
        for _ in range(R):
            pre.replay()
            T = int(rows.item())
            bodies[next(i for i, x in enumerate(lengths) if x >= T)].replay()
        s.synchronize()
    host_us = (time.perf_counter() - t0) / R * 1e6
    res = {"batch": B, "verify_rows": int(rows.item()), "body": int(chosen.item()),
           "device_dispatch_us_per_step": dev_us, "host_dispatch_us_per_step": host_us,
           "timing": "host wall clock over 200 back-to-back steps (device: graph launches, no sync per step)"}
    d.close()
    return res


def draft_bench(ev, torch, stream):
    """NEXT-4 (P2): draft-tree builder on EAGLE-3-shaped drafter tables (steps 6, topk 10,
    budget 60 — the C2/C5 trees).  Algorithmic bytes per tree: table in steps·topk²·8 B
    (tokens + probs, 4.8 KB) + rows out 12·N + 8 B.  65,536 trees (315 MB ≫ L2) for throughput;
    batch-64 latency by CUDA events (inputs L2-resident after the first call)."""
    import numpy as np
    from gen.draft import drafter_tables
    steps, topk, N = 6, 10, 60
    res = {}
    for name, B in (("b64", 64), ("b65536", 65536)):
        tok, pr = drafter_tables(13, B, steps, topk)
        t, p = torch.from_numpy(tok).cuda(), torch.from_numpy(pr).cuda()
        out = ev.evict_build_draft_tree(t, p, N, stream=stream)
        reps = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            ev.evict_build_draft_tree(t, p, N, out=out, stream=stream)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        byt = B * (steps * topk * topk * 8 + 12 * N + 8)
        peak, _ = hbm_peak()
        ach = byt / (ms / 1e3) / 1e9
        res[name] = {"trees": B, "us": ms * 1e3, "trees_per_s": B / (ms / 1e3),
                     "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak},
                     "note": "issue-bound, not HBM-bound: warp-per-tree kernel (batch >= 4 SMs) ~12K warp "
                             "instructions per tree (profiles/r01_draft_v4_ncu.md); CTA-per-tree below that"}
        del t, p, out
    torch.cuda.empty_cache()
    return res


def router_bench(ev, gen, torch, stream):
    """A8: router logits GEMM (tcgen05) + TopK + union on the C2/C3/C4 shapes and
    the Ling-flash-2.0 shape.  Bytes = L·(T·d + E·d)·2, flops = 2·L·T·d·E with T = packed kept
    rows (Σ k*).  µs per call: median over 100 CUDA-graph replays (memset + router + finalize),
    each after a 256 MB write that evicts the inputs from L2."""
    import numpy as np
    res = {}
    peaks_ = peaks()
    tf_peak = float(peaks_.get("bf16_tflops", 1590.0))
    hbm, _ = hbm_peak()
    for name, B, Nn, steps, topk, L, d, E in (("c2", 1, 60, 6, 10, 48, 2048, 128),
                                               ("c3_b16", 16, 60, 6, 10, 94, 4096, 128),
                                               ("c4", 64, 128, 8, 10, 48, 2048, 128),
                                               ("ling_b1", 1, 60, 6, 10, 32, 4096, 256),
                                               ("ling_b16", 16, 60, 6, 10, 32, 4096, 256)):
        P, Q, n = gen.trees(3, B, Nn, steps, topk)
        cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        sel = ev.evict_select(cu(P), cu(Q), cu(gen.cost_table(Nn)), n_nodes=cu(n))
        b = ev.evict_build_verify_tree(cu(P), sel["keep_bits"], n_nodes=cu(n))
        h = gen.hidden_cuda(11, B, Nn, L, d, mode=1)
        w = gen.wgate_cuda(12, L, E, d, mode=1, scale_log2=-5)
        T = int(b["verify_offsets"][-1])
        rc = ev.RouterCall(b["verify_offsets"], b["retrieve_index"], h, w, TOP_K, B, Nn, max_rows=T)
        gs = torch.cuda.Stream()
        with torch.cuda.stream(gs):
            for _ in range(3):
                rc(gs)
            gs.synchronize()
            # the call (bitset clear + router + finalize) captured once, as in a serving graph
            # (PAPER.md:198-204); replays are timed, so launch gaps are not counted
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=gs):
                rc(gs)
            for _ in range(5):
                graph.replay()
        # cold L2: W_g + the kept hidden rows (25–95 MB) would otherwise stay resident in the
        # 126 MB L2 across replays; a 256 MB write evicts them before every timed replay
        reps = 100
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda.synchronize()
        with torch.cuda.stream(gs):
            for a, c in evs:
                flush.fill_(1)
                torch.cuda.nvtx.range_push(f"evict.router.{name}")
                a.record(gs)
                graph.replay()
                c.record(gs)
                torch.cuda.nvtx.range_pop()
        gs.synchronize()
        us = float(np.median([a.elapsed_time(c) for a, c in evs])) * 1e3
        del flush
        byt = L * (T * d + E * d) * 2
        fl = 2.0 * L * T * d * E
        res[name] = {"B": B, "N": Nn, "L": L, "d": d, "E": E, "rows": T, "us": us,
                     "gbs": byt / (us / 1e6) / 1e9, "hbm_frac": byt / (us / 1e6) / 1e9 / hbm,
                     "tflops": fl / (us / 1e6) / 1e12, "tensor_frac": fl / (us / 1e6) / 1e12 / tf_peak,
                     "bound": f"hbm (intensity <= E = {E} flop/B; ridge 220)"}
        del h, w
    torch.cuda.empty_cache()
    return res


def make_shard(args, ev, gen, torch, dev, base, M):
    """Device-resident inputs of tree ids [base, base + M) (generation excluded from timing)."""
    P, Q, n = gen.trees_cuda(SEED, M, N_NODES, STEPS, TOPK, tree_base=base)
    cost = torch.from_numpy(gen.cost_table(N_NODES)).to(dev)
    ids8 = gen.routing_cuda(SEED, M, N_NODES, L_LAYERS, N_EXPERTS, TOP_K, tree_base=base)
    if args.id_format == "u8":
        ids, id_bytes = ids8, 1
    elif args.id_format == "i32":
        ids, id_bytes = ids8.to(torch.int32), 4
        del ids8
    else:
        ids, id_bytes = gen.ids_to_mask_cuda(ids8, N_EXPERTS), 8
        del ids8
    torch.cuda.synchronize()
    return P, Q, n, cost, ids, id_bytes


def timed_sweep(args, ev, torch, dist, dev, stream, P, Q, n, cost, ids, M, world, local_rank, K, W):
    """W warm-up + K timed steps (one fused A1–A7 + A9 launch: the statistics are accumulated
    inside it; then the NCCL all-reduce of the statistics) between barrier + synchronize; CUDA
    events on the launching stream; max over ranks."""
    from paper_2605_00342_b200.dist import allreduce_stats, max_over_ranks
    call = ev.FusedCall(P, Q, cost, ids, N_EXPERTS, n_nodes=n, with_stats=True)
    bufs = call.buffers.t
    stats_t, dstats_t = bufs["stats"], bufs["dstats"]

    def step(ev0=None, ev1=None):
        # NVTX ranges: the fused A1–A7 (+ A9) call and the statistics all-reduce, for nsys
        torch.cuda.nvtx.range_push("evict.fused_step")
        if ev0 is not None:
            ev0.record(stream)
        call(stream)
        if ev1 is not None:
            ev1.record(stream)
        torch.cuda.nvtx.range_pop()
        torch.cuda.nvtx.range_push("evict.stats_allreduce")
        allreduce_stats(stats_t, dstats_t)
        torch.cuda.nvtx.range_pop()

    for _ in range(max(3, W)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local_rank)
    clk.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk.region(True)
    t0.record(stream)
    for i in range(K):
        step(*evs[i])
    t1.record(stream)
    torch.cuda.synchronize()
    clk.region(False)
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    elapsed_ms = t0.elapsed_time(t1)
    kern_ms = sum(a.elapsed_time(b) for a, b in evs) / K
    tm = max_over_ranks(torch.tensor([elapsed_ms, kern_ms], dtype=torch.float64, device=dev))
    reduced = stats_t.cpu().numpy()
    # single-rank stats of this shard (the all-reduced vector sums every rank): one more call
    call(stream)
    torch.cuda.synchronize()
    return dict(elapsed_ms=float(tm[0]), kern_ms=float(tm[1]), clocks=clocks, bufs=bufs,
                stats=reduced, local=stats_t.cpu().numpy())


def run_native(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import gen
    import paper_2605_00342_b200 as ev
    from paper_2605_00342_b200.dist import shard

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ev.lib()
    if args.scaling == "strong":
        base, M = shard(rank, world, 0, total=args.trees)
        total = args.trees
    else:
        base, M = shard(rank, world, args.trees)
        total = args.trees * world
    P, Q, n, cost, ids, id_bytes = make_shard(args, ev, gen, torch, dev, base, M)
    stream = torch.cuda.current_stream()
    K = args.steps
    sw = timed_sweep(args, ev, torch, dist, dev, stream, P, Q, n, cost, ids, M, world, local_rank, K,
                     args.warmup)
    elapsed_ms, kern_ms, st, lst = sw["elapsed_ms"], sw["kern_ms"], sw["stats"], sw["local"]
    bufs = sw["bufs"]
    value = total * K / (elapsed_ms / 1e3)
    abytes, parts = algorithmic_bytes(int(lst[2]), int(lst[1]), M, id_bytes,
                                      id_format=args.id_format)
    peak, peak_kind = hbm_peak()
    achieved = abytes / (kern_ms / 1e3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"fused_{args.id_format}_{M}")
        except Exception:
            traffic = None
    result = {
        "metric": METRIC, "value": value, "unit": "trees/s", "n_gpus": world, "steps": K,
        "warmup": max(3, args.warmup), "ms_per_step": elapsed_ms / K, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args, world, M, total),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": ("evict_select_build_union: k_select_g (A1-A5 + chunk sums) -> k_scan_offsets -> "
                                "k_fused PRE (A6 + A7 + folded A9); one call = the whole path"
                                if M > 2048 and args.id_format == "u8" else "k_fused (A1-A7 + A9)"),
                     "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": abytes, "bytes_split": parts,
                     "kernel_ms": kern_ms},
        "union_hbm_gbs": parts["union"] / (kern_ms / 1e3) / 1e9,
        "gpu_launches": (3 if M > 2048 and args.id_format == "u8" else 1) * K,
        "k_star_mean": float(lst[1]) / max(1, M - int(lst[4])),
        "union_mean_per_layer": float(lst[3]) / max(1, (M - int(lst[4])) * L_LAYERS),
        "stats_allreduced_trees": int(st[0]),
        "shard": {"rank0_tree_ids": [base, base + M], "collective": "NCCL all_reduce(SUM) of the "
                  "A9 stats vector + all_reduce(MAX) of the elapsed time" if world > 1 else None},
        "clocks": sw["clocks"],
    }
    if world > 1 and not args.no_extras and args.scaling == "strong":
        # weak scaling beside the headline: 1M trees per rank (tree ids [r·1M, (r+1)·1M))
        wb, wM = shard(rank, world, args.trees)
        wP, wQ, wn, wc, wi, _ = make_shard(args, ev, gen, torch, dev, wb, wM)
        ws = timed_sweep(args, ev, torch, dist, dev, stream, wP, wQ, wn, wc, wi, wM, world, local_rank,
                         K, args.warmup)
        result["weak_scaling"] = {"value": wM * world * K / (ws["elapsed_ms"] / 1e3), "unit": "trees/s",
                                  "trees_per_rank": wM, "ms_per_step": ws["elapsed_ms"] / K,
                                  "kernel_ms": ws["kern_ms"], "stats_allreduced_trees": int(ws["stats"][0])}
        del wP, wQ, wn, wc, wi, ws
        torch.cuda.empty_cache()
    # ---- end-to-end through the public API with host buffers (rank-local)
    result["e2e"] = e2e(args, ev, torch, P, Q, n, cost, ids, M, world, stream)
    if not args.no_extras and args.id_format == "u8":
        try:
            result["variants"] = {"mask": mask_variant(ev, gen, torch, P, Q, n, cost, ids, M, stream,
                                                       max(3, K // 2))}
        except Exception as e:  # pragma: no cover
            result["variants"] = {"mask": {"error": repr(e)}}
        try:
            result["variants"]["ling"] = ling_variant(ev, gen, torch, P, Q, n, cost, M, stream, max(3, K // 2))
        except Exception as e:  # pragma: no cover
            result["variants"]["ling"] = {"error": repr(e)}
        try:
            result["policies"] = policy_variants(ev, torch, P, Q, n, cost, ids, M, stream, max(3, K // 2))
        except Exception as e:  # pragma: no cover
            result["policies"] = {"error": repr(e)}
        try:
            result["union_curve"] = union_curve_bench(ev, torch, P, Q, n, cost, ids, M, stream)
        except Exception as e:  # pragma: no cover
            result["union_curve"] = {"error": repr(e)}
    if rank == 0 and not args.no_extras:
        try:
            result["router"] = router_bench(ev, gen, torch, stream)
        except Exception as e:  # pragma: no cover
            result["router"] = {"error": repr(e)}
        try:
            result["draft_tree"] = draft_bench(ev, torch, stream)
        except Exception as e:  # pragma: no cover
            result["draft_tree"] = {"error": repr(e)}
        try:
            result["dispatch"] = dispatch_bench(ev, gen, torch)
        except Exception as e:  # pragma: no cover
            result["dispatch"] = {"error": repr(e)}
        try:
            result["verify"] = verify_bench(ev, gen, torch, stream)
        except Exception as e:  # pragma: no cover
            result["verify"] = {"error": repr(e)}
        try:
            lat = {}
            for B, N, steps, topk in ((64, 60, 6, 10), (1, 60, 6, 10), (64, 128, 8, 10)):
                lat.update(latency(ev, torch, gen, B=B, N=N, steps=steps, topk=topk))
            result["latency"] = lat
        except Exception as e:  # pragma: no cover
            result["latency"] = {"error": repr(e)}
    if rank == 0:
        # the oracle leg: timed on a bounded sample of rank 0's shard, and its outputs compared with
        # the GPU's for the same trees (outside every timed region)
        S_par = min(M, 20_000)
        gpu_out = {k: bufs[k][:S_par].cpu().numpy() for k in ("k_star", "e_hat", "utility", "keep_bits",
                                                             "union_count", "union_total", "status")}
        result["cpu_baseline"] = cpu_baseline(args, result["k_star_mean"], gpu_out, base)
        print(json.dumps(result), flush=True)
    return 0


def e2e(args, ev, torch, P, Q, n, cost, ids, M, world, stream):
    """Same metric through the public API with the inputs in pinned host memory, every step:
    parent / q / n_nodes are copied H2D (480 B per tree, chunked, double-buffered on two
    streams), the routing table stays in page-locked host memory mapped into the device address
    space and the fused call reads only the kept nodes' rows over PCIe (zero-copy: k*·L·K bytes
    per tree, not the 23 KB row block of every node), and the per-tree results (k*, e_hat,
    utility, keep_bits, union_total, status) are read back D2H."""
    import numpy as np
    # host-memory guard: pinned copies of the inputs must fit comfortably
    per_tree = (P[0].numel() * 4 + Q[0].numel() * 4 + 4 + ids[0].numel() * ids.element_size() + 64)
    try:
        avail = int([l for l in open("/proc/meminfo") if l.startswith("MemAvailable")][0].split()[1]) * 1024
    except Exception:
        avail = 0
    if avail and per_tree * M > 0.35 * avail:
        M = max(1 << 16, int(0.35 * avail / per_tree) // (1 << 16) * (1 << 16))
        P, Q, n, ids = P[:M], Q[:M], n[:M], ids[:M]
    try:
        hP = torch.empty(P.shape, dtype=P.dtype, pin_memory=True)
        hQ = torch.empty(Q.shape, dtype=Q.dtype, pin_memory=True)
        hn = torch.empty(n.shape, dtype=n.dtype, pin_memory=True)
        hI = torch.empty(ids.shape, dtype=ids.dtype, pin_memory=True)
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "trees/s", "error": f"pinned alloc failed: {e!r}"}
    hP.copy_(P); hQ.copy_(Q); hn.copy_(n); hI.copy_(ids)
    chunk = 1 << 16
    nch = (M + chunk - 1) // chunk
    dev = P.device
    cp = [torch.cuda.Stream() for _ in range(2)]
    dP = [torch.empty((chunk,) + tuple(P.shape[1:]), dtype=P.dtype, device=dev) for _ in range(2)]
    dQ = [torch.empty((chunk,) + tuple(Q.shape[1:]), dtype=Q.dtype, device=dev) for _ in range(2)]
    dn = [torch.empty((chunk,), dtype=n.dtype, device=dev) for _ in range(2)]
    res_k = torch.empty(M, dtype=torch.int32, pin_memory=True)
    res_e = torch.empty(M, dtype=torch.float32, pin_memory=True)
    res_u = torch.empty(M, dtype=torch.float32, pin_memory=True)
    res_b = torch.empty((M, 1), dtype=torch.int64, pin_memory=True)
    res_t = torch.empty(M, dtype=torch.int32, pin_memory=True)
    res_s = torch.empty(M, dtype=torch.int32, pin_memory=True)
    bufs = [ev.FusedBuffers(chunk, N_NODES, L_LAYERS, N_EXPERTS, dev) for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    h2d = d2h = 0

    def one_step():
        nonlocal h2d, d2h
        h2d = d2h = 0
        for c in range(nch):
            j = c & 1
            lo, hi = c * chunk, min(M, (c + 1) * chunk)
            m = hi - lo
            s = cp[j]
            s.wait_event(done[j])
            with torch.cuda.stream(s):
                dP[j][:m].copy_(hP[lo:hi], non_blocking=True)
                dQ[j][:m].copy_(hQ[lo:hi], non_blocking=True)
                dn[j][:m].copy_(hn[lo:hi], non_blocking=True)
                h2d += dP[j][:m].numel() * 4 + dQ[j][:m].numel() * 4 + m * 4
                t = ev.evict_select_build_union(dP[j][:m], dQ[j][:m], cost, hI[lo:hi], N_EXPERTS,
                                                n_nodes=dn[j][:m], buffers=_slice_bufs(bufs[j], m, ev),
                                                stream=s)
                res_k[lo:hi].copy_(t["k_star"][:m], non_blocking=True)
                res_e[lo:hi].copy_(t["e_hat"][:m], non_blocking=True)
                res_u[lo:hi].copy_(t["utility"][:m], non_blocking=True)
                res_b[lo:hi].copy_(t["keep_bits"][:m], non_blocking=True)
                res_t[lo:hi].copy_(t["union_total"][:m], non_blocking=True)
                res_s[lo:hi].copy_(t["status"][:m], non_blocking=True)
                d2h += m * 28
                done[j].record(s)
        for s in cp:
            s.synchronize()

    one_step()
    torch.cuda.synchronize()
    # the routing rows the kernel pulls over PCIe: k* rows of L·K ids per tree
    kept_row_bytes = int(res_k.numpy().astype(np.int64).sum()) * L_LAYERS * TOP_K * ids.element_size()
    K = max(1, args.e2e_steps)
    t0 = time.perf_counter()
    for _ in range(K):
        one_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / K
    v = M * world / dt
    ok = int((res_k.numpy() > 0).sum())
    return {"value": v, "unit": "trees/s", "h2d_bytes_per_step": h2d + kept_row_bytes,
            "d2h_bytes_per_step": d2h, "h2d_copied_bytes": h2d, "h2d_zero_copy_bytes": kept_row_bytes,
            "ms_per_step": dt * 1e3, "chunk_trees": chunk, "trees_with_result": ok,
            "trees_per_rank": M, "host_mem_available_gb": avail / 1e9,
            "routing": "pinned host memory mapped into the device address space; kept rows read "
                       "by the kernel over PCIe",
            "timing": "host wall clock around fully synchronised steps (pinned H2D/D2H included)"}


def _slice_bufs(b, m, ev):
    """View the first m trees of pre-allocated FusedBuffers (batch shrinks on the last chunk)."""
    if m == b.t["k_star"].shape[0]:
        return b
    class _V:  # noqa: N801
        pass
    v = _V()
    v.t = {k: (t[:m] if k not in ("verify_offsets",) else t[:m + 1]) for k, t in b.t.items()}
    v.workspace = b.workspace
    v.struct = lambda pos_offset=None: ev._FusedOut(**{f: ev._p(v.t.get(f)) for f in ev._OUT_FIELDS})
    return v


def spawn(args):
    """`--gpus N` outside torchrun: re-execute this script under torch.distributed.run with N local
    ranks (the driver's own launch line); rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    if not args.dry_run:
        # communicator init lines (comm_nranks) in the log, so the world size is checkable
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


def dry_run(args, rank, world):
    """CPU check of the multi-rank plumbing (gloo): every rank takes its shard of the tree ids,
    the per-rank counters are summed by all_reduce and the elapsed time max-reduced, exactly the
    collectives of the GPU step.  No kernels run; the line says so."""
    import torch
    import torch.distributed as dist
    from paper_2605_00342_b200.dist import allreduce_stats, max_over_ranks, shard
    if args.scaling == "strong":
        base, M = shard(rank, world, 0, total=args.trees)
    else:
        base, M = shard(rank, world, args.trees)
    ids = torch.arange(base, base + M, dtype=torch.int64)
    st = torch.tensor([M, int(ids.sum()), int((ids * ids).sum())], dtype=torch.int64)
    dst = torch.tensor([float(M), 0.0], dtype=torch.float64)
    t0 = time.perf_counter()
    allreduce_stats(st, dst)
    el = max_over_ranks(torch.tensor([time.perf_counter() - t0], dtype=torch.float64))
    shards = [None] * world
    if world > 1:
        dist.all_gather_object(shards, [base, M])
    else:
        shards = [[base, M]]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "scaling": args.scaling,
                          "backend": dist.get_backend() if world > 1 else None,
                          "shards": shards, "trees": int(st[0]), "id_sum": int(st[1]),
                          "id_sq_sum": int(st[2]), "elapsed_s": float(el[0]),
                          "config": config_dict(args, world, M)}), flush=True)
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus and rank == 0:
        print(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}; reporting n_gpus={world}", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    import torch
    import torch.distributed as dist
    if args.dry_run:
        if world > 1:
            dist.init_process_group("gloo")
        try:
            return dry_run(args, rank, world)
        finally:
            if world > 1:
                dist.destroy_process_group()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        print(f"bench: rank {rank}/{world} on cuda:{local_rank}, backend {dist.get_backend()}, "
              f"comm_nranks {dist.get_world_size()}", file=sys.stderr, flush=True)
    try:
        return run_native(args, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
