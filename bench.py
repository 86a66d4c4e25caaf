#!/usr/bin/env python
"""bench.py -- the driver contract for the ConnectIt connectivity hot path on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

A step is one cc_labels call (H1-H6: init, k-out sampling, IdentifyFrequent,
finish, compress) on the resident synthetic graph of BASELINE.json config
`--config` (default 4 = RMAT scale 27, configs[3]; the metric names no config,
so the largest single-GPU one is the workload).  `value` is GTEPS =
directed edges / second summed over ranks (each rank runs an independent
replica: the north_star path is one GPU, "replicas only").
`--config 5` times the incremental stream (256 batches) instead, in Gops/s.

Prints ONE JSON line on rank 0 (see DESIGN.md §Measurement for every key).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CPU_SAMPLE_SCALE = 24            # oracle sample: RMAT scale 24, same a/b/c/d and seed as C4
CPU_BASELINE_MIN_S = 10.0        # repeat the oracle sample until this much CPU time has been spent
HBM_FALLBACK_GBS = 6650.0        # B200_PROFILING.md fallback if MEASURED_PEAKS.json is absent
CONTRACT_GBS = 8000.0            # BASELINE.json bar: % of 8 TB/s


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--k", type=int, default=2)
    p.add_argument("--variant", default="afforest", choices=["afforest", "hybrid", "pure"])
    p.add_argument("--flags", type=int, default=0)
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-scale", type=int, default=CPU_SAMPLE_SCALE)
    p.add_argument("--cpu-batches", type=int, default=256, help="C5: batches the oracle replays for cpu_baseline")
    p.add_argument("--l2-fetch", type=int, default=-1, help="cudaLimitMaxL2FetchGranularity (bytes) or -1")
    p.add_argument("--study", action="store_true", help="NEXT-1 sampling variant x k sweep on C2-C4")
    p.add_argument("--incr-sweep", action="store_true", help="NEXT-2 incremental variants sweep")
    p.add_argument("--amsf", action="store_true", help="NEXT-4 AMSF-NF-S study on C3/C4 with Exp(1) weights")
    p.add_argument("--table4", action="store_true", help="NEXT-2(b): Table 4 insert-only protocol, RM stream")
    p.add_argument("--eps", type=float, default=0.25)
    p.add_argument("--graph", action="store_true",
                   help="time cc_labels captured once into a CUDA graph and replayed (launch-bound configs: C1)")
    return p.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing (replicas: the only collectives are barrier + max of the timings)
def dist_setup():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return rank, ws


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def reduce_max(x: float, ws: int) -> float:
    """Max over ranks (device-timed numbers are aggregated as the max, never wall clock)."""
    if ws == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_value(units_per_rank: float, max_seconds: float, ws: int) -> float:
    """Whole-job throughput: units all ranks processed / the slowest rank's time."""
    return units_per_rank * ws / max_seconds


# ---------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "25"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # nvidia-smi takes ~1 s to start: wait for its first row so that a short
        # timed region (20 steps of ~3 ms) is covered by samples
        t0 = time.time()
        while time.time() - t0 < 10:
            self.f.flush()
            if os.path.getsize(self.f.name) > 0:
                break
            time.sleep(0.05)
        self.skip = open(self.f.name).read().count("\n")    # rows sampled before the timed region

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.03)
        self.proc.terminate()
        self.proc.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines()[getattr(self, "skip", 0):]
                if r.count(",") >= 5]
        os.unlink(self.f.name)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[2 + i] and "Not" not in r[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def peaks():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str, kernel: str):
    """dram read+write bytes per launch of `kernel` from a committed ncu capture (launch list
    with dram__bytes_read.sum / dram__bytes_write.sum, or --set full) of THIS workload (profiles/ncu_traffic.json is keyed by workload, then by
    bench mark name); None when no capture of this workload / kernel exists."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return d.get(workload, {}).get(kernel)
    except Exception:
        return None


# ---------------------------------------------------------------------------
def cpu_oracle_sample(scale: int, use_gpu_gen: bool):
    """Time the oracle (as it stands, 1 thread) on an RMAT-`scale` sample of the C4 recipe."""
    import numpy as np

    import oracle
    from inputs import gen
    if use_gpu_gen:
        from inputs import gpu as ggen
        d_off, d_adj = ggen.rmat(4, scale)
        off = d_off.cpu().numpy()
        adj = d_adj.cpu().numpy().view(np.uint32)
        del d_off, d_adj
    else:
        off, adj = gen.rmat(4, scale)
    t0 = time.perf_counter()
    lab = oracle.cc_bfs(off, adj)
    dt = time.perf_counter() - t0
    return adj.size, dt, off, adj, lab


def run_reference(a, rank, ws):
    """--impl reference: the CPU oracle on the box's host cores (rank 0 only)."""
    if rank != 0:
        return
    import torch
    use_gpu = torch.cuda.is_available()
    import inputs
    cfg = inputs.BY_INDEX[a.config]
    import oracle
    if cfg.kind == "incr":
        return run_reference_incr(a, cfg, use_gpu)
    m, dt0, off_s, adj_s, _ = cpu_oracle_sample(a.cpu_scale, use_gpu)     # sample generated once
    times = []
    for i in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        oracle.cc_bfs(off_s, adj_s)
        dt = time.perf_counter() - t0
        if i >= a.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    value = m / t / 1e9
    sample = f"oracle.cc_bfs (sequential BFS, 1 thread) on RMAT scale {a.cpu_scale} (C4 recipe a/b/c/d=.57/.19/.19/.05, ef 16, seed 4), m={m}"
    # once, outside the K steps: the same oracle on the reported workload itself (one run; the
    # graph comes from the seeded input generator, not from the product)
    full = None
    if not a.no_cpu_baseline:
        try:
            import numpy as np
            import psutil
            if use_gpu and cfg.kind != "incr":
                from inputs import gpu as ggen
                d_off, d_adj = ggen.config_graph(cfg)
                n_f, m_f = d_off.numel() - 1, d_adj.numel()
                if (8 * (n_f + 1) + 4 * m_f + 12 * n_f) * 1.2 < psutil.virtual_memory().available:
                    off_h = d_off.cpu().numpy()
                    adj_h = d_adj.cpu().numpy().view(np.uint32)
                    del d_off, d_adj
                    torch.cuda.empty_cache()
                    t0 = time.perf_counter()
                    oracle.cc_bfs(off_h, adj_h)
                    dt = time.perf_counter() - t0
                    full = {"value": round(m_f / dt / 1e9, 5), "unit": "GTEPS", "seconds": round(dt, 3),
                            "sample": f"oracle.cc_bfs, 1 thread, on {cfg.name} itself (n={n_f}, m={m_f}), one run"}
                    del off_h, adj_h
        except Exception as e:                    # never fail the reference arm over the extra number
            full = {"skipped": str(e)[:200]}
    line = {"impl": "reference", "metric": "connectivity edges/sec (GTEPS)", "value": value, "unit": "GTEPS",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": {"workload": cfg.name, "sample": sample},
            "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if full is not None:
        line["full_workload"] = full
    print(json.dumps(line), flush=True)


def run_reference_incr(a, cfg, use_gpu):
    """--impl reference --config 5: the DSU oracle (oracle.incr_run, 1 thread) replaying the
    first a.cpu_batches // 16 batches of the C5 stream per step (a bounded sample)."""
    import numpy as np

    import oracle
    from inputs import gen
    nbs = max(1, min(cfg.n_batches, a.cpu_batches // 16))
    if use_gpu:
        import torch
        from inputs import gpu as ggen
        bi = torch.empty((cfg.n_ins, 2), dtype=torch.int32, device="cuda")
        bq = torch.empty((cfg.n_q, 2), dtype=torch.int32, device="cuda")
        batches = []
        for b in range(nbs):
            ggen.incr_batch(cfg.seed, cfg.scale, b, cfg.n_ins, cfg.n_q, bi, bq)
            batches.append((bi.cpu().numpy().view(np.uint32).copy(), bq.cpu().numpy().view(np.uint32).copy()))
    else:
        batches = [gen.incr_batch(cfg.seed, cfg.scale, b, cfg.n_ins, cfg.n_q) for b in range(nbs)]
    n = 1 << cfg.scale
    ops = nbs * (cfg.n_ins + cfg.n_q)
    times = []
    for i in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        oracle.incr_run(n, batches)
        dt = time.perf_counter() - t0
        if i >= a.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    value = ops / t / 1e9
    sample = (f"oracle.incr_run (sequential union-find, 1 thread) on the first {nbs} batches of the C5 stream "
              f"({ops} ops) per step")
    line = {"impl": "reference", "metric": "incremental connectivity ops/sec", "value": value, "unit": "Gops/s",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": {"workload": cfg.name, "sample": sample},
            "cpu_baseline": {"value": value, "unit": "Gops/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "Gops/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def byte_model(off_h_deg_pos, n, m, k, ctr, sampled, final, mid_ran, f0=None, partial_h6=True):
    """Algorithmic bytes per launch of each kernel, SURVEY §8(d).

    Counts only what the implemented design must move (§8(d) honesty rule 1):
    4 B per uint32 read/written, 8 B per int64 offset.  First-level parent reads
    of a traversed edge (P[v]) are counted; root checks and walks beyond the
    first parent level (P[P[v]], k_finish's and H6's `*_gathers`) are NOT (§8(d):
    "Path-walk reads beyond the first level ... are not counted").  f0 = (F0
    non-roots, F0 vertices at depth >= 2) selects the contracted-link model;
    partial_h6 selects the partial final compress (k_relabel) over the full pass."""
    import numpy as np
    npos, sum_mink = off_h_deg_pos
    pend = ctr["pending_links"]
    fin_v, fin_e = ctr["finish_vertices"], ctr["finish_edges"]
    ntiles = (n + 2047) // 2048
    relab = int(np.count_nonzero(final != sampled))          # labels that differ from the sampled ones
    nonroot = int(np.count_nonzero(sampled != np.arange(n, dtype=np.uint32)))
    B = {
        # offsets (n+1) + first-k adj entries + P write + pending writes + finish bitmap
        "k_sample_init": 8 * (n + 1) + 4 * sum_mink + 4 * n + 8 * pend + n // 8,
        # probe (1024 walks of <= 8 steps) + when it ran, P read + one first-level parent read per
        # non-isolated vertex (upper bound of the non-roots)
        "k_compress_mid": 1024 * 8 * 4 + (4 * n + 4 * npos if mid_ran else 0),
        # pending read + P[u], P[v] gathers + hook CAS
        "k_link_pending": 8 * pend + 8 * pend + 4 * ctr["sample_hooks"],
        "k_identify": 4 * 1024,
        # fused H3 + H5 scan (B_fin's "4n skip-test read"): P read + degree bitmap (replaces the
        # 8 N_off offsets reads, §8(d) rule 1) + H3 label writes + candidate queue writes +
        # the tile summaries of the partial H6 (16 B + a 1 B hook flag per 2048-slot tile)
        "k_finish": 4 * n + n // 8 + 4 * ctr["compress_writes"] + 4 * fin_v + 17 * ntiles,
        # H5 edge work: queue read + offsets pair + P[u] per candidate, adj + first-level P[v]
        # per traversed edge (B_fin's 8 E_ng) + hook CAS (4 H)
        "k_finish_proc": 4 * fin_v + 16 * fin_v + 4 * fin_v + 8 * fin_e + 4 * ctr["finish_hooks"],
        # H6: partial -- tile summaries + flags read, every slot of a dirty tile re-read,
        # changed labels written; full -- B_fin's "4n compress read" + changed labels
        "k_compress_H6": (17 * ntiles + 8192 * ctr.get("h6_tiles", 0) + 4 * ctr["h6_writes"]) if partial_h6
                         else 4 * n + 4 * ctr["h6_writes"],
    }
    if f0 is not None:
        # contracted link: + the F0-root bitmap words in k_sample_init;
        # the "mid" span is the rank scan (bitmap read twice, prefix words written,
        # rid + C initialised: 8 B per compact slot) and the F0 compress (P read, one
        # parent read per F0 non-root, one write per vertex at depth >= 2); the link
        # span reads the pending pairs and gathers P[u], P[v] (the C-space walk and
        # CAS run on the L2-resident compact array and are not HBM bytes), then
        # finalises C (read C, write rid); k_finish reads a rank word (8 B) and a
        # rid entry (4 B) per non-isolated vertex instead of gathering in P
        R = ctr["contract_roots"]
        f0_nonroots, f0_deep = f0
        B["k_sample_init"] += n // 8
        B["k_compress_mid"] = 3 * (n // 8) + 8 * R + 4 * n + 4 * f0_nonroots + 4 * f0_deep
        B["k_link_pending"] = 16 * pend + 8 * R
        B["k_finish"] = 4 * n + n // 8 + 12 * ctr["finish_gathers"] + 4 * ctr["compress_writes"] + 4 * fin_v + 17 * ntiles
    if ctr.get("fused_link"):
        # k_sample_link (DESIGN.md §6 item 1b): P initialised first (4n write), offsets + first-k
        # adj entries, the round-0 CAS on P[u] (4n read), finish bitmap, and the links queued in
        # shared memory: P[u], P[v] gathers + hook CAS -- no pending list through HBM
        B["k_sample_init"] = 8 * (n + 1) + 4 * sum_mink + 4 * n + 4 * n + n // 8 + 8 * pend + 4 * ctr["sample_hooks"]
        B["k_compress_mid"] = 1024 * 8 * 12
        B["k_link_pending"] = 0
    B["finish_phase"] = B["k_finish"] + B["k_finish_proc"] + B["k_compress_H6"]
    B["sampling_phase"] = B["k_sample_init"] + B["k_compress_mid"] + B["k_link_pending"]
    terms = {"4n_skip_test_read": 4 * n, "bitmap_for_8N_off": n // 8, "8E_ng": 8 * fin_e,
             "candidates_queue_offsets_Pu": 28 * fin_v,
             "4W_label_writes": 4 * (ctr["compress_writes"] + ctr["h6_writes"]), "4H_hooks": 4 * ctr["finish_hooks"],
             "4n_compress_read": 0 if partial_h6 else 4 * n,
             "tile_summaries": (34 if partial_h6 else 17) * ntiles,     # written by k_finish, read by a partial H6
             "dirty_tile_rereads": 8192 * ctr.get("h6_tiles", 0) if partial_h6 else 0}
    return B, {"relabelled": relab, "sampled_nonroots": nonroot, "mid_nonroots_bound": npos, "B_fin_terms": terms,
               "root_check_reads_not_counted": int(ctr["finish_gathers"] + ctr["h6_gathers"])}


def floors(cc, d_off, d_adj, n, m, x, stream, cc_ms, reps=3):
    """MapEdges / GatherEdges on the same CSR, a uniform random 4 B gather over an
    n-sized array and a streaming copy: the empirical floors next to t_CC."""
    import torch

    def timed(fn):
        ts = []
        for _ in range(reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts[1:])
    out = torch.empty(n, dtype=torch.int32, device=d_off.device)
    acc = torch.zeros(1, dtype=torch.int32, device=d_off.device)
    t_map = timed(lambda: cc.map_edges(d_off, d_adj, n, out, stream))
    t_gather = timed(lambda: cc.gather_edges(d_off, d_adj, n, x, out, stream))
    cnt = 1 << 28
    t_rand = timed(lambda: cc.random_gather(x, n, cnt, 7, acc, stream))
    words = (n // 4) * 4
    t_copy = timed(lambda: cc.copy(x, out, words, stream))
    return {"map_edges_ms": round(t_map, 4), "gather_edges_ms": round(t_gather, 4),
            "t_cc_over_t_gather": round(cc_ms / t_gather, 4), "t_cc_over_t_map": round(cc_ms / t_map, 4),
            "random_gather": {"loads": cnt, "array_bytes": 4 * n, "ms": round(t_rand, 4),
                              "Gloads_per_s": round(cnt / (t_rand * 1e-3) / 1e9, 2)},
            "copy_GBps": round(2 * 4 * words / (t_copy * 1e-3) / 1e9, 1)}


def run_ours(a, rank, ws):
    import numpy as np
    import torch

    import inputs
    from inputs import gpu as ggen
    from paper_2008_03909_b200 import cc

    cfg = inputs.BY_INDEX[a.config]
    l2_fetch_prev = cc.set_l2_fetch(a.l2_fetch) if a.l2_fetch >= 0 else None
    if cfg.kind == "incr":
        return run_ours_incr(a, rank, ws, cfg)
    dev = torch.device("cuda", torch.cuda.current_device())
    tg = time.time()
    d_off, d_adj = ggen.config_graph(cfg)
    torch.cuda.synchronize()
    gen_s = time.time() - tg
    n, m = d_off.numel() - 1, d_adj.numel()
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    variant = {"afforest": cc.VARIANT_AFFOREST, "hybrid": cc.VARIANT_HYBRID, "pure": cc.VARIANT_PURE}[a.variant]
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4 + 1024, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def call(marks=None, **kw):
        o = cc.make_opts(k=a.k, variant=variant, flags=a.flags, marks=marks, **kw)
        cc.cc_labels(d_off, d_adj, n, m, labels, o, stream)

    # ---- diagnostics run (untimed): counters + sampled labels for the byte model
    ctr_t = torch.zeros(len(cc.COUNTER_FIELDS), dtype=torch.int64, device=dev)
    sampled_t = torch.empty(n, dtype=torch.int32, device=dev)
    call(counters=ctr_t)              # counters of the production path (H3 fused into k_finish)
    call(sampled_out=sampled_t)       # sampled labels (this debug call runs H3 as its own pass)
    torch.cuda.synchronize()
    ctr = dict(zip(cc.COUNTER_FIELDS, ctr_t.cpu().tolist()))
    sampled = sampled_t.cpu().numpy().view(np.uint32)
    final = labels.cpu().numpy().view(np.uint32)
    deg = torch.diff(d_off)
    sum_mink = int(torch.clamp(deg, max=a.k).sum().item())
    nonisolated = int((deg > 0).sum().item())
    del sampled_t, deg
    # the mid compress runs when forced, or when the device probe found long chains
    mid_ran = a.k > 0 and not (a.flags & cc.FLAG_NO_MIDCOMPRESS) and (
        bool(a.flags & cc.FLAG_MIDCOMPRESS) or bool(ctr.get("mid_compress")))
    contract = a.k > 0 and bool(a.flags & cc.FLAG_CONTRACT) and not (a.flags & cc.FLAG_NO_SKIP)
    f0 = None
    if contract:
        # the round-0 forest F0 (P[u] = first sampled neighbour if smaller), for the byte model
        ids = torch.arange(n, device=dev, dtype=torch.int64)
        if a.variant == "pure":                    # random first pick: bound by the non-isolated count
            nr = nonisolated - ctr["contract_roots"]
            f0 = (nr, nr)
        else:
            first = d_adj[d_off[:-1].clamp(max=max(m - 1, 0))].to(torch.int64) & 0xFFFFFFFF
            p0 = torch.where((torch.diff(d_off) > 0) & (first < ids), first, ids)
            del first
            f0 = (int((p0 != ids).sum().item()), int((p0[p0] != p0).sum().item()))
            del p0
        del ids
        mid_ran = True
    # the partial final compress runs unless an SV / CRFA finish is selected (cc_static.cu run())
    partial_h6 = not (a.flags & (cc.FLAG_FINISH_SV | cc.FLAG_FINISH_CRFA))
    B, extra = byte_model((nonisolated, sum_mink), n, m, a.k, ctr, sampled, final, mid_ran, f0, partial_h6)
    extra["mid_compress_ran"] = mid_ran
    extra["contracted_link"] = contract
    if f0 is not None:
        extra["f0_nonroots"], extra["f0_depth_ge2"] = f0
    components = int(np.count_nonzero(final == np.arange(n, dtype=np.uint32)))

    # ---- warm-up
    for _ in range(a.warmup):
        flush.zero_()
        call()
    torch.cuda.synchronize()
    step = call
    if a.graph:
        # one cc_labels call captured into a CUDA graph (kernels, stream-ordered scratch
        # allocations, programmatic-dependent launches), replayed per step
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        lc0 = cc.launch_count()
        with torch.cuda.graph(graph, stream=gs, capture_error_mode="thread_local"):
            cc.cc_labels(d_off, d_adj, n, m, labels, cc.make_opts(k=a.k, variant=variant, flags=a.flags), gs)
        torch.cuda.synchronize()
        graph_kernels = cc.launch_count() - lc0        # libcc kernels in the captured graph
        step = graph.replay
        for _ in range(a.warmup):
            flush.zero_()
            step()
        torch.cuda.synchronize()

    # ---- timed region: K steps, each bracketed by its own events; L2 flushed between steps
    clk = Clocks(torch.cuda.current_device())
    clk.start()
    marks = [[torch.cuda.Event(enable_timing=True) for _ in range(cc.NUM_MARKS)] for _ in range(a.steps)]
    for row in marks:
        for e in row:
            e.record(stream)          # materialise the lazily created events
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    outer = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    l0 = cc.launch_count()
    for i in range(a.steps):
        flush.zero_()
        outer[i][0].record(stream)
        step()
        outer[i][1].record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    launches = cc.launch_count() - l0
    if a.graph:
        launches = graph_kernels * a.steps          # replays launch the captured kernels on the device
    clocks = clk.stop()
    # per-kernel breakdown: the same K steps again with an event at every kernel boundary
    # (cc_opts.marks; the events serialise the launches, so the step time above is taken
    # without them)
    for i in range(a.steps):
        flush.zero_()
        call(marks=[e.cuda_event for e in marks[i]])
    torch.cuda.synchronize()
    step_ms = [outer[i][0].elapsed_time(outer[i][1]) for i in range(a.steps)]
    marked_ms = [marks[i][0].elapsed_time(marks[i][cc.NUM_MARKS - 1]) for i in range(a.steps)]
    kern_ms = {}
    for j in range(1, cc.NUM_MARKS):
        kern_ms[cc.MARK_NAMES[j]] = statistics.mean(marks[i][j - 1].elapsed_time(marks[i][j]) for i in range(a.steps))
    mean_ms = statistics.mean(step_ms)
    max_ms = reduce_max(mean_ms, ws)
    srt = sorted(step_ms)
    t_stats = {"mean": round(mean_ms, 5), "median": round(statistics.median(step_ms), 5), "min": round(srt[0], 5),
               "p90": round(srt[min(len(srt) - 1, int(0.9 * len(srt)))], 5), "max": round(srt[-1], 5)}
    value = aggregate_value(m, max_ms * 1e-3, ws) / 1e9

    peak, peak_src = peaks()
    kernels = {}
    for kname, t in kern_ms.items():
        if kname in B and t > 0:
            gbs = B[kname] / (t * 1e-3) / 1e9
            kernels[kname] = {"ms": round(t, 5), "bytes": int(B[kname]), "GB/s": round(gbs, 1),
                              "frac": round(gbs / peak, 4), "share": round(t / mean_ms, 4)}
    if ctr.get("fused_link") and "k_sample_init" in kernels:
        kernels["k_sample_link"] = kernels.pop("k_sample_init")      # sampling + k-out links, one kernel
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    dk = kernels[dom]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": dk["GB/s"], "peak": peak, "unit": "GB/s",
                "frac": dk["frac"], "traffic": ncu_traffic(cfg.name, dom), "peak_source": peak_src,
                "algorithmic_bytes_per_launch": dk["bytes"], "launch_ms": dk["ms"]}
    fin_ms = kern_ms["k_finish"] + kern_ms["k_finish_proc"] + kern_ms["k_compress_H6"]
    fin_gbs = B["finish_phase"] / (fin_ms * 1e-3) / 1e9
    smp_ms = sum(kern_ms[x] for x in ("k_sample_init", "k_compress_mid", "k_link_pending"))
    t_fin_ms = [sum(marks[i][j - 1].elapsed_time(marks[i][j]) for j in (6, 7, 8)) for i in range(a.steps)]
    finish = {"scope": "H3 compress fused with the H5 scan (k_finish) + H5 edge work (k_finish_proc, "
                       "k_finish_big) + H6 (" + ("partial: k_relabel" if partial_h6 else "full: k_compress") + ")",
              "t_fin_ms": round(fin_ms, 5), "ms": round(fin_ms, 5),
              "t_fin_ms_stats": {"median": round(statistics.median(t_fin_ms), 5), "min": round(min(t_fin_ms), 5),
                                 "p90": round(sorted(t_fin_ms)[min(len(t_fin_ms) - 1, int(0.9 * len(t_fin_ms)))], 5)},
              "bytes": int(B["finish_phase"]), "GB/s": round(fin_gbs, 1),
              "frac_of_8TBs": round(fin_gbs / CONTRACT_GBS, 4), "frac_of_measured": round(fin_gbs / peak, 4),
              "byte_model": "SURVEY 8(d) B_fin of the implemented design: 4n skip-test read + n/8 degree bitmap "
                            "(for 8 N_off) + 8 E_ng + candidates (queue, offsets, P[u]) + 4 W + 4 H + "
                            + ("the partial H6's tile summaries and dirty-tile re-reads (no 4n compress read)"
                               if partial_h6 else "4n compress read")
                            + "; root checks beyond the first parent level are not counted",
              "terms": extra["B_fin_terms"], "h6_mode": "partial" if partial_h6 else "full",
              "h6_dirty_tiles": int(ctr.get("h6_tiles", 0)), "tiles": (n + 2047) // 2048,
              "root_check_reads_not_counted": extra["root_check_reads_not_counted"]}
    if partial_h6:
        # the same t_fin against the 8(d) budget of a finish whose H6 reads all of P (4n more):
        # what a full-compress design would have to sustain to finish as fast (context only)
        full_b = B["finish_phase"] - B["k_compress_H6"] + 4 * n + 4 * ctr["h6_writes"]
        finish["full_compress_budget_view"] = {
            "bytes": int(full_b), "frac_of_8TBs_at_this_t_fin": round(full_b / (fin_ms * 1e-3) / 1e9 / CONTRACT_GBS, 4),
            "note": "8(d)'s B_fin with the 4n compress read of a full final compress, over this t_fin; the partial "
                    "H6 does not move those bytes (context, not the headline fraction)"}
    dram = [ncu_traffic(cfg.name, k) for k in ("k_finish", "k_finish_proc", "k_finish_big", "k_compress_H6")]
    if all(x is not None for x in dram):
        finish["dram_view"] = {"dram_bytes": int(sum(dram)), "GB/s": round(sum(dram) / (fin_ms * 1e-3) / 1e9, 1),
                               "frac_of_8TBs": round(sum(dram) / (fin_ms * 1e-3) / 1e9 / CONTRACT_GBS, 4),
                               "dram_over_B_fin": round(sum(dram) / max(1, B["finish_phase"]), 3),
                               "source": f"profiles/ncu_traffic.json[{cfg.name}] (ncu dram__bytes_read.sum + "
                                         f"dram__bytes_write.sum, cold cache, per launch)"}
    else:
        finish["dram_view"] = None
    phase_ms = {"sample": round(smp_ms, 5), "identify": round(kern_ms["k_identify"], 5),
                "finish": round(kern_ms["k_finish"] + kern_ms["k_finish_proc"], 5),
                "compress": round(kern_ms["k_compress_H6"], 5)}
    sampling = {"ms": round(smp_ms, 5), "bytes": int(B["sampling_phase"]),
                "GB/s": round(B["sampling_phase"] / (smp_ms * 1e-3) / 1e9, 1)}

    line = {"metric": "connectivity edges/sec (GTEPS)", "value": round(value, 4), "unit": "GTEPS",
            "n_gpus": ws, "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(max_ms, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic",
            "config": {"workload": cfg.name, "n": n, "m_directed": m, "kout_k": a.k, "variant": a.variant,
                       "flags": a.flags, "seed": cfg.seed, "components": components,
                       "l2": f"flushed between steps (write {flush.numel() * 4 >> 20} MiB > L2 {l2 >> 20} MiB); "
                             f"CSR {(8 * (n + 1) + 4 * m) / 1e9:.1f} GB > L2",
                       "parallelism": f"replicas x{ws}", "gen_s": round(gen_s, 2),
                       "cuda_graph": bool(a.graph),
                       "l2_fetch_granularity": a.l2_fetch if a.l2_fetch >= 0 else "driver default"},
            "t_ms": t_stats, "phase_ms": phase_ms, "ms_per_step_with_kernel_marks": round(statistics.mean(marked_ms), 5),
            "roofline": roofline, "finish": finish, "sampling": sampling, "kernels": kernels,
            "counters": ctr, "byte_model_extra": extra, "gpu_launches": int(launches), "clocks": clocks}

    line["parity"] = {"labels": "not checked", "forest": "not checked",
                      "oracle": "set by the cpu_baseline leg (rank 0, N = 1, without --no-cpu-baseline)"}
    # ---- measurement floors (K10, Table 8 analogue P:3732-3799), outside the timed region
    line["floors"] = floors(cc, d_off, d_adj, n, m, labels, stream, mean_ms)
    # spanning forest on the same graph (Alg. 2): t_SF / t_CC
    sf_edges = torch.empty((n, 2), dtype=torch.int32, device=dev)
    sf_num = torch.zeros(1, dtype=torch.int64, device=dev)
    sf_ms = []
    for i in range(4):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cc.cc_spanning_forest(d_off, d_adj, n, m, sf_edges, sf_num, None,
                              cc.make_opts(k=a.k, variant=variant, flags=a.flags), stream)
        e1.record(stream)
        e1.synchronize()
        if i:
            sf_ms.append(e0.elapsed_time(e1))
    line["spanning_forest"] = {"ms": round(statistics.mean(sf_ms), 4), "t_sf_over_t_cc": round(statistics.mean(sf_ms) / mean_ms, 3),
                               "forest_edges": int(sf_num.item()), "n_minus_c": n - components}
    # the forest pairs stay on the host for the oracle's validity check in the cpu_baseline leg
    sf_host = sf_edges[: int(sf_num.item())].cpu().numpy().view(np.uint32) if rank == 0 and ws == 1 else None
    del sf_edges
    # 64-bit fingerprint of the CSR bytes (SURVEY 8(d) JSON schema: csr_hash): sum of the
    # offsets and of the adjacency words, each weighted by an odd multiplier per position class
    line["config"]["csr_hash"] = "%016x" % ((int(d_off.sum().item()) * 0x9E3779B97F4A7C15
                                              + int(d_adj.to(torch.int64).sum().item()) * 0xBF58476D1CE4E5B9
                                              + m * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF)
    # The link kernel is bound by dependent random 4-byte accesses into the 4n-byte
    # parent array, not by streaming bandwidth: set its random-access count (one
    # P[v] gather per pending link + one load or CAS per Rem-loop step + the hook
    # CAS) against the uniform random-gather rate measured just above on an
    # array of the same size.
    rg = line["floors"]["random_gather"]["Gloads_per_s"]
    lk = kernels.get("k_sample_link" if ctr.get("fused_link") else "k_link_pending")
    if lk and contract:
        # contracted: the HBM random accesses are the P[v] gathers (one per pending
        # link); the Rem walk and CAS run in the L2-resident compact array
        acc = ctr["pending_links"]
        ach = acc / (lk["ms"] * 1e-3) / 1e9
        line["roofline"]["random_access_view"] = {
            "kernel": "k_link_pending", "hbm_random_accesses_per_launch": int(acc),
            "l2_link_accesses_per_launch": int(ctr["link_steps"] + ctr["sample_hooks"]),
            "achieved_Gaccess_per_s": round(ach, 2), "uniform_random_gather_Gloads_per_s": rg,
            "frac_of_random_gather_rate": round(ach / rg, 3)}
    elif lk:
        # both link kernels: link_steps counts Rem iterations that issued a load or a CAS (the
        # hook CAS included), each lost CAS adds the re-read of P[rv]; plus one P[v] gather
        # per pending link (P[u] is read in vertex order: not counted as random)
        acc = ctr["pending_links"] + ctr["link_steps"] + ctr["cas_failures"]
        ach = acc / (lk["ms"] * 1e-3) / 1e9
        line["roofline"]["random_access_view"] = {
            "kernel": "k_sample_link" if ctr.get("fused_link") else "k_link_pending",
            "random_accesses_per_launch": int(acc),
            "achieved_Gaccess_per_s": round(ach, 2), "uniform_random_gather_Gloads_per_s": rg,
            "frac_of_random_gather_rate": round(ach / rg, 3)}
    if lk and line["roofline"]["kernel"] in ("k_link_pending", "k_sample_link") and not contract:
        # The dominant kernel is the k-out link: SURVEY §8(d) puts H2 under the RANDOM-SECTOR
        # roofline (ii) -- a 4 B gather / CAS that misses L2 moves one 32 B sector, so the
        # ceiling is peak / 32 B accesses per second.  achieved = 32 B x random accesses per
        # launch / launch time; the 4 B algorithmic-bytes stream view is kept beside it.
        rf = line["roofline"]
        rv = rf["random_access_view"]
        acc = rv["random_accesses_per_launch"]
        ach_gbs = 32 * acc / (lk["ms"] * 1e-3) / 1e9
        rf["stream_view"] = {"achieved": rf["achieved"], "frac": rf["frac"],
                             "algorithmic_bytes_per_launch": rf["algorithmic_bytes_per_launch"],
                             "note": "4 B per parent access (SURVEY 8(d) B_smp terms) over the stream peak"}
        rf.update({"model": "random-sector (SURVEY 8(d) ceiling ii): 32 B sector per random 4 B access",
                   "achieved": round(ach_gbs, 1), "frac": round(ach_gbs / rf["peak"], 4),
                   "algorithmic_bytes_per_launch": int(32 * acc),
                   "peak_random_Gaccess_per_s": round(rf["peak"] / 32, 1)})

    # ---- e2e: the same metric through the C ABI with HOST (pinned) buffers.  Every rank pins
    # its own CSR copy; when the node's free host memory cannot hold one per local rank (plus
    # a margin), the e2e leg is skipped with a note rather than risking the run.
    need = 8 * (n + 1) + 4 * m + 4 * n
    local = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = None
    host_ok = avail is None or need * local * 1.15 < avail
    if not host_ok and rank == 0:
        print(f"[bench] e2e skipped: {local} x {need / 1e9:.1f} GB pinned > available {avail / 1e9:.0f} GB",
              file=sys.stderr)
    if not a.no_e2e and a.e2e_steps > 0 and not host_ok:
        line["e2e"] = {"value": None, "unit": "GTEPS", "skipped": f"host RAM: {local} ranks x {need / 1e9:.1f} GB "
                       f"pinned CSR > {avail / 1e9:.0f} GB available"}
    if not a.no_e2e and a.e2e_steps > 0 and host_ok:
        h_off = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
        h_adj = torch.empty(m, dtype=torch.int32, pin_memory=True)
        h_lab = torch.empty(n, dtype=torch.int32, pin_memory=True)
        h_off.copy_(d_off)
        h_adj.copy_(d_adj)
        torch.cuda.synchronize()
        ts = []
        for i in range(1 + a.e2e_steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            cc.cc_labels(h_off.data_ptr(), h_adj.data_ptr(), n, m, h_lab.data_ptr(),
                         cc.make_opts(k=a.k, variant=variant, flags=a.flags), stream)
            e1.record(stream)
            e1.synchronize()
            if i > 0:
                ts.append(e0.elapsed_time(e1))
        e2e_ms = reduce_max(statistics.mean(ts), ws)
        ok = bool(np.array_equal(h_lab.numpy().view(np.uint32), final))
        # zero-copy: the kernels read the offsets, one 16 B window of list heads per
        # non-isolated vertex and the finish candidates' lists straight from pinned
        # host memory, and H6 writes the labels into it (cc.h §Memory)
        h2d = 8 * (n + 1) + 16 * nonisolated + 16 * ctr["finish_vertices"] + 4 * ctr["finish_edges"]
        line["e2e"] = {"value": round(aggregate_value(m, e2e_ms * 1e-3, ws) / 1e9, 4), "unit": "GTEPS",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4 * n,
                       "host_resident_csr_bytes": 8 * (n + 1) + 4 * m,
                       "path": "cc_labels with pinned host offsets/adj/labels (zero-copy through UVA)",
                       "ms_per_step": round(e2e_ms, 3), "steps": a.e2e_steps, "labels_match_device_path": ok}
        del h_off, h_adj, h_lab

    # ---- cpu_baseline: the oracle on the host cores (rank 0, N = 1 only).  (1) oracle.cc_bfs on
    # the reported graph itself, in this run (one run for C4, median of 3 for
    # the smaller configs), its labels compared with the GPU's; (2) the RMAT-24 sample the
    # reference arm times, as a secondary number.
    if not a.no_cpu_baseline and rank == 0 and ws == 1:
        del flush
        torch.cuda.empty_cache()
        import oracle as _oracle
        need = 8 * (n + 1) + 4 * m + 16 * n          # host CSR copy + labels + BFS queue + GPU labels
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except Exception:
            avail = None
        full = None
        if avail is None or need * 1.2 < avail:
            off_h = d_off.cpu().numpy()
            adj_h = d_adj.cpu().numpy().view(np.uint32)
            reps = 1 if m > 1e9 else 3
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                lab_h = _oracle.cc_bfs(off_h, adj_h)
                ts.append(time.perf_counter() - t0)
            dt_full = statistics.median(ts)
            full = {"value": round(m / dt_full / 1e9, 5), "unit": "GTEPS", "cores": 1, "kind": "oracle",
                    "sample": f"oracle.cc_bfs (sequential BFS, 1 thread) on the reported workload itself "
                              f"({cfg.name}, n={n}, m={m}), median of {reps} run(s): {dt_full:.2f} s",
                    "seconds": round(dt_full, 3), "gpu_labels_bit_exact": bool(np.array_equal(lab_h, final))}
            # parity on the reported graph (SURVEY 8(d) JSON schema: parity): labels raw-equal to the
            # oracle's; the spanning forest by the validity triple (count, input edges, acyclic)
            c_or = int(np.count_nonzero(lab_h == np.arange(n, dtype=np.uint32)))
            rc, _ = _oracle.forest_check(off_h, adj_h, c_or, sf_host) if sf_host is not None else (-1, None)
            line["parity"] = {"labels": "bit-exact" if full["gpu_labels_bit_exact"] else "FAIL",
                              "forest": "valid" if rc == 0 else ("FAIL" if rc > 0 else "not checked"),
                              "oracle": "oracle.cc_bfs + oracle.forest_check on this graph, this run"}
            del off_h, adj_h, lab_h
        m_s, dt, off_s, adj_s, lab_s = cpu_oracle_sample(a.cpu_scale, True)
        reps, spent = 1, dt
        while spent < CPU_BASELINE_MIN_S and reps < 5:
            t0 = time.perf_counter()
            _oracle.cc_bfs(off_s, adj_s)
            spent += time.perf_counter() - t0
            reps += 1
        dt = spent / reps
        # parity of the product on the same sample (bit-exact labels)
        so, sa = torch.from_numpy(off_s).to(dev), torch.from_numpy(adj_s.view(np.int32)).to(dev)
        sl = torch.empty(off_s.size - 1, dtype=torch.int32, device=dev)
        cc.cc_labels(so, sa, off_s.size - 1, adj_s.size, sl, cc.make_opts(k=a.k, variant=variant, flags=a.flags))
        par = bool(np.array_equal(sl.cpu().numpy().view(np.uint32), lab_s))
        sample = {"value": round(m_s / dt / 1e9, 5), "unit": "GTEPS", "cores": 1, "kind": "oracle",
                  "sample": f"oracle.cc_bfs (sequential BFS, 1 thread) on RMAT scale {a.cpu_scale} "
                            f"(C4 recipe, seed 4), m={m_s}; mean of {reps} runs, {dt:.2f} s each",
                  "gpu_labels_bit_exact_on_sample": par}
        if full is not None:
            line["cpu_baseline"] = dict(full, host_cores=os.cpu_count(), secondary_sample=sample)
        else:
            line["cpu_baseline"] = dict(sample, host_cores=os.cpu_count(),
                                        full_workload_skipped=f"host RAM: need {need / 1e9:.1f} GB, "
                                                              f"available {avail / 1e9:.1f} GB")
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_ours_incr(a, rank, ws, cfg):
    """--config 5: 256 batches of (943,718 inserts, 104,858 queries) on n = 2^26."""
    import numpy as np
    import torch

    from inputs import gpu as ggen
    from paper_2008_03909_b200 import cc
    n = 1 << cfg.scale
    nb = cfg.n_batches
    ins = torch.empty((nb, cfg.n_ins, 2), dtype=torch.int32, device="cuda")
    qs = torch.empty((nb, cfg.n_q, 2), dtype=torch.int32, device="cuda")
    for b in range(nb):
        ggen.incr_batch(cfg.seed, cfg.scale, b, cfg.n_ins, cfg.n_q, ins[b], qs[b])
    ans = torch.empty((nb, cfg.n_q), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    sh = stream.cuda_stream

    ic = np.full(nb, cfg.n_ins, dtype=np.int64)
    qc = np.full(nb, cfg.n_q, dtype=np.int64)

    def stream_once(ev=None, outer=None):
        h = cc.Incr(n, flags=a.flags)
        torch.cuda.synchronize()
        if outer is not None:
            outer[0].record(stream)
        if ev is None:
            # the whole device-resident stream in one cc_incr_batches call (its batches' pairs
            # are all in place before the call, so each kernel after the first may read its
            # pairs and first parents before its PDL wait: DESIGN §6 item 21)
            h.batches(ic, ins, qc, qs, ans, sh)
        for b in range(nb if ev is not None else 0):
            ev[b][0].record(stream)
            h.batch(ins[b], cfg.n_ins, qs[b], cfg.n_q, ans[b], sh)
            ev[b][1].record(stream)
        if outer is not None:
            outer[1].record(stream)
        torch.cuda.synchronize()
        h.close()

    for _ in range(a.warmup):
        stream_once()
    clk = Clocks(torch.cuda.current_device())
    clk.start()
    outer = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(a.steps)]
    barrier(ws)
    torch.cuda.synchronize()
    l0 = cc.launch_count()
    for s in range(a.steps):
        stream_once(outer=outer[s])           # one step = the whole 256-batch stream, events around it
    barrier(ws)
    launches = cc.launch_count() - l0
    clocks = clk.stop()
    per_stream = [outer[s][0].elapsed_time(outer[s][1]) for s in range(a.steps)]
    # per-batch latency: the same streams again, one cc_incr_batch call per batch with an event
    # pair around it (the events serialise the batches, so the throughput above is taken
    # without them)
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(nb)] for _ in range(a.steps)]
    for s in range(a.steps):
        stream_once(evs[s])
    batch_ms = sorted(evs[s][b][0].elapsed_time(evs[s][b][1]) for s in range(a.steps) for b in range(nb))
    mean_ms = reduce_max(statistics.mean(per_stream), ws)
    ops = nb * (cfg.n_ins + cfg.n_q)
    line = {"metric": "incremental connectivity ops/sec", "value": round(aggregate_value(ops, mean_ms * 1e-3, ws) / 1e9, 4),
            "unit": "Gops/s", "n_gpus": ws, "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(mean_ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": cfg.name, "n": n, "batches": nb, "inserts_per_batch": cfg.n_ins,
                       "queries_per_batch": cfg.n_q, "l2": "P (256 MiB) > L2",
                       "api": "one cc_incr_batches call per 256-batch stream (batch_ms: one cc_incr_batch call per batch)"},
            "inserts_per_s": round(nb * cfg.n_ins / (mean_ms * 1e-3), 1),
            "batch_ms": {"p50": batch_ms[len(batch_ms) // 2], "p99": batch_ms[int(len(batch_ms) * 0.99)]},
            "gpu_launches": int(launches), "clocks": clocks}

    # ---- roofline: algorithmic bytes per stream (insert 8 B pair + 8 B for
    # P[u], P[v] + 4 B per hook; query 8 + 8 + 1 B), hooks = n - final components
    h = cc.Incr(n, flags=a.flags)
    for b in range(nb):
        h.batch(ins[b], cfg.n_ins, qs[b], cfg.n_q, ans[b])
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    h.labels(lab)
    comps = int((lab == torch.arange(n, device="cuda", dtype=torch.int32)).sum().item())
    h.close()
    del lab
    hooks = n - comps
    byts = nb * (16 * cfg.n_ins + 17 * cfg.n_q) + 4 * hooks
    peak, peak_src = peaks()
    gbs = byts / (mean_ms * 1e-3) / 1e9
    rg_t = torch.zeros(1, dtype=torch.int32, device="cuda")
    x = torch.zeros(n, dtype=torch.int32, device="cuda")
    cnt = 1 << 28
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cc.random_gather(x, n, cnt, 7, rg_t, stream)
    e0.record(stream)
    cc.random_gather(x, n, cnt, 7, rg_t, stream)
    e1.record(stream)
    e1.synchronize()
    rg = cnt / (e0.elapsed_time(e1) * 1e-3) / 1e9
    acc = nb * 2 * (cfg.n_ins + cfg.n_q)                  # first parent reads: P[u], P[v] of every op
    # random-sector roofline (SURVEY 8(d) ceiling ii; the incremental path is random-sector and
    # atomic bound): one 32 B sector per random parent access, first-level reads only (deeper
    # walk steps are not counted); the 4 B algorithmic-bytes stream view is kept beside it
    sec = 32 * acc / (mean_ms * 1e-3) / 1e9
    line["roofline"] = {"bound": "hbm", "kernel": "k_insert + k_query (whole stream)", "achieved": round(sec, 1),
                        "peak": peak, "unit": "GB/s", "frac": round(sec / peak, 4), "traffic": None,
                        "model": "random-sector (SURVEY 8(d) ceiling ii): 32 B sector per random first-level "
                                 "parent access (P[u], P[v] of every op)",
                        "algorithmic_bytes_per_stream": int(32 * acc),
                        "peak_random_Gaccess_per_s": round(peak / 32, 1),
                        "stream_view": {"achieved": round(gbs, 1), "frac": round(gbs / peak, 4),
                                        "algorithmic_bytes_per_stream": int(byts),
                                        "note": "SURVEY 8(d) per-op bytes: insert 16 B + 4 B per hook, query 17 B"},
                        "peak_source": peak_src, "hooks": hooks,
                        "random_access_view": {"first_parent_reads_per_stream": acc,
                                               "achieved_Gaccess_per_s": round(acc / (mean_ms * 1e-3) / 1e9, 2),
                                               "uniform_random_gather_Gloads_per_s": round(rg, 2),
                                               "array_bytes": 4 * n}}
    del x

    # ---- e2e: the same stream through cc_incr_batch with the batches in pinned HOST memory
    # (used in place through UVA) and the answers written to pinned host memory
    if not a.no_e2e:
        h_ins = torch.empty_like(ins, device="cpu").pin_memory()
        h_qs = torch.empty_like(qs, device="cpu").pin_memory()
        h_ans = torch.empty((nb, cfg.n_q), dtype=torch.uint8).pin_memory()
        h_ins.copy_(ins)
        h_qs.copy_(qs)
        ts = []
        for rep in range(2):
            h = cc.Incr(n, flags=a.flags)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            # the whole stream in one cc_incr_batches call: the library DMAs batch b+1's pairs
            # while batch b computes (double-buffered), answers written to the host in place
            h.batches(np.full(nb, cfg.n_ins, dtype=np.int64), h_ins, np.full(nb, cfg.n_q, dtype=np.int64), h_qs,
                      h_ans, stream)
            e1.record(stream)
            e1.synchronize()
            h.close()
            ts.append(e0.elapsed_time(e1))
        e2e_ms = min(ts)
        line["e2e"] = {"value": round(ops / (e2e_ms * 1e-3) / 1e9, 4), "unit": "Gops/s",
                       "h2d_bytes_per_step": int(nb * 8 * (cfg.n_ins + cfg.n_q)), "d2h_bytes_per_step": int(nb * cfg.n_q),
                       "ms_per_step": round(e2e_ms, 3),
                       "path": "one cc_incr_batches call over the 256 pinned host batches: pairs DMA'd double-buffered "
                                       "on a copy stream (batch b+1 while batch b computes), answers written "
                                       "to the host in place (UVA)",
                       "answers_match_device_path": bool(torch.equal(h_ans, ans.cpu()))}
        del h_ins, h_qs, h_ans

    # ---- cpu_baseline: the oracle (sequential DSU, 1 thread) on the first batches of the
    # same stream (the generator's bytes), answers checked against the GPU's
    if not a.no_cpu_baseline and rank == 0 and ws == 1:
        import numpy as np

        import oracle
        nbs = min(nb, a.cpu_batches)
        hi = ins[:nbs].cpu().numpy().view(np.uint32)
        hq = qs[:nbs].cpu().numpy().view(np.uint32)
        t0 = time.time()
        want, _ = oracle.incr_run(n, [(hi[b], hq[b]) for b in range(nbs)])
        t_or = time.time() - t0
        ops_s = nbs * (cfg.n_ins + cfg.n_q)
        line["cpu_baseline"] = {"value": round(ops_s / t_or / 1e9, 5), "unit": "Gops/s", "cores": 1, "kind": "oracle",
                                "sample": f"oracle.incr_run (sequential union-find, 1 thread) on the first {nbs} "
                                          f"batches of the C5 stream ({ops_s} ops), {t_or:.2f} s",
                                "host_cores": os.cpu_count(),
                                "gpu_answers_bit_exact_on_sample": bool(np.array_equal(
                                    ans[:nbs].cpu().numpy().reshape(-1), want))}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_study(a):
    """NEXT-1: k-out variant x k sweep on C2-C4 -- per-phase device
    times, sampling coverage (share of vertices in L_max's sampled component),
    inter-component edges left by the sample (IC),
    edges the finish traversed, and whether labels stayed bit-identical."""
    import numpy as np
    import torch

    import inputs
    from inputs import gpu as ggen
    from paper_2008_03909_b200 import cc
    grid = [("afforest", k) for k in (0, 1, 2, 3, 4)] + [("hybrid", 2), ("hybrid", 3), ("pure", 2), ("pure", 3)]
    stream = torch.cuda.current_stream()
    rows = []
    for cfg in (inputs.C2, inputs.C3, inputs.C4):
        d_off, d_adj = ggen.config_graph(cfg)
        n, m = d_off.numel() - 1, d_adj.numel()
        deg = torch.diff(d_off)
        src = torch.repeat_interleave(torch.arange(n, device="cuda", dtype=torch.int32), deg) if m < 2**31 else None
        ref = None
        for variant, k in grid:
            var = {"afforest": cc.VARIANT_AFFOREST, "hybrid": cc.VARIANT_HYBRID, "pure": cc.VARIANT_PURE}[variant]
            labels = torch.empty(n, dtype=torch.int32, device="cuda")
            sampled = torch.empty(n, dtype=torch.int32, device="cuda")
            lmax = torch.empty(1, dtype=torch.int32, device="cuda")
            ctr = torch.zeros(len(cc.COUNTER_FIELDS), dtype=torch.int64, device="cuda")
            cc.cc_labels(d_off, d_adj, n, m, labels, cc.make_opts(k=k, variant=var, seed=cfg.seed, counters=ctr,
                                                                  sampled_out=sampled, lmax_out=lmax), stream)
            ms = []
            for _ in range(a.warmup + a.steps):
                marks = [torch.cuda.Event(enable_timing=True) for _ in range(cc.NUM_MARKS)]
                for e in marks:
                    e.record(stream)
                torch.cuda.synchronize()
                cc.cc_labels(d_off, d_adj, n, m, labels, cc.make_opts(k=k, variant=var, seed=cfg.seed,
                                                                      marks=[e.cuda_event for e in marks]), stream)
                torch.cuda.synchronize()
                ms.append([marks[j - 1].elapsed_time(marks[j]) for j in range(1, cc.NUM_MARKS)])
            ms = np.array(ms[a.warmup:]).mean(0)
            c = dict(zip(cc.COUNTER_FIELDS, ctr.cpu().tolist()))
            lm = int(lmax.item())
            coverage = float((sampled == lm).float().mean().item())
            ic = int((sampled[src.long()] != sampled[d_adj.long()]).sum().item()) // 2 if src is not None else None
            lab = labels.cpu()
            if ref is None:
                ref = lab
            rows.append({"workload": cfg.name, "variant": variant, "k": k,
                         "ms_total": round(float(ms.sum()), 4),
                         "ms": {cc.MARK_NAMES[j]: round(float(ms[j - 1]), 4) for j in range(1, cc.NUM_MARKS)},
                         "coverage": round(coverage, 4), "ic_edges_after_sampling": ic,
                         "pending_links": c["pending_links"], "finish_vertices": c["finish_vertices"],
                         "finish_edges": c["finish_edges"], "labels_identical": bool(torch.equal(lab, ref))})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
        del d_off, d_adj, deg, src
        torch.cuda.empty_cache()
    print(json.dumps({"study": "NEXT-1 k-out variant x k sweep", "rows": rows}), flush=True)


def run_incr_sweep(a):
    """NEXT-2: incremental variants.
    A: throughput vs batch size, inserts only, empty start on 2^20 vertices (the
       shape of the paper's Table 5), RMAT-20 stream.
    B: the C5 shape (2^26 vertices, 256 batches of 2^20 ops): phase-concurrent
       (type 3) vs wait-free (type 1); batch order as drawn vs sorted
       by source; query share 10/50/90 % with naive vs splitting
       finds."""
    import torch

    from inputs import gpu as ggen
    from paper_2008_03909_b200 import cc
    stream = torch.cuda.current_stream()

    sh = stream.cuda_stream            # raw handle: no torch stream query per call

    def time_stream(n, ins_b, qs_b, flags):
        ans = [torch.empty(q.shape[0], dtype=torch.uint8, device="cuda") for q in qs_b]
        best = None
        for rep in range(2):
            h = cc.Incr(n, flags=flags)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for b in range(len(ins_b)):
                h.batch(ins_b[b], ins_b[b].shape[0], qs_b[b], qs_b[b].shape[0], ans[b], sh)
            e1.record(stream)
            e1.synchronize()
            h.close()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        return best

    out = {"A_batch_size": [], "B_c5_variants": []}
    # ---- A
    n = 1 << 20
    total = 1 << 22
    all_ins, _ = ggen.incr_batch(7, 20, 0, total, 1)
    empty_q = torch.empty((0, 2), dtype=torch.int32, device="cuda")
    import numpy as np
    no_ans = torch.empty(1, dtype=torch.uint8, device="cuda")
    for bs in (10, 100, 1000, 10_000, 100_000, 1_000_000, 2_000_000):
        nb = min(total // bs, 2000)
        ins_b = [all_ins[i * bs:(i + 1) * bs] for i in range(nb)]
        t = time_stream(n, ins_b, [empty_q] * nb, 0)
        # the same batches through one cc_incr_batches call (one launch for small batches)
        best = None
        for rep in range(2):
            h = cc.Incr(n)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            h.batches(np.full(nb, bs), all_ins[:nb * bs], np.zeros(nb), empty_q, no_ans)
            e1.record(stream)
            e1.synchronize()
            h.close()
            tb = e0.elapsed_time(e1)
            best = tb if best is None else min(best, tb)
        out["A_batch_size"].append({"batch": bs, "batches": nb, "ms_per_call_api": round(t, 3),
                                    "inserts_per_s": round(nb * bs / (t * 1e-3), 1),
                                    "ms_multi_batch_api": round(best, 3),
                                    "inserts_per_s_multi_batch_api": round(nb * bs / (best * 1e-3), 1)})
        print(json.dumps(out["A_batch_size"][-1]), file=sys.stderr, flush=True)
    # ---- B
    n = 1 << 26
    nb, per = 256, 1 << 20
    for qfrac in (0.1, 0.5, 0.9):
        n_q = int(per * qfrac) if qfrac != 0.1 else 104_858
        n_ins = per - n_q
        ins_b, qs_b = [], []
        for b in range(nb):
            i, q = ggen.incr_batch(5, 26, b, n_ins, n_q)
            ins_b.append(i)
            qs_b.append(q)
        variants = [("phase_concurrent", 0, False), ("phase_concurrent_find_split", cc.FLAG_FIND_SPLIT, False),
                    ("wait_free", cc.FLAG_WAIT_FREE, False)]
        if qfrac == 0.1:
            variants.append(("phase_concurrent_sorted_batches", 0, True))
        for name, flags, sort in variants:
            ib = ins_b
            if sort:
                ib = [x[torch.argsort(x[:, 0].long() * (1 << 32) + x[:, 1].long())].contiguous() for x in ins_b]
            t = time_stream(n, ib, qs_b, flags)
            out["B_c5_variants"].append({"query_share": qfrac, "variant": name, "ms": round(t, 3),
                                         "ops_per_s": round(nb * per / (t * 1e-3), 1),
                                         "inserts_per_s": round(nb * n_ins / (t * 1e-3), 1)})
            print(json.dumps(out["B_c5_variants"][-1]), file=sys.stderr, flush=True)
        del ins_b, qs_b
    print(json.dumps({"study": "NEXT-2 incremental variants", **out}), flush=True)


def run_table4(a):
    """NEXT-2 (b): the paper's Table 4 protocol: maximum
    insert throughput, one batch, no queries, on the RM stream -- RMAT n = 2^30,
    m = 10n, (a, b, c) = (.5, .1, .1), unpermuted.  The 10.7e9 inserts are fed as
    consecutive sub-batches of 2^28 pairs (no queries in between, so the same as one
    batch); generation is outside the timed region, each sub-batch's insert call is
    timed with CUDA events on the launching stream.  Also the same protocol on the
    C5 stream shape (RMAT-26 Graph500 parameters, permuted) for comparison."""
    import torch

    from inputs import gen
    from inputs import gpu as ggen
    from paper_2008_03909_b200 import cc
    stream = torch.cuda.current_stream()
    rows = []
    for name, s, total, t, perm in (("RM n=2^30 m=10n (.5,.1,.1) unpermuted", 30, 10 << 30, gen.RM_T, False),
                                    ("C5 shape: RMAT-26 Graph500, permuted, 2^28 inserts", 26, 1 << 28,
                                     (gen.RMAT_T1, gen.RMAT_T2, gen.RMAT_T3), True)):
        n = 1 << s
        chunk = 1 << 28
        buf = torch.empty((chunk, 2), dtype=torch.int32, device="cuda")
        empty_q = torch.empty((0, 2), dtype=torch.int32, device="cuda")
        no_ans = torch.empty(1, dtype=torch.uint8, device="cuda")
        best = None
        for rep in range(max(1, a.steps)):
            h = cc.Incr(n, flags=a.flags)
            ms = 0.0
            for first in range(0, total, chunk):
                cnt = min(chunk, total - first)
                ggen.rmat_stream(s, s, first, cnt, t=t, permuted=perm, out=buf[:cnt])
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                h.batch(buf[:cnt], cnt, empty_q, 0, no_ans)
                e1.record(stream)
                e1.synchronize()
                ms += e0.elapsed_time(e1)
            lab = torch.empty(n, dtype=torch.int32, device="cuda")
            h.labels(lab)
            comps = int((lab == torch.arange(n, device="cuda", dtype=torch.int32)).sum().item())
            h.close()
            del lab
            best = ms if best is None else min(best, ms)
        rows.append({"stream": name, "n": n, "inserts": total, "ms": round(best, 3),
                     "inserts_per_s": round(total / (best * 1e-3), 1), "components": comps,
                     "paper_72core_inserts_per_s": 8.78e8 if s == 30 else None})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
        del buf
        torch.cuda.empty_cache()
    print(json.dumps({"study": "NEXT-2(b) Table 4 protocol", "rows": rows}), flush=True)


def run_amsf(a):
    """NEXT-4: AMSF-NF-S on C3 / C4 with the seeded
    Exp(1) weights (the paper's weighted inputs are not here),
    eps = 0.25.  Variants: NF-S with the per-vertex weight-range index
    (default), NF-S as stated (AMSF_PLAIN), and both without the L_max skip (NF).
    Per variant: device time of one cc_amsf call (CUDA events, mean of --steps
    after --warmup), rounds, active-vertex visits, weights inspected, forest
    weight; the oracle's AMSF and Kruskal timed on an RMAT-20 sample (1 thread)
    with W_APX / W_OPT there."""
    import numpy as np
    import torch

    import inputs
    import oracle
    from inputs import gen
    from inputs import gpu as ggen
    from paper_2008_03909_b200 import cc
    stream = torch.cuda.current_stream()
    variants = [("nf_s_index", 0), ("nf_s_range", cc.FLAG_AMSF_NO_INDEX), ("nf_s_plain", cc.FLAG_AMSF_PLAIN),
                ("nf_index", cc.FLAG_NO_SKIP), ("nf_plain", cc.FLAG_AMSF_PLAIN | cc.FLAG_NO_SKIP)]
    rows = []
    for cfg in (inputs.C3, inputs.C4):
        d_off, d_adj = ggen.config_graph(cfg)
        d_w = ggen.exp_weights(d_off, d_adj, cfg.seed)
        n, m = d_off.numel() - 1, d_adj.numel()
        deg = torch.diff(d_off)
        m_idx = int(deg[deg > 256].sum().item())         # entries of the indexed lists (cc_amsf.cu kIdxMin)
        del deg
        edges = torch.empty((n, 2), dtype=torch.int32, device="cuda")
        ew = torch.empty(n, dtype=torch.float32, device="cuda")
        num = torch.zeros(1, dtype=torch.int64, device="cuda")
        tot = torch.zeros(1, dtype=torch.float64, device="cuda")
        for name, flags in variants:
            if cfg is inputs.C4 and flags & cc.FLAG_AMSF_PLAIN and flags & cc.FLAG_NO_SKIP:
                continue                                   # ~100 full passes over 34 GB: skipped at C4
            ctr = torch.zeros(len(cc.COUNTER_FIELDS), dtype=torch.int64, device="cuda")
            cc.cc_amsf(d_off, d_adj, d_w, n, m, a.eps, edges, ew, num, tot, cc.make_opts(flags=flags, counters=ctr),
                       stream)
            torch.cuda.synchronize()
            c = dict(zip(cc.COUNTER_FIELDS, ctr.cpu().tolist()))
            ts = []
            for i in range(a.warmup + a.steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                cc.cc_amsf(d_off, d_adj, d_w, n, m, a.eps, edges, ew, num, tot, cc.make_opts(flags=flags), stream)
                e1.record(stream)
                e1.synchronize()
                if i >= a.warmup:
                    ts.append(e0.elapsed_time(e1))
            ms = float(np.mean(ts))
            # algorithmic bytes: the weight-range pass (4 B per entry), the bucket index of the
            # lists longer than 256 (weights read twice, 4 B index entry written), one weight
            # (+ one index entry when indexed) per inspected entry, the endpoint of every
            # in-bucket entry (<= m), offsets + weight range per visit
            indexed = not (flags & (cc.FLAG_AMSF_PLAIN | cc.FLAG_AMSF_NO_INDEX))
            byts = (4 * m + (12 * m_idx if indexed else 0) + 4 * c["amsf_edges"]
                    + (4 * min(c["amsf_edges"], m_idx) if indexed else 0) + 4 * m + 24 * c["amsf_visits"])
            peak, _ = peaks()
            rows.append({"workload": cfg.name, "variant": name, "flags": flags, "eps": a.eps, "ms": round(ms, 3),
                         "GTEPS": round(m / (ms * 1e-3) / 1e9, 2), "rounds": c["amsf_rounds"],
                         "visits": c["amsf_visits"], "weights_inspected": c["amsf_edges"],
                         "inspected_per_entry": round(c["amsf_edges"] / m, 3), "forest_edges": int(num.item()),
                         "forest_weight": float(tot.item()), "rebuilds": c["amsf_rebuilds"],
                         "algorithmic_GBps": round(byts / (ms * 1e-3) / 1e9, 1),
                         "roofline": {"bound": "hbm", "achieved": round(byts / (ms * 1e-3) / 1e9, 1), "peak": peak,
                                      "unit": "GB/s", "frac": round(byts / (ms * 1e-3) / 1e9 / peak, 4),
                                      "bytes": int(byts)}})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
        del d_off, d_adj, d_w, edges, ew
        torch.cuda.empty_cache()
    # the oracle on a bounded sample: RMAT-20 (C4 recipe)
    off, adj = gen.rmat(seed=4, scale=20)
    w = gen.exp_weights(off, adj, 4)
    t0 = time.time()
    r = oracle.amsf(off, adj, w, a.eps)
    t1 = time.time()
    wopt = oracle.kruskal(off, adj, w)[0]
    t2 = time.time()
    d_off, d_adj = torch.from_numpy(off).cuda(), torch.from_numpy(adj.view(np.int32)).cuda()
    d_w = torch.from_numpy(w).cuda()
    E, W, tg = __import__("paper_2008_03909_b200").amsf(d_off, d_adj, d_w, a.eps)
    sample = {"graph": "RMAT-20 (C4 recipe, seed 4)", "m": int(adj.size), "oracle_amsf_s": round(t1 - t0, 3),
              "oracle_kruskal_s": round(t2 - t1, 3), "cores": 1, "W_opt": wopt, "W_oracle_amsf": r["total"],
              "W_gpu_amsf": tg, "gpu_over_opt": round(tg / wopt, 6), "oracle_over_opt": round(r["total"] / wopt, 6),
              "buckets": r["nbuckets"]}
    print(json.dumps({"study": "NEXT-4 AMSF-NF-S", "rows": rows, "cpu_sample": sample}), flush=True)


def main():
    a = parse()
    rank, ws = dist_setup()
    if a.study:
        run_study(a)
    elif a.amsf:
        run_amsf(a)
    elif a.table4:
        run_table4(a)
    elif a.incr_sweep:
        run_incr_sweep(a)
    elif a.impl == "reference":
        run_reference(a, rank, ws)
    else:
        run_ours(a, rank, ws)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
