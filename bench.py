#!/usr/bin/env python
"""bench.py -- Bingo hot path on B200, the paper's protocol (S6.1: rounds of
(BATCHSIZE updates -> application)).

Headline (BASELINE.json configs[3], the config its "1/2/4/8 B200" metric is quoted on):
Twitter-shaped R-MAT (46.2M V / 1.47B arcs, degree biases), a step = one round =
  broadcast of rank 0's 100K-arc-record update batch (Mixed)
  -> bingo_apply_updates on every replica
  -> personalized PageRank walks (stop w.p. 1/80 after each step) of one walker per
     vertex, the walker ids split evenly over the ranks (strong scaling: fixed total work)
  -> the visit counts combined with ONE all-reduce (ReplicatedBingo.visit_counts).
Secondary (configs[1], same line, key "secondary"): LiveJournal-shaped R-MAT, one update
batch + biased DeepWalk of one walker per vertex x 80 steps, paths written to HBM.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

The graph is generated in HBM (synth.DeviceWorkload, seeded), with a held-out set of 10
batches that does not depend on --steps, so both arms run the same graph and the
same batches.  Inputs (graph pools, 1.5-3 GB of outputs per step) exceed the 126 MB L2.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0   # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent
HOLD_ROUNDS = 10            # the held-out edges of 10 rounds of updates
CFG_INDEX = {"c1": 0, "c2": 1, "c3": 2, "c4": 3, "c5": 4}
METRIC = "walk steps/s (round = update batch + walk of one walker per vertex [+ PPR count all-reduce])"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", help="headline config (BASELINE configs[3] = c4)")
    ap.add_argument("--secondary", default="c2", help="second workload in the same line ('' = none)")
    ap.add_argument("--length", type=int, default=80)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ceiling", action="store_true", help="skip the trace/replay gather ceiling")
    ap.add_argument("--no-meter", action="store_true", help="skip the in-run CUPTI DRAM counters")
    ap.add_argument("--trace-records", type=float, default=1.2e9, help="max traced steps for the ceiling")
    ap.add_argument("--sort-records", type=float, default=6e8, help="traced steps replayed in window-sorted order")
    ap.add_argument("--cpu-walkers", type=int, default=1 << 15, help="oracle walker sample per step")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for N > 1 (gloo: test the multi-rank path without NVLink)")
    ap.add_argument("--share-device", action="store_true",
                    help="test only: every rank on cuda:0 (exercise the N > 1 code path on a 1-GPU box)")
    return ap.parse_args()


def app_of(config):
    import synth
    return synth.CONFIGS[config]["app"]


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": HBM_FALLBACK_GBS}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def rd():
            for line in self.proc.stdout:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
        self.thread = threading.Thread(target=rd, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=1)
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for i, nme in enumerate(names):
                if s[3 + i].lower().startswith("active"):
                    reasons.add(nme)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def bind_to_gpu_numa(local: int):
    """Run on the CPUs local to the GPU, so pinned host buffers (first touch) sit on the GPU's
    NUMA node.  Best effort: silently skipped where sysfs does not say."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(local)
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bdf}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            if "-" in part:
                lo, hi = part.split("-")
                cpus.update(range(int(lo), int(hi) + 1))
            elif part:
                cpus.add(int(part))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return sorted(cpus)
    except Exception:
        return None
    return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def config_block(config, V, arcs, nrec, ws, extra=None):
    import synth
    cfg = synth.CONFIGS[config]
    app = cfg["app"]
    walk = {"ppr": "personalized PageRank, stop 1/80 after each step (P:536), visit counts, no paths",
            "deepwalk": "biased DeepWalk x 80 steps, step-major paths in HBM",
            "node2vec": "node2vec p=2 q=0.5 x 80 steps"}[app]
    c = {"workload": f"BASELINE configs[{CFG_INDEX[config]}]: {cfg['desc']}", "config": config, "V": int(V),
         "arcs": int(arcs), "walk": f"{walk}; one walker per vertex ({V}), walker ids split over {ws} rank(s)",
         "update_batch_arc_records": int(nrec), "update_batch_edges": int(nrec // 2),
         "held_out_rounds": HOLD_ROUNDS, "bias": "w(u,v)=max(1,deg(v)) (P:664)", "alpha_beta": [40, 10],
         "generator": "synth.DeviceWorkload (R-MAT 0.57/0.19/0.19/0.05, seeds 1/2), generated in HBM",
         "l2": "inputs larger than L2 (graph pools of 3-75 GB, outputs of 0.4-1.5 GB per step): no flush needed"}
    if extra:
        c.update(extra)
    return c


# ---------------------------------------------------------------- in-run hardware counters
class Meter:
    """CUPTI range profiler around one launch (tools/dram_meter.cpp): DRAM bytes read + written
    and the L2 sector hit rate of the region, measured in this process (None if unavailable,
    e.g. under ncu)."""
    METRICS = ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct")

    def __init__(self):
        from paper_2504_10233_b200 import _build
        self.L = None
        if os.path.exists(_build.METER_LIB):
            try:
                self.L = ctypes.CDLL(_build.METER_LIB)
                self.L.dm_begin.argtypes = [ctypes.c_char_p]
                self.L.dm_end.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
            except OSError:
                self.L = None

    def measure(self, fn, max_passes=4):
        import torch
        if self.L is None:
            return None, "meter library unavailable"
        torch.cuda.synchronize()
        rc = self.L.dm_begin(",".join(self.METRICS).encode())
        if rc != 0:
            return None, f"CUPTI range profiler unavailable (step {rc})"
        done = 0
        for _ in range(max_passes):
            if self.L.dm_pass_begin() != 0:
                self.L.dm_abort()
                return None, "pass begin failed"
            fn()
            torch.cuda.synchronize()
            done = self.L.dm_pass_end()
            if done != 0:
                break
        if done != 1:
            self.L.dm_abort()
            return None, "passes not completed"
        vals = (ctypes.c_double * len(self.METRICS))()
        if self.L.dm_end(vals, len(self.METRICS)) != 0:
            return None, "evaluation failed"
        return dict(zip(self.METRICS, list(vals))), "ok"


# ---------------------------------------------------------------- graph setup
def make_graph(args, config, rounds, dev, ws, rank, dist):
    """Rank 0 generates the workload in HBM; with NCCL the CSR and the batches are broadcast
    to the other ranks over NVLink (every replica is built from the same arrays)."""
    import torch
    import synth
    import paper_2504_10233_b200 as pb
    t0 = time.time()
    share = dist is not None          # rank 0 generates, the others receive (NCCL over NVLink; gloo in tests)
    if rank == 0 or not share:
        w = synth.make_workload(config, rounds=rounds, hold_rounds=HOLD_ROUNDS, device=dev, resident=True)
        ro, dst, bias, batches, V, A = w.row_offsets, w.dst, w.bias, w.batches, w.V, w.num_arcs
    if share:
        meta = torch.zeros(3, dtype=torch.int64, device=dev)
        if rank == 0:
            meta[0], meta[1], meta[2] = V, A, batches[0].shape[0]
        dist.broadcast(meta, 0)
        V, A, nrec = (int(x) for x in meta.tolist())
        if rank != 0:
            ro = torch.empty(V + 1, dtype=torch.int64, device=dev)
            dst = torch.empty(A, dtype=torch.int32, device=dev)
            bias = torch.empty(A, dtype=torch.int32, device=dev)
        for t in (ro, dst, bias):
            dist.broadcast(t, 0)
        bt = (torch.from_numpy(np.stack(batches).view(np.int32)).to(dev) if rank == 0
              else torch.empty((rounds, nrec, 4), dtype=torch.int32, device=dev))
        dist.broadcast(bt, 0)
        batches = [b for b in bt.cpu().numpy().view(np.uint32)]
    t_gen = time.time() - t0
    host_csr = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and config == args.config:
        host_csr = (ro.cpu().numpy().view(np.uint64), dst.cpu().numpy().view(np.uint32),
                    bias.cpu().numpy().view(np.uint32))
    t0 = time.time()
    g = pb.Graph(ro, dst, bias, device=dev)
    torch.cuda.synchronize()
    t_build = time.time() - t0
    del ro, dst, bias
    if rank == 0 or not share:
        del w
    torch.cuda.empty_cache()
    return g, batches, V, A, host_csr, {"gen_s": round(t_gen, 2), "build_s": round(t_build, 2)}


# ---------------------------------------------------------------- one workload
def run_workload(args, config, dev, ws, rank, local, dist, primary):
    import torch
    import paper_2504_10233_b200 as pb
    from paper_2504_10233_b200.distributed import ReplicatedBingo, shard_range
    app = app_of(config)
    K, W = args.steps, args.warmup
    e2e_steps = 0 if args.no_e2e or not primary else K
    rounds = W + K + e2e_steps + (1 if primary else 2)
    g, batches, V, A, host_csr, times = make_graph(args, config, rounds, dev, ws, rank, dist)
    nrec = batches[0].shape[0]
    dev_batches = [torch.from_numpy(b.view(np.int32)).to(dev) for b in batches[:W + K]] if rank == 0 \
        else [None] * (W + K)
    rb = ReplicatedBingo(g, device=dev)
    first, count = shard_range(V, rank, ws)
    L = args.length
    stream = torch.cuda.current_stream()
    lens = [torch.empty(count, dtype=torch.int32, device=dev) for _ in range(K)]
    scratch_len = torch.empty(count, dtype=torch.int32, device=dev)
    if app == "ppr":
        wkw = dict(app=pb.PPR, length=pb.NO_CAP, stop=(1, 80), paths=None)
        paths = None
    else:
        paths = torch.empty((L + 1, count), dtype=torch.int32, device=dev)
        wkw = dict(app=pb.DEEPWALK, length=L, paths=paths)
    g.reset_visit_counts()

    def step(i, out_len, ev=None):
        if ev is not None:
            ev[0].record(stream)
        rb.apply_updates(dev_batches[i] if rank == 0 else None, n=nrec)   # broadcast + apply
        if ev is not None:
            ev[1].record(stream)
        rb.walk(num_walkers=V, seed=1000 + i, lengths=out_len, **wkw)      # this rank's walker share
        if ev is not None:
            ev[2].record(stream)
        if app == "ppr":
            rb.visit_counts(reset=True)                                     # the one all-reduce
        if ev is not None:
            ev[3].record(stream)

    for i in range(W):
        step(i, scratch_len)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    launches0 = g.info()["kernel_launches"]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    start.record(stream)
    for k in range(K):
        step(W + k, lens[k], evs[k])
    end.record(stream)
    torch.cuda.synchronize()
    launches = g.info()["kernel_launches"] - launches0
    clk = clocks.stop()
    t_ms = start.elapsed_time(end)
    upd_ms = [e[0].elapsed_time(e[1]) for e in evs]
    walk_ms = [e[1].elapsed_time(e[2]) for e in evs]
    red_ms = [e[2].elapsed_time(e[3]) for e in evs]
    steps_local = sum(int(x.to(torch.int64).sum()) for x in lens)
    t_local = t_ms
    if dist is not None:
        t = torch.tensor([t_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t)
        s = torch.tensor([steps_local], device=dev, dtype=torch.int64)
        dist.all_reduce(s)
        steps_total = int(s)
    else:
        steps_total = steps_local
    value = steps_total / (t_ms / 1e3)
    walk_avg_s = statistics.mean(walk_ms) / 1e3

    # ---- roofline of the dominant kernel (k_walk): algorithmic bytes of one launch of the
    # same configuration from exact per-record load counts (bingo_walk_profile)
    pkw = dict(app=wkw["app"], length=wkw["length"], stop=(1, 80), seed=1000 + W, first_walker=first,
               num_walkers=count, paths=(app != "ppr"))
    prof = g.walk_profile(**pkw)
    gather_sectors = prof["hdr"] + prof["bkt"] + prof["mem"] + prof["arc"]
    gather_bytes = 32 * gather_sectors
    alg_bytes = gather_bytes + 4 * count                                   # + lengths
    if app == "ppr":
        alg_bytes += 64 * (prof["visit"] + prof["walkers"])                # counter RMW: 2 sectors per visit
    else:
        alg_bytes += 4 * count * (L + 1)                                   # path columns
    pk, pk_src = peaks()
    peak = float(pk["hbm_gbs"])
    achieved = alg_bytes / walk_avg_s / 1e9
    g.reset_visit_counts()

    # in-run DRAM counters of one walk launch (CUPTI), same configuration
    traffic, meter_note, l2_hit = None, "skipped", None
    if not args.no_meter:
        mk = dict(pkw)
        mk.pop("paths")
        mk["paths"] = paths if app != "ppr" else None
        mk["lengths"] = scratch_len

        def one_walk():
            g.walk(**mk)
        vals, meter_note = Meter().measure(one_walk)
        if vals:
            traffic = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
            l2_hit = vals["lts__t_sector_hit_rate.pct"]
        g.reset_visit_counts()

    # gather ceiling for the walk's own footprint and skew: trace + dependency-free replay
    ceiling = None
    if not args.no_ceiling:
        ceiling = gather_ceiling(args, g, app, pkw, prof, count, first, dev, stream)
        g.reset_visit_counts()
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "peak_source": f"{pk_src} hbm_gbs (MEASURED_PEAKS.json copy bandwidth)",
            "kernel": f"k_walk<{app.upper()}> (bingo_walk)", "alg_bytes_per_launch": alg_bytes,
            "alg_bytes_def": ("32 B x (vertex headers + alias buckets + members + dense arc attempts) "
                              + ("+ 64 B x visit-counter RMWs " if app == "ppr" else "+ 4 B x path entries ")
                              + "+ 4 B x lengths; exact counts from bingo_walk_profile of the same launch"),
            "load_counts": {k: prof[k] for k in ("steps", "hdr", "bkt", "mem", "arc", "visit", "walkers")},
            "traffic_source": f"CUPTI range profiler in this run (dram__bytes_read.sum + dram__bytes_write.sum): "
                              f"{meter_note}",
            "dram_gbs": (traffic / walk_avg_s / 1e9) if traffic else None,
            "dram_frac_of_peak": (traffic / walk_avg_s / 1e9 / peak) if traffic else None,
            "l2_sector_hit_pct": l2_hit}
    if ceiling:
        walk_gather_gbs = gather_bytes / walk_avg_s / 1e9
        ceiling["walk_gather_gbs"] = walk_gather_gbs
        ceiling["frac"] = walk_gather_gbs / ceiling["ceiling_gbs"]
        ceiling["north_star_target"] = ">= 0.5 of the achievable random-gather bandwidth (BASELINE north_star)"
        ceiling["north_star_met"] = ceiling["frac"] >= 0.5
        roof["gather_ceiling"] = ceiling
    out = {"value": value, "t_ms": t_ms, "t_local_ms": t_local, "K": K, "steps_total": steps_total,
           "launches": int(launches), "clocks": clk, "roofline": roof, "V": V, "A": A, "nrec": nrec,
           "update_ms": statistics.mean(upd_ms), "walk_ms": walk_avg_s * 1e3,
           "allreduce_ms": statistics.mean(red_ms), "setup": times, "first": first, "count": count}

    # ---- e2e through the public API with HOST buffers: batch H2D in, result D2H out
    if e2e_steps:
        out["e2e"] = run_e2e(args, g, rb, batches[W + K:W + K + e2e_steps], app, V, count, first, L, dev, dist, rank,
                             ws)
    # ---- a11: streaming single-record updates (synchronous C-ABI calls, host batch)
    if not primary and rank == 0:
        out["streaming"] = streaming(g, batches, stream)
    out["host_csr"] = host_csr
    out["batches"] = batches
    g.close()
    del g, rb, dev_batches, paths, lens
    torch.cuda.empty_cache()
    return out


def gather_ceiling(args, g, app, pkw, prof, count, first, dev, stream):
    """Record the walk's own loads (bingo_walk_trace) for a prefix of this rank's walkers and
    replay them with no dependency between loads (bingo_walk_replay): the bandwidth the memory
    system delivers for exactly this footprint, skew and cache-policy mix when latency is
    hidden -- the denominator of the north_star's 'achievable random-gather bandwidth'."""
    import torch
    lens = (prof["lengths"].to(torch.int64) if prof.get("lengths") is not None else None)
    if lens is None:
        return None
    cum = torch.cumsum(lens, 0)
    budget = int(min(args.trace_records, (torch.cuda.mem_get_info()[0] * 0.6) / 16))
    Wt = int(torch.searchsorted(cum, torch.tensor([budget], device=cum.device), right=True)[0])
    Wt = max(1, min(Wt, count))
    n = int(cum[Wt - 1])
    rec_off = torch.zeros(Wt + 1, dtype=torch.int64, device=dev)
    rec_off[1:] = cum[:Wt]
    trace = torch.empty((n, 4), dtype=torch.int32, device=dev)
    kw = dict(app=pkw["app"], length=pkw["length"], stop=pkw["stop"], seed=pkw["seed"], first_walker=first,
              num_walkers=Wt)
    tp = g.walk_trace(rec_off, trace, **kw)
    assert tp["steps"] == n, (tp["steps"], n)
    # the ceiling is the best replay over a sweep of in-flight depth x occupancy (more
    # concurrency is not always faster here: concurrent cold misses contend for translation)
    sweep = {}
    cnt = None
    for ahead in (1, 2, 4, 8):
        for bps in (2, 4, 6, 8, 16):
            ms = []
            for _ in range(2):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                cnt = g.walk_replay(trace, rec_off, ahead=ahead, blocks_per_sm=bps)
                e1.record(stream)
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            sweep[f"ahead{ahead}_bps{bps}"] = min(ms)
    best = min(sweep, key=sweep.get)
    rep_ms = sweep[best]
    sectors = cnt["hdr"] + cnt["bkt"] + cnt["mem"] + cnt["arc"]
    walker_gbs = 32 * sectors / (rep_ms / 1e3) / 1e9
    # second order: the same records sorted by vertex inside windows of one walker per vertex
    # (what one step of a level-synchronous walk over every walker could issue; DESIGN 6.1,
    # tools/sorted_replay.py), replayed in chunks of 8 records per thread
    del rec_off
    torch.cuda.empty_cache()
    srt = None
    try:
        V = g.V
        n2 = int(min(n, args.sort_records, torch.cuda.mem_get_info()[0] * 0.8 / 40))
        key = trace[:n2, 0].to(torch.int64) + (torch.arange(n2, device=dev, dtype=torch.int64) // V << 40)
        idx = torch.sort(key).indices
        del key
        st = trace[:n2].index_select(0, idx)
        del idx
        coff = torch.unique_consecutive(torch.arange(0, n2 + 8, 8, dtype=torch.int64, device=dev).clamp_(max=n2))
        ssweep, scnt = {}, None
        for ahead in (1, 8):
            for bps in (2, 4):
                ms = []
                for _ in range(2):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    scnt = g.walk_replay(st, coff, ahead=ahead, blocks_per_sm=bps)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ms.append(e0.elapsed_time(e1))
                ssweep[f"ahead{ahead}_bps{bps}"] = min(ms)
        sbest = min(ssweep, key=ssweep.get)
        ssect = scnt["hdr"] + scnt["bkt"] + scnt["mem"] + scnt["arc"]
        srt = {"records": n2, "window_records": V, "replay_ms": ssweep[sbest], "replay_best": sbest,
               "replay_sweep_ms": ssweep, "ceiling_gbs": 32 * ssect / (ssweep[sbest] / 1e3) / 1e9}
        del st, coff
    except torch.cuda.OutOfMemoryError:
        srt = {"skipped": "not enough free memory for the sort"}
    del trace
    torch.cuda.empty_cache()
    ceil_gbs = max(walker_gbs, srt.get("ceiling_gbs", 0.0))
    return {"method": "bingo_walk_trace + bingo_walk_replay: the traced walks' own loads (header, bucket, "
                      "member / first two dense attempts) re-issued walker by walker with the walk's widths, L2 "
                      "policies and 64 B fetch hints, but 1-8 steps (up to 32 loads) in flight per thread and no "
                      "dependency, 2-16 blocks of 256 per SM; the best of that sweep: the walk with perfect "
                      "prefetching.  ceiling = 32 B x "
                      "loads / replay time; the replay also streams the 16 B trace record of every step, so the "
                      "ceiling is, if anything, low by that share.  PPR visit-counter RMWs are not replayed "
                      "(they cost the walk time, so the fraction understates)",
            "walkers_traced": Wt, "steps_traced": n, "replay_ms": rep_ms, "replay_best": best,
            "replay_sweep_ms": sweep, "replay_loads": cnt, "walker_order_gbs": walker_gbs,
            "window_sorted": srt,
            "ceiling_def": "the better of the two orders: walker by walker (the walk's own order), and sorted "
                           "by vertex inside windows of one walker per vertex (a level-synchronous order)",
            "ceiling_gbs": ceil_gbs}


def run_e2e(args, g, rb, host_batches, app, V, count, first, L, dev, dist, rank, ws):
    import torch
    import paper_2504_10233_b200 as pb
    stream = torch.cuda.current_stream()
    hb = [torch.from_numpy(b.view(np.int32)).pin_memory() for b in host_batches]
    nrec = host_batches[0].shape[0]
    if app == "ppr":
        # step k's counts go to host buffer k % 2 on a copy stream, overlapping step k + 1's walk
        # (the D2H of 370 MB at c4 is ~7 ms); every copy completes inside the timed region
        hcs = [torch.empty(V, dtype=torch.int64).pin_memory() for _ in range(2)]
        cstream = torch.cuda.Stream(device=dev)
        tot = torch.zeros(1, dtype=torch.int64, device=dev)
    else:
        hp = torch.empty((L + 1, count), dtype=torch.int32).pin_memory()
        hls = [torch.empty(count, dtype=torch.int32).pin_memory() for _ in host_batches]
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k, b in enumerate(hb):
        if ws == 1:
            g.apply_updates(b.numpy().view(np.uint32))                       # HOST batch through the C-ABI
        else:
            rb.apply_updates(b.to(dev, non_blocking=True) if rank == 0 else None, n=nrec)
        if app == "ppr":
            rb.walk(num_walkers=V, app=pb.PPR, length=pb.NO_CAP, stop=(1, 80), seed=5000 + k, paths=None,
                    lengths=None)
            c = rb.visit_counts(reset=True)
            tot += c.sum()
            cstream.wait_stream(stream)
            with torch.cuda.stream(cstream):
                hcs[k % 2].copy_(c, non_blocking=True)                       # the result, D2H
            c.record_stream(cstream)
        else:
            g.walk_host(app=pb.DEEPWALK, length=L, seed=5000 + k, first_walker=first, num_walkers=count, paths=hp,
                        lengths=hls[k])
    if app == "ppr":
        stream.wait_stream(cstream)
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = e0.elapsed_time(e1)
    if app == "ppr":
        steps = int(tot) - V * len(hb)            # sum(counts) = sum(lengths + 1) over all walkers
        if dist is not None and ws > 1:
            steps = steps                         # counts are already all-reduced: global steps
    else:
        steps = sum(int(h.numpy().astype(np.int64).sum()) for h in hls)
    if dist is not None:
        t = torch.tensor([e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t)
        if app != "ppr":
            s = torch.tensor([steps], device=dev, dtype=torch.int64)
            dist.all_reduce(s)
            steps = int(s)
    d2h = 8 * V if app == "ppr" else 4 * count * (L + 2)
    return {"value": steps / (e_ms / 1e3), "unit": "steps/s", "h2d_bytes_per_step": int(nrec * 16),
            "d2h_bytes_per_step": int(d2h), "steps": len(hb),
            "note": ("bingo_apply_updates(HOST batch) + bingo_walk(PPR) + all-reduced visit counts copied to "
                     "pinned host memory each step (on a copy stream, overlapping the next step's walk; all "
                     "copies complete inside the timed region)" if app == "ppr" else
                     "bingo_apply_updates(HOST batch) + bingo_walk(HOST_OUTPUT paths+lengths), pinned")}


def streaming(g, batches, stream):
    """One bingo_apply_updates call per arc record, through the Python binding and raw ctypes."""
    import torch
    from paper_2504_10233_b200 import bingo as bb
    recs = batches[-1][:300]
    lat_host, lat_dev = [], []
    for r in recs:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        g.apply_updates(r[None, :])
        e1.record(stream)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        lat_host.append(1e6 * (t1 - t0))
        lat_dev.append(1e3 * e0.elapsed_time(e1))
    packed = np.ascontiguousarray(batches[-2][:300], dtype=np.uint32)
    lib, h, sp = bb._lib(), g.handle, stream.cuda_stream
    base = packed.ctypes.data
    lat_c = []
    for i in range(len(packed)):
        t0 = time.perf_counter()
        rc = lib.bingo_apply_updates(h, base + 16 * i, 1, bb.UPD_HOST_BATCH, None, sp)
        lat_c.append(1e6 * (time.perf_counter() - t0))
        assert rc == 0, rc
    # f2: the same kind of records through the persistent streaming queue (bingo_stream_update):
    # raw C-ABI call, host post -> device apply -> host sees the result
    qrec = np.ascontiguousarray(batches[-3][:2000], dtype=np.uint32)
    st = bb.UpdateStats()
    qbase = qrec.ctypes.data
    lat_q = []
    for i in range(len(qrec)):
        t0 = time.perf_counter()
        rc = lib.bingo_stream_update(h, qbase + 16 * i, ctypes.byref(st), sp)
        lat_q.append(1e6 * (time.perf_counter() - t0))
        assert rc == 0, rc
    # the queue's own round trip: records rejected by validation (src = V) do no graph work
    bad = np.array([[0, 0xFFFFFFFF, 0, 1]] * 300, dtype=np.uint32)
    lat_b = []
    for i in range(len(bad)):
        t0 = time.perf_counter()
        rc = lib.bingo_stream_update(h, bad.ctypes.data + 16 * i, None, sp)
        lat_b.append(1e6 * (time.perf_counter() - t0))
        assert rc == bb.E_INVAL, rc
    torch.cuda.synchronize()
    return {"records": len(recs), "queue_records": len(lat_q),
            "queue_roundtrip_us_p50": float(np.percentile(lat_b, 50)),
            "queue_us_p50": float(np.percentile(lat_q, 50)), "queue_us_p90": float(np.percentile(lat_q, 90)),
            "queue_us_p99": float(np.percentile(lat_q, 99)),
            "queue_updates_per_s": float(len(lat_q) / (1e-6 * sum(lat_q))),
            "call_us_p50": float(np.percentile(lat_host, 50)),
            "call_us_p99": float(np.percentile(lat_host, 99)),
            "device_us_p50": float(np.percentile(lat_dev, 50)), "device_us_p99": float(np.percentile(lat_dev, 99)),
            "abi_call_us_p50": float(np.percentile(lat_c, 50)), "abi_call_us_p99": float(np.percentile(lat_c, 99)),
            "abi_updates_per_s": float(len(lat_c) / (1e-6 * sum(lat_c))),
            "note": "one call per arc record (epoch per record); queue_us: bingo_stream_update (persistent "
                    "device-side queue, no launch per record), host to completion via ctypes; call_us: "
                    "bingo_apply_updates through the Python binding; abi_call_us: bingo_apply_updates via ctypes"}


# ---------------------------------------------------------------- the oracle (CPU) legs
def oracle_sample(host_csr, batches, config, steps_idx, walkers, V, seed_base, warm=True):
    """The oracle as it stands (lazy build: vertices are materialised on first access), per
    step: one full update batch (single-threaded) + a sample of the step's walkers (OpenMP,
    all host cores).  First-touch materialisation is never billed: the batch's vertices are
    materialised before the update is timed, and the walk is timed on a second pass over
    the same walkers."""
    import oracle
    app = app_of(config)
    oapp = {"ppr": oracle.APP_PPR, "deepwalk": oracle.APP_DEEPWALK}[app]
    length = oracle.NONE if app == "ppr" else 80
    o = oracle.OracleGraph(*host_csr, lazy=True)
    out = []
    for i in steps_idx:
        # first-touch materialisation of the batch's vertices is not update work: done untimed
        o.touch(np.unique(batches[i][:, 1:3]), threads=os.cpu_count())
        t0 = time.perf_counter()
        o.apply_updates(batches[i])
        t_upd = time.perf_counter() - t0
        first = (i * 7919 * 4099) % max(1, V - walkers)
        kw = dict(app=oapp, length=length, seed=seed_base + i, first_walker=first, num_walkers=walkers,
                  paths=False, counts=(app == "ppr"), threads=os.cpu_count())
        if warm:
            o.walk(**kw)
        t0 = time.perf_counter()
        r = o.walk(**kw)
        t_walk = time.perf_counter() - t0
        out.append((t_upd, t_walk, int(r["lengths"].astype(np.int64).sum())))
    return out


def cpu_line_from(samples, V, walkers, nrec):
    t_upd = sum(s[0] for s in samples)
    t_walk = sum(s[1] for s in samples)
    steps = sum(s[2] for s in samples)
    scale = V / walkers
    t_full = t_upd + t_walk * scale
    return steps * scale / t_full, {"update_s_per_batch": t_upd / len(samples), "walk_s_per_sample": t_walk / len(samples),
                                   "walk_steps_per_s": steps / t_walk, "update_arcs_per_s": nrec * len(samples) / t_upd,
                                   "scale": scale}


def run_reference(args):
    """--impl reference: the oracle as it stands, on the host cores, on the same workload as the
    CUDA arm (same graph, same batches); each step = one full update batch + a walker sample
    of the step, scaled to one walker per vertex.  Only rank 0 runs."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    import torch
    import synth
    config = args.config
    dev = torch.device("cuda", local) if torch.cuda.is_available() else torch.device("cpu")
    rounds = args.warmup + args.steps
    t0 = time.time()
    w = synth.make_workload(config, rounds=rounds, hold_rounds=HOLD_ROUNDS, device=dev,
                            resident=dev.type == "cuda")
    host = w.host_csr() if hasattr(w, "host_csr") else (w.row_offsets, w.dst, w.bias)
    V, A, nrec = w.V, w.num_arcs, w.batches[0].shape[0]
    batches = w.batches
    del w
    if dev.type == "cuda":
        torch.cuda.empty_cache()
    gen_s = time.time() - t0
    walkers = min(V, max(1, args.cpu_walkers // 4))
    samples = oracle_sample(host, batches, config, range(rounds), walkers, V, 1000, warm=True)
    timed = samples[args.warmup:]
    val, det = cpu_line_from(timed, V, walkers, nrec)
    ms_step = 1e3 * (sum(s[0] for s in timed) + det["scale"] * sum(s[1] for s in timed)) / len(timed)
    sample = (f"per step: 1 full update batch ({nrec} arc records, single-threaded, lazy oracle, its vertices "
              f"materialised untimed) + "
              f"{app_of(config)} walk of {walkers} walkers (OpenMP, {os.cpu_count()} threads; second pass over the "
              f"same walkers, the first materialises their vertices), walk time scaled x{det['scale']:.1f} to "
              f"{V} walkers; generation {gen_s:.0f} s (torch on the GPU, not timed)")
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": val, "unit": "steps/s", "n_gpus": ws,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                      "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
                      "config": config_block(config, V, A, nrec, 1, {"parallelism": "oracle on host cores"}),
                      "cpu_baseline": {"value": val, "unit": "steps/s", "cores": os.cpu_count(), "kind": "oracle",
                                       "sample": sample, **det},
                      "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    ws, rank, local = dist_env()
    if args.share_device:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    numa_cpus = bind_to_gpu_numa(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    head = run_workload(args, args.config, dev, ws, rank, local, dist, primary=True)
    sec = None
    if args.secondary:
        sec = run_workload(args, args.secondary, dev, ws, rank, local, dist, primary=False)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and head["host_csr"] is not None:
        walkers = min(head["V"], args.cpu_walkers)
        samples = oracle_sample(head["host_csr"], head["batches"], args.config, [0], walkers, head["V"], 99)
        val, det = cpu_line_from(samples, head["V"], walkers, head["nrec"])
        cpu = {"value": val, "unit": "steps/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": (f"lazy oracle on the same graph: 1 update batch of {head['nrec']} arc records "
                          f"(single-threaded) + {app_of(args.config)} walk of {walkers} walkers (OpenMP; timed on a "
                          f"second pass, the first materialises their vertices), walk scaled x{det['scale']:.0f} to "
                          f"the full step"), **det}
    if rank == 0:
        K = args.steps
        line = {
            "metric": METRIC, "value": head["value"], "unit": "steps/s", "n_gpus": ws, "steps": K,
            "warmup": args.warmup, "ms_per_step": head["t_ms"] / K, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config_block(args.config, head["V"], head["A"], head["nrec"], ws,
                                   {"parallelism": f"replicated graph x{ws}, walker ids split {ws} ways, batch "
                                                   f"broadcast + visit-count all-reduce"
                                                   f" ({'NCCL' if args.backend == 'nccl' else args.backend})"
                                                   + (", every rank on one device (test)" if args.share_device else ""),
                                    "setup": head["setup"]}),
            "walk_steps_per_s": head["steps_total"] / K / (head["walk_ms"] / 1e3),
            "update_edges_per_s": head["nrec"] / (head["update_ms"] / 1e3),
            "update_ms": head["update_ms"], "walk_ms": head["walk_ms"], "allreduce_ms": head["allreduce_ms"],
            "roofline": head["roofline"], "clocks": head["clocks"], "gpu_launches": head["launches"],
            "e2e": head.get("e2e"), "cpu_baseline": cpu,
        }
        if sec is not None:
            line["secondary"] = {
                "config": config_block(args.secondary, sec["V"], sec["A"], sec["nrec"], ws,
                                       {"setup": sec["setup"]}),
                "value": sec["value"], "unit": "steps/s", "ms_per_step": sec["t_ms"] / K,
                "walk_steps_per_s": sec["steps_total"] / K / (sec["walk_ms"] / 1e3),
                "update_edges_per_s": sec["nrec"] / (sec["update_ms"] / 1e3), "update_ms": sec["update_ms"],
                "walk_ms": sec["walk_ms"], "roofline": sec["roofline"], "clocks": sec["clocks"],
                "gpu_launches": sec["launches"], "streaming_update": sec.get("streaming")}
        if numa_cpus:
            line["host_cpus"] = f"{len(numa_cpus)} CPUs local to the GPU"
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
