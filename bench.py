#!/usr/bin/env python
"""bench.py -- Bingo hot path on B200: batched updates + biased DeepWalk, the paper's
protocol (S6.1: rounds of (BATCHSIZE updates -> application)).

A step = one round on BASELINE.json configs[1] (LiveJournal-shaped R-MAT, 4.7M V /
69M arcs, degree biases): apply one update batch (50K undirected edge events = 100K
arc records, Mixed insert/delete) then one biased DeepWalk of one walker
per vertex x 80 steps, paths written to HBM.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU (torchrun): every rank holds a replica, rank 0's update batch is broadcast
(NCCL) inside the step, each rank walks its own walker-id range (weak scaling, one
walker per vertex per rank); time = max over ranks of the device-timed region.
"""
from __future__ import annotations

import argparse
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--length", type=int, default=80)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-walkers", type=int, default=1 << 21,
                    help="oracle walker sample (cpu_baseline; --impl reference uses a quarter per step)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for N > 1 (gloo: test the multi-rank path without NVLink)")
    ap.add_argument("--share-device", action="store_true",
                    help="test only: every rank on cuda:0 (exercise the N > 1 code path on a 1-GPU box)")
    ap.add_argument("--e2e-layout", default="step", choices=["walker", "step"],
                    help="path layout of the e2e pass (walker-major: one contiguous D2H per chunk)")
    ap.add_argument("--layout", default="step", choices=["walker", "step"],
                    help="path layout written by the walk (walker-major: one contiguous walk per walker)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
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
    """Run this process on the CPUs local to the GPU, so pinned host buffers (first touch) sit on
    the GPU's NUMA node: a remote node cost the e2e pass ~40% of its PCIe bandwidth (7.5 vs 12.4
    G steps/s between runs).  Best effort: silently skipped where sysfs does not say."""
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


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        return ws, rank, local, dist
    return 1, 0, 0, None


def workload(args, rounds):
    import synth
    return synth.make_workload(args.config, rounds=rounds)


def config_block(args, w, extra=None):
    import synth
    cfg = synth.CONFIGS[args.config]
    c = {"workload": f"BASELINE configs[1]: {cfg['desc']}", "config": args.config, "V": int(w.V),
         "arcs": int(w.num_arcs), "walk": f"biased DeepWalk, {w.V} walkers (1/vertex) x {args.length} steps",
         "update_batch_arc_records": int(2 * w.batch), "update_batch_edges": int(w.batch),
         "bias": "w(u,v)=max(1,deg(v)) (P:664)", "alpha_beta": [40, 10],
         "l2": "inputs larger than L2: graph pools + 1.5 GB paths per step (> 126 MB L2), no flush needed"}
    if extra:
        c.update(extra)
    return c


def run_reference(args):
    """The oracle as it stands, on host cores, on the same workload: a bounded sample per step
    (one full update batch + a walker sample), scaled to the full step."""
    ws, rank, _, dist = dist_setup(args)
    if rank != 0:
        return
    import oracle
    w = workload(args, args.warmup + args.steps)
    o = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    Ws = min(w.V, args.cpu_walkers // 4)
    ncores = os.cpu_count()
    times, steps_full = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        o.apply_updates(w.batches[i])
        t1 = time.perf_counter()
        r = o.walk(length=args.length, seed=1000 + i, first_walker=(i * 7919) % w.V, num_walkers=Ws, paths=True)
        t2 = time.perf_counter()
        sample_steps = int(r["lengths"].astype(np.int64).sum())
        full_steps = sample_steps * (w.V / Ws)
        t_step = (t1 - t0) + (t2 - t1) * (w.V / Ws)
        if i >= args.warmup:
            times.append(t_step)
            steps_full.append(full_steps)
    T = sum(times)
    val = sum(steps_full) / T
    sample = (f"per step: 1 full update batch ({2 * w.batch} arc records, single-threaded) + DeepWalk of {Ws} "
              f"walkers x {args.length} steps (OpenMP, all cores), walk time scaled x{w.V / Ws:.1f} to {w.V} walkers")
    print(json.dumps({"impl": "reference", "metric": "walk steps/s (round = update batch + DeepWalk)",
                      "value": val, "unit": "steps/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                      "ms_per_step": 1e3 * T / len(times), "higher_is_better": True, "scaling": "weak",
                      "vs_baseline": None, "dtype": "u32", "data": "synthetic",
                      "config": config_block(args, w),
                      "cpu_baseline": {"value": val, "unit": "steps/s", "cores": ncores, "kind": "oracle",
                                       "sample": sample},
                      "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


def cpu_baseline(args, w, batch):
    import oracle
    t0 = time.perf_counter()
    o = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    o.apply_updates(batch)
    t_upd = time.perf_counter() - t0
    Ws = min(w.V, args.cpu_walkers)
    t0 = time.perf_counter()
    r = o.walk(length=args.length, seed=99, num_walkers=Ws, paths=True)
    t_walk = time.perf_counter() - t0
    steps = int(r["lengths"].astype(np.int64).sum())
    scale = w.V / Ws
    t_step = t_upd + t_walk * scale
    return {"value": steps * scale / t_step, "unit": "steps/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": (f"oracle built once (untimed, {t_build:.1f} s); 1 update batch of {len(batch)} arc records "
                       f"({t_upd:.2f} s, single-threaded) + DeepWalk of {Ws} walkers x {args.length} steps "
                       f"({t_walk:.2f} s, OpenMP); walk scaled x{scale:.1f} to the full step"),
            "walk_steps_per_s": steps / t_walk, "update_arcs_per_s": len(batch) / t_upd}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    ws, rank, local, dist = dist_setup(args)
    if args.share_device:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    numa_cpus = bind_to_gpu_numa(local)
    if dist is not None:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    import paper_2504_10233_b200 as pb
    from paper_2504_10233_b200 import bingo

    K, W = args.steps, args.warmup
    e2e_steps = 0 if args.no_e2e else K
    rounds = W + K + e2e_steps + 1
    w = workload(args, rounds)
    V, L = w.V, args.length
    g = pb.Graph(w.row_offsets, w.dst, w.bias, device=dev)
    batches = [torch.from_numpy(b.view(np.int32)) for b in w.batches]
    nrec = batches[0].shape[0]
    # inputs resident in HBM before the timed region (rank 0 holds the stream; others receive it)
    dev_batches = [b.to(dev) for b in batches[:W + K]] if rank == 0 else [None] * (W + K)
    first = rank * V            # this rank's first walker id (weak scaling: V walkers per rank)
    wmajor = args.layout == "walker"
    paths = torch.empty((V, L + 1) if wmajor else (L + 1, V), dtype=torch.int32, device=dev)
    lens = [torch.empty(V, dtype=torch.int32, device=dev) for _ in range(K)]
    scratch_len = torch.empty(V, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    from paper_2504_10233_b200.distributed import ReplicatedBingo
    rb = ReplicatedBingo(g, device=dev)

    def step(i, out_len, ev=None):
        if ev is not None:
            ev[0].record(stream)
        # rank 0's batch is broadcast to every replica inside the step (NCCL over NVLink)
        rb.apply_updates(dev_batches[i] if rank == 0 else None)
        if ev is not None:
            ev[1].record(stream)
        # walker ids [rank*V, (rank+1)*V): one walker per vertex per rank (weak scaling)
        rb.walk(num_walkers=V * ws, app=pb.DEEPWALK, length=L, seed=1000 + i, paths=paths, lengths=out_len,
                walker_major=wmajor)
        if ev is not None:
            ev[2].record(stream)

    for i in range(W):
        step(i, scratch_len)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
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
    steps_local = sum(int(x.to(torch.int64).sum()) for x in lens)
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

    # ---- roofline of the dominant kernel (the walk): algorithmic bytes from an exact
    # per-record load count of one launch of the same configuration
    prof = g.walk_profile(app=pb.DEEPWALK, length=L, seed=1000 + W, first_walker=first, num_walkers=V)
    sectors = prof["hdr"] + prof["bkt"] + prof["mem"] + prof["arc"]
    alg_bytes = 32 * sectors + 4 * V * (L + 1) + 4 * V          # dependent 32 B sectors + path + lengths
    walk_avg_s = statistics.mean(walk_ms) / 1e3
    pk, pk_src = peaks()
    peak = float(pk["hbm_gbs"])
    achieved = alg_bytes / walk_avg_s / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "walk_dram_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                traffic = json.load(f).get("bytes_per_launch")
        except Exception:
            traffic = None
    gather = measure_gather(dev) if rank == 0 else None

    # ---- e2e through the C-ABI with HOST buffers (pinned): H2D batch + D2H paths each step
    e2e = None
    if e2e_steps:
        ewm = args.e2e_layout == "walker"
        hp = torch.empty((V, L + 1) if ewm else (L + 1, V), dtype=torch.int32).pin_memory()
        # one pinned lengths buffer per step: the step counts are summed after the timed region
        hls = [torch.empty(V, dtype=torch.int32).pin_memory() for _ in range(e2e_steps)]
        hb = [b.pin_memory() for b in batches[W + K:W + K + e2e_steps]]
        # one untimed pass through the host buffers (first DMA into freshly pinned pages)
        g.walk_host(app=pb.DEEPWALK, length=L, seed=4999, first_walker=first, num_walkers=V, paths=hp,
                    lengths=hls[0], walker_major=ewm)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0
        e0.record(stream)
        for k in range(e2e_steps):
            g.apply_updates(hb[k].numpy())
            g.walk_host(app=pb.DEEPWALK, length=L, seed=5000 + k, first_walker=first, num_walkers=V,
                        paths=hp, lengths=hls[k], walker_major=ewm)
        e1.record(stream)
        torch.cuda.synchronize()
        tot = sum(int(h.numpy().astype(np.int64).sum()) for h in hls)
        e_ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t)
            s = torch.tensor([tot], device=dev, dtype=torch.int64)
            dist.all_reduce(s)
            tot = int(s)
        e2e = {"value": tot / (e_ms / 1e3), "unit": "steps/s", "h2d_bytes_per_step": int(nrec * 16),
               "host_cpus": f"{len(numa_cpus)} CPUs local to the GPU" if numa_cpus else "unbound",
               "d2h_bytes_per_step": int(4 * V * (L + 2)), "steps": e2e_steps,
               "path_layout": "walker-major" if ewm else "step-major",
               "note": "bingo_apply_updates(HOST batch) + bingo_walk(HOST_OUTPUT paths+lengths), pinned"}

    # ---- a11: streaming single-record updates (synchronous C-ABI calls, host batch)
    streaming = None
    if rank == 0:
        recs = w.batches[-1][:300]
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
        # the same C-ABI call without the Python wrapper (ctypes directly on pre-packed records):
        # the library's own per-record latency, host call to completion
        from paper_2504_10233_b200 import bingo as bb
        packed = np.ascontiguousarray(w.batches[-2][:300], dtype=np.uint32)
        lib, h, sp = bb._lib(), g.handle, stream.cuda_stream
        base = packed.ctypes.data
        lat_c = []
        for i in range(len(packed)):
            t0 = time.perf_counter()
            rc = lib.bingo_apply_updates(h, base + 16 * i, 1, bb.UPD_HOST_BATCH, None, sp)
            lat_c.append(1e6 * (time.perf_counter() - t0))
            assert rc == 0, rc
        streaming = {"records": len(recs), "call_us_p50": float(np.percentile(lat_host, 50)),
                     "call_us_p99": float(np.percentile(lat_host, 99)),
                     "device_us_p50": float(np.percentile(lat_dev, 50)),
                     "device_us_p99": float(np.percentile(lat_dev, 99)),
                     "abi_call_us_p50": float(np.percentile(lat_c, 50)),
                     "abi_call_us_p99": float(np.percentile(lat_c, 99)),
                     "abi_updates_per_s": float(len(lat_c) / (1e-6 * sum(lat_c))),
                     "note": "one bingo_apply_updates call per arc record (epoch per record), c2 graph; call_us: "
                             "through the Python binding; abi_call_us: the C-ABI call via ctypes, host to "
                             "completion (the library synchronises)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, w, w.batches[0])

    if rank == 0:
        upd_avg = statistics.mean(upd_ms) / 1e3
        line = {
            "metric": "walk steps/s (round = update batch + DeepWalk)",
            "value": value, "unit": "steps/s", "n_gpus": ws, "steps": K, "warmup": W,
            "ms_per_step": t_ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config_block(args, w, {"parallelism": f"replicated graph x{ws}, walkers sharded by id",
                                             "path_layout": "walker-major" if wmajor else "step-major"}),
            "walk_steps_per_s": steps_total / ws / K / walk_avg_s * ws,
            "update_edges_per_s": nrec / upd_avg,
            "update_ms": upd_avg * 1e3, "walk_ms": walk_avg_s * 1e3,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "peak_source": f"{pk_src} hbm_gbs (MEASURED_PEAKS.json copy bandwidth)",
                         "kernel": "k_walk<DEEPWALK> (bingo_walk)",
                         "alg_bytes_per_launch": alg_bytes,
                         "alg_bytes_def": "32 B x (vertex headers + alias buckets + members + dense arc attempts) "
                                          "+ 4 B x path entries + 4 B x lengths, exact counts from bingo_walk_profile",
                         "load_counts": {k: prof[k] for k in ("steps", "hdr", "bkt", "mem", "arc")},
                         "gather_roofline": gather},
            "l2_plan": {"l2_persist_bytes": g.info()["l2_persist_bytes"],
                        "hot_bucket_degree": g.info()["hot_degree"] & 0xFFFFFFFF,
                        "hot_member_degree": g.info()["hot_degree"] >> 32},
            "streaming_update": streaming,
            "clocks": clk, "gpu_launches": int(launches),
            "e2e": e2e, "cpu_baseline": cpu,
        }
        if gather and gather.get("chase1_gbs"):
            line["roofline"]["frac_of_gather_chase"] = achieved / gather["chase1_gbs"]
            line["roofline"]["frac_of_gather_independent"] = achieved / gather["independent_gbs"]
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def measure_gather(dev):
    """Random 32 B-sector gather bandwidth over 8 GiB (>> L2): independent loads (8 in flight
    per thread) and dependent pointer chases (1/2/4 chains per thread, the walker pattern)."""
    import ctypes
    import torch
    from paper_2504_10233_b200 import _build
    lib_path = _build.TOOLS_LIB
    if not os.path.exists(lib_path):
        return None
    L = ctypes.CDLL(lib_path)
    L.gather_fill.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
    L.gather_run.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                             ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float),
                             ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]
    nbytes = 8 << 30
    try:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    except RuntimeError:
        return None
    scratch = torch.zeros(16, dtype=torch.int32, device=dev)
    nslots = nbytes // 32
    s = torch.cuda.current_stream().cuda_stream
    L.gather_fill(buf.data_ptr(), nslots, 12345, s)
    torch.cuda.synchronize()
    out = {"buffer_gib": 8}
    for mode, name, blocks, threads, iters in ((0, "independent", 148 * 8, 256, 64), (1, "chase1", 148 * 8, 256, 64),
                                               (2, "chase2", 148 * 8, 256, 32), (3, "chase4", 148 * 8, 256, 16)):
        best = 0.0
        for rep in range(3):
            ms = ctypes.c_float()
            loads = ctypes.c_double()
            L.gather_run(buf.data_ptr(), nslots, mode, blocks, threads, iters, 777 + rep, scratch.data_ptr(),
                         ctypes.byref(ms), ctypes.byref(loads), s)
            best = max(best, 32 * loads.value / (ms.value / 1e3) / 1e9)
        out[name + "_gbs"] = best
    del buf
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
