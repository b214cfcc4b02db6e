#!/usr/bin/env python
"""bench.py -- the hot path on B200: SFC reorder -> linear-octree build -> fixed-radius search.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg1]

One step = one pass of the hot path over the config's synthetic cloud: encode + radix sort
+ gather (reorder_cloud), octree build (LinearOctree), then a full radius batch (count ->
u64 scan -> fill, every point a query) at every radius of the config.  `value` is radius
queries/s over the whole step with the cloud already resident in HBM; `e2e` is the same
metric through the C ABI with host buffers (pinned H2D of the cloud, D2H of each batch's
counts + FNV digests -- BatchResult's default content, search.hpp:121-131).  The kNN batches
of cfg2 (same cloud) are timed after the main region and reported under "knn".

Multi-GPU (torchrun, one rank per GPU): rank 0 reorders + builds, the structure is broadcast
over NCCL, each rank searches its contiguous SFC slice of the queries (strong scaling: the
total work is the config's fixed batch).  Time = max over ranks of CUDA-event time.

`--impl reference` times the reference's own CPU implementation (oracle/_ref, compiled from
the reference sources) on this host with all its threads, same config / metric / unit, on a
bounded sample (full-size reorder + build, radius on a contiguous slice of the sorted
centres, extrapolated to the full batch).
"""
from __future__ import annotations

import argparse
import ctypes as C
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

PEAKS = {"hbm_gbs": 6542.7}
try:
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        PEAKS.update(json.load(f))
        PEAK_SRC = "measured (MEASURED_PEAKS.json hbm_gbs)"
except OSError:
    PEAKS["hbm_gbs"] = 6650.0
    PEAK_SRC = "fallback (B200_PROFILING.md 6.65 TB/s)"

# SURVEY.md §8d.  Seeds: cfg i -> 1000 + i.
CONFIGS = {
    "cfg0": dict(kind="uniform", n=1_000_000, seed=1000, extent=100.0, curve=0, n_max=32,
                 radii=[2.5], ks=[], desc="1M uniform [0,100]^3, Morton, leaf 32, r=2.5"),
    "cfg1": dict(kind="terrain", n=10_000_000, seed=1001, extent=1000.0, curve=1, n_max=32,
                 radii=[0.5, 1.0, 2.0, 3.0], ks=[8, 16, 32, 64],
                 desc="10M terrain [0,1000]^2 (10 pts/m^2), Hilbert, leaf 32, r=0.5/1/2/3; "
                      "kNN k=8/16/32/64 on the same cloud (cfg2)"),
    "cfg3": dict(kind="mixed", n=100_000_000, seed=1003, extent=3000.0, curve=1, n_max=64,
                 radii=[1.0], ks=[16], desc="100M mixed (70% terrain/20% clusters/10% noise), "
                                            "Hilbert, leaf 64, r=1.0, kNN k=16"),
    "cfg4": dict(kind="uniform", n=50_000_000, seed=1004, extent=500.0, curve=1, n_max=32,
                 radii=[3.0], ks=[16], desc="50M uniform [0,500]^3, Hilbert, leaf 32, r=3.0, k=16"),
}


def generate(cfg):
    from paper_2603_06771_b200 import linoct as lo
    if cfg["kind"] == "uniform":
        return lo.generate_uniform(cfg["n"], cfg["seed"], cfg["extent"])
    if cfg["kind"] == "terrain":
        return lo.generate_terrain(cfg["n"], cfg["seed"], cfg["extent"])
    return lo.generate_mixed(cfg["n"], cfg["seed"])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 25 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * (mx or 1)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---- reference arm / CPU baseline -----------------------------------------------------------
def cpu_reference_step(cfg, xyz, sample: int, threads: int | None = None):
    """One bounded step of the reference CPU path: full-size reorder_cloud + LinearOctree
    (timed by the reference's own steady_clock in oracle/ref_driver.cpp), radius search
    over a contiguous slice of `sample` sorted centres per radius (neighbours_lin, dynamic
    OpenMP, FNV digests -- run_batch_loop's work), extrapolated to all n centres."""
    from oracle.oracle_py import Ref
    ref = Ref()
    th = threads or ref.max_threads()
    n = cfg["n"]
    p = ref.pipeline(xyz, cfg["curve"], cfg["n_max"], threads=th)
    t_reorder, t_build = float(p.timings[0]), float(p.timings[1])
    s = min(sample, n)
    b0 = (n - s) // 2
    t_search = 0.0
    mus = []
    for r in cfg["radii"]:
        wall, counts, _ = p.radius_range(r, b0, b0 + s, threads=th)
        t_search += wall * n / s
        mus.append(float(counts.mean()))
    t_step = t_reorder + t_build + t_search
    q = len(cfg["radii"]) * n
    knn = {}
    for k in cfg["ks"]:
        ks = max(1, s // 4)
        wall, _ = p.knn_range(k, b0, b0 + ks, threads=th)
        knn[str(k)] = n / (wall * n / ks)
    del p
    return dict(value=q / t_step, t_step=t_step, t_reorder=t_reorder, t_build=t_build,
                t_search=t_search, mu=mus, threads=th, sample=s, knn_qps=knn)


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    xyz = generate(cfg)
    sample = args.cpu_sample
    steps = []
    for i in range(args.warmup + args.steps):
        st = cpu_reference_step(cfg, xyz, sample)
        if i >= args.warmup:
            steps.append(st)
    v = statistics.median(s["value"] for s in steps)
    th = steps[0]["threads"]
    desc = (f"full-size reorder_cloud + LinearOctree, then neighbours_lin over a contiguous "
            f"slice of {steps[0]['sample']} sorted centres per radius, extrapolated to "
            f"{cfg['n']} centres; median of {len(steps)} steps")
    line = {
        "impl": "reference", "metric": metric_name(cfg), "value": v, "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(s["t_step"] for s in steps) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY.md §8d)", "config": config_block(args, cfg),
        "cpu_baseline": {"value": v, "unit": "queries/s", "cores": th, "kind": "reference",
                         "sample": desc},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "stages_s": {"reorder": statistics.median(s["t_reorder"] for s in steps),
                     "build": statistics.median(s["t_build"] for s in steps),
                     "search_extrapolated": statistics.median(s["t_search"] for s in steps)},
        "mu": steps[0]["mu"],
        "knn_qps": steps[0]["knn_qps"],
    }
    print(json.dumps(line), flush=True)
    return 0


def metric_name(cfg):
    return ("radius queries/s per hot-path step (reorder + octree build + full radius batch at "
            "each radius; " + cfg["desc"] + ")")


def config_block(args, cfg):
    return {"workload": args.config, "points": cfg["n"], "cloud": cfg["kind"],
            "curve": "hilbert" if cfg["curve"] else "morton", "leaf_bucket": cfg["n_max"],
            "radii": cfg["radii"], "knn_k": cfg["ks"], "queries_per_step": len(cfg["radii"]) * cfg["n"],
            "parallelism": (f"query-shard x{args.gpus} (" + ("structure built on every rank"
                                                            if os.environ.get("LO_BENCH_REPLICATE") == "1"
                                                            else "structure broadcast from rank 0") + ")")
            if args.gpus > 1 else "1 GPU",
            "l2": "inputs larger than L2 (cloud 24 B/pt + multi-GB CSR per step)"}


# ---- our arm --------------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2603_06771_b200 import _lib, linoct as lo
    from paper_2603_06771_b200 import distributed as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # test hooks for exercising the N > 1 code path on a single-GPU box (correctness only, the
    # numbers of such a run mean nothing): every rank on cuda:0, collectives over gloo
    if os.environ.get("LO_BENCH_SAME_DEVICE") == "1":
        local = 0
    backend = os.environ.get("LO_BENCH_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    L = _lib.lib()
    ctx = lo.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{local}")
    n = cfg["n"]
    radii = cfg["radii"]

    # N > 1: rank 0 builds and broadcasts the structure over NCCL (north star);
    # LO_BENCH_REPLICATE=1 has every rank build the (deterministic, bit-identical) structure from its
    # own copy of the cloud instead -- §8e's alternative, no communication (not measurable on the
    # one-GPU boxes of this round)
    replicate = world > 1 and os.environ.get("LO_BENCH_REPLICATE") == "1"
    builds = rank == 0 or replicate
    xyz_host = generate(cfg) if builds else None
    xyz_dev = C.c_void_p()
    if builds:
        _lib.check(L.lo_device_alloc(ctx.h, 24 * n, C.byref(xyz_dev)))
        _lib.check(L.lo_memcpy_h2d(ctx.h, xyz_dev, xyz_host.ctypes.data, 24 * n))

    def barrier():
        if world > 1:
            dist.barrier()

    def build_structure():
        coded = tree = None
        if builds:
            coded = C.c_void_p()
            _lib.check(L.lo_reorder_device(ctx.h, xyz_dev, n, cfg["curve"], 21, C.byref(coded)))
            tree = C.c_void_p()
            _lib.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))
        if world > 1 and not replicate:
            coded, tree, _, _ = D.broadcast_structure(ctx, coded, tree, src=0)
        return coded, tree

    b0, b1 = D.shard_range(n, rank, world)
    totals = {}

    def step(timing_tag=None):
        coded, tree = build_structure()
        for r in radii:
            csr = C.c_void_p()
            _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, b0, b1, 0, C.byref(csr)))
            info = _lib.CsrInfo()
            _lib.check(L.lo_csr_info_get(csr, C.byref(info)))
            totals[r] = int(info.total)
            if timing_tag is not None:
                timing_tag.append((r, ctx.stage_times()))
            L.lo_csr_destroy(csr)
        return coded, tree

    def free(coded, tree):
        L.lo_octree_destroy(tree)
        L.lo_coded_destroy(coded)

    # warm-up
    for _ in range(args.warmup):
        free(*step())
    ctx.synchronize()

    # timed region: K steps bracketed by barrier + synchronize, CUDA events on our stream
    launches0 = L.lo_launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            free(*step())
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = L.lo_launch_count() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = len(radii) * n / (ms * 1e-3)
    nbrs = sum(totals.values())
    if world > 1:
        _, nbrs = D.global_row_base(nbrs, device=f"cuda:{local}")

    # per-stage device times (CUDA events on the context stream), instrumented steps
    ctx.set_timing(True)
    stage_acc: dict[str, list[float]] = {}
    for _ in range(max(2, min(args.steps, 5))):
        tags = []
        coded, tree = build_structure()
        for name, t in ctx.stage_times():
            stage_acc.setdefault(name, []).append(t)
        for r in radii:
            csr = C.c_void_p()
            _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, b0, b1, 0, C.byref(csr)))
            for name, t in ctx.stage_times():
                stage_acc.setdefault(f"{name}@r={r}", []).append(t)
            L.lo_csr_destroy(csr)
        tinfo = lo._lib.OctreeInfo()
        _lib.check(L.lo_octree_info_get(tree, C.byref(tinfo)))
        free(coded, tree)
    ctx.set_timing(False)
    stages = {k: statistics.mean(v) for k, v in stage_acc.items()}

    # kNN (cfg2) on a resident tree
    knn_out = {}
    if cfg["ks"] and not args.no_knn:
        coded, tree = build_structure()
        for k in cfg["ks"]:
            res = C.c_void_p()
            _lib.check(L.lo_knn_range(ctx.h, tree, coded, k, b0, b1, 0, C.byref(res)))  # warm
            L.lo_knn_destroy(res)
            reps = max(1, min(args.steps, 3))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record(stream)
            for _ in range(reps):
                res = C.c_void_p()
                _lib.check(L.lo_knn_range(ctx.h, tree, coded, k, b0, b1, 0, C.byref(res)))
                L.lo_knn_destroy(res)
            e1.record(stream)
            torch.cuda.synchronize()
            kms = e0.elapsed_time(e1) / reps
            if world > 1:
                t = torch.tensor([kms], device=f"cuda:{local}")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                kms = float(t.item())
            qps = n / (kms * 1e-3)
            byts = n * (24 + 12 * k)
            knn_out[str(k)] = {"ms": kms, "queries_per_s": qps, "neighbours_per_s": qps * k,
                               "hbm_frac": byts / (kms * 1e-3) / (PEAKS["hbm_gbs"] * 1e9 * world)}
        free(coded, tree)

    # e2e through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        pinned = C.c_void_p()
        if builds:
            _lib.check(L.lo_host_alloc_pinned(24 * n, C.byref(pinned)))
            C.memmove(pinned, xyz_host.ctypes.data, 24 * n)
        rows = b1 - b0
        # one pinned (counts, digests) pair per radius and step parity: radius i's results travel
        # on the copy stream while radius i + 1 computes (lo_csr_download_async), and step s's
        # last results land while step s + 1 starts; step s + 2 waits for them (lo_d2h_wait)
        # before reusing their host buffers
        per_step_sync = os.environ.get("LO_BENCH_E2E_SYNC") is not None
        hc = [[C.c_void_p() for _ in radii] for _ in range(2)]
        hf = [[C.c_void_p() for _ in radii] for _ in range(2)]
        for a, b in zip(hc[0] + hc[1], hf[0] + hf[1]):
            _lib.check(L.lo_host_alloc_pinned(4 * max(rows, 1), C.byref(a)))
            _lib.check(L.lo_host_alloc_pinned(8 * max(rows, 1), C.byref(b)))

        # input pipeline: step s+1's cloud uploads (lo_h2d_begin, its own stream) while step s
        # computes; every step still moves its 24 B/pt in and its counts + digests out
        dev_in = [C.c_void_p(), C.c_void_p()]
        if builds:
            for d in dev_in:
                _lib.check(L.lo_device_alloc(ctx.h, 24 * n, C.byref(d)))

        def e2e_run(steps):
            if builds:
                _lib.check(L.lo_h2d_begin(ctx.h, dev_in[0], pinned, 24 * n, 0))
            for s in range(steps):
                cur = s % 2
                coded = tree = None
                if builds:
                    if s + 1 < steps:
                        _lib.check(L.lo_h2d_begin(ctx.h, dev_in[1 - cur], pinned, 24 * n, 1 - cur))
                    _lib.check(L.lo_h2d_wait(ctx.h, cur))
                    coded = C.c_void_p()
                    _lib.check(L.lo_reorder_device(ctx.h, dev_in[cur], n, cfg["curve"], 21, C.byref(coded)))
                    tree = C.c_void_p()
                    _lib.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))
                if world > 1 and not replicate:
                    coded, tree, _, _ = D.broadcast_structure(ctx, coded, tree, src=0)
                if s >= 2:
                    _lib.check(L.lo_d2h_wait(ctx.h, cur))  # step s - 2's results are on the host
                for i, r in enumerate(radii):
                    csr = C.c_void_p()
                    _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, b0, b1, 1, C.byref(csr)))
                    _lib.check(L.lo_csr_download_async(ctx.h, csr, hc[cur][i], hf[cur][i], None, None))
                    L.lo_csr_destroy(csr)
                _lib.check(L.lo_d2h_fence(ctx.h, cur))
                free(coded, tree)
                if per_step_sync:
                    _lib.check(L.lo_context_synchronize(ctx.h))
            _lib.check(L.lo_context_synchronize(ctx.h))  # every step's results on the host

        e2e_run(max(2, args.warmup // 2))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        e2e_run(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = e0.elapsed_time(e1) / args.steps
        if world > 1:
            t = torch.tensor([ems], device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": len(radii) * n / (ems * 1e-3), "unit": "queries/s", "ms_per_step": ems,
               "h2d_bytes_per_step": 24 * n * (world if replicate else 1), "d2h_bytes_per_step": len(radii) * 12 * n,
               "path": "lo_h2d_begin(pinned cloud, next step's upload overlapped) -> lo_reorder_device -> "
                       "lo_octree_build -> lo_radius_range(+FNV) -> lo_csr_download_async(counts, digests; "
                       "overlapped with the next radius and step; host buffers double-buffered behind "
                       "lo_d2h_fence/lo_d2h_wait) -> lo_context_synchronize"}
        if builds:
            L.lo_host_free_pinned(pinned)
            for d in dev_in:
                L.lo_device_free(ctx.h, d)
        for a, b in zip(hc[0] + hc[1], hf[0] + hf[1]):
            L.lo_host_free_pinned(a)
            L.lo_host_free_pinned(b)

    # roofline of the dominant kernel (largest device time in the step)
    mus = {r: totals[r] / max(1, b1 - b0) for r in radii}
    q = b1 - b0

    def algo_bytes(stage):
        name, _, rtag = stage.partition("@r=")
        if name == "radius_fill":
            return q * (24 + 8 + 4 * mus[float(rtag)])
        if name == "radius_count":
            return q * (24 + 4)
        if name == "radius_scan":
            return q * (4 + 8)
        if name == "encode":
            return n * 36
        if name == "gather":
            return n * 52
        if name == "sort":
            return n * (8 + 24 * 8)
        if name == "build":
            return 8 * n + 56 * tinfo.internal + 12 * (tinfo.leaves + 1)
        if name == "bbox":
            return 24 * n
        return 0
    dom = max(stages, key=stages.get)
    dom_bytes = algo_bytes(dom)
    achieved = dom_bytes / (stages[dom] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": PEAKS["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / PEAKS["hbm_gbs"], "traffic": None,
                "peak_source": PEAK_SRC, "algorithmic_bytes_per_launch": dom_bytes,
                "launch_ms": stages[dom],
                "note": "bytes are algorithmic (SURVEY.md §8d: 24 + 4 B/query for the count kernel, "
                        "24 + 8 + 4*mu for the fill); the search kernels are instruction-issue "
                        "bound (issue_active from ncu), the fill is the HBM-moving kernel"}
    traffic = {}
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        try:
            tr = json.load(open(traffic_file))
            if tr.get("config") == args.config:
                traffic = tr.get("stages", {})
        except (OSError, ValueError):
            traffic = {}
    if dom in traffic:
        roofline["traffic"] = traffic[dom]["dram_bytes_per_launch"]
        roofline["traffic_source"] = traffic[dom].get("source")
        if traffic[dom].get("issue_active_pct") is not None:
            roofline["issue_active"] = traffic[dom]["issue_active_pct"] / 100.0
    # every stage against the same HBM roofline (algorithmic bytes / device time)
    per_stage = {}
    for st, st_ms in stages.items():
        b = algo_bytes(st)
        if b and st_ms > 0:
            rec = {"ms": round(st_ms, 4), "achieved_gbs": round(b / (st_ms * 1e-3) / 1e9, 1),
                   "frac": round(b / (st_ms * 1e-3) / 1e9 / PEAKS["hbm_gbs"], 4)}
            name = st.partition("@r=")[0]
            if name in ("bbox", "encode", "sort", "gather", "build"):  # keys/s per stage
                rec["keys_per_s"] = round(n / (st_ms * 1e-3))
            elif name in ("radius_count", "radius_fill"):
                rec["queries_per_s"] = round(q / (st_ms * 1e-3))
            if st in traffic:
                rec["traffic_gbs"] = round(traffic[st]["dram_bytes_per_launch"] / (st_ms * 1e-3) / 1e9, 1)
                if traffic[st].get("issue_active_pct") is not None:
                    rec["issue_active"] = round(traffic[st]["issue_active_pct"] / 100.0, 3)
            per_stage[st] = rec
    roofline["stages"] = per_stage

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            st = cpu_reference_step(cfg, xyz_host, args.cpu_sample)
            cpu = {"value": st["value"], "unit": "queries/s", "cores": st["threads"],
                   "kind": "reference",
                   "sample": f"oracle/_ref (reference sources): full reorder+build "
                             f"({st['t_reorder']:.2f}s + {st['t_build']:.3f}s), radius via "
                             f"neighbours_lin on {st['sample']} contiguous sorted centres per "
                             f"radius, extrapolated to {n}",
                   "knn_queries_per_s": st["knn_qps"]}
        except FileNotFoundError as e:
            cpu = {"value": None, "unit": "queries/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": metric_name(cfg), "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, SURVEY.md §8d; generated on host, identical for the CPU "
                    "reference)",
            "config": config_block(args, cfg),
            "neighbours_per_s": nbrs / (ms * 1e-3),
            "mu": {str(r): mus[r] for r in radii},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "stages_ms": stages,
            "knn": knn_out,
        }
        print(json.dumps(line), flush=True)
    if rank == 0:
        L.lo_device_free(ctx.h, xyz_dev)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg1")
    ap.add_argument("--cpu-sample", type=int, default=200_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-knn", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
