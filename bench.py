#!/usr/bin/env python
"""bench.py -- the hot path on B200: SFC reorder -> linear-octree build -> fixed-radius search.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg3]

One step = one pass of the hot path over the config's synthetic cloud: encode + radix sort
+ gather (reorder_cloud), octree build (LinearOctree), then a full radius batch (count ->
u64 scan -> fill -> FNV-1a row digests, every point a query: run_radius_batch with
BatchOptions' defaults, search.hpp:110-117) at every radius of the config.  The default
workload is cfg3 (100M mixed points, Hilbert, leaf 64, r = 1, k = 16), the largest config that
fits one B200 and the one the metric's 1/2/4/8-GPU figures are quoted on; cfg1 (10M terrain,
r = 0.5/1/2/3, kNN k = 8/16/32/64 = cfg2) runs after it under "extra".

  value     radius queries/s over the whole step, cloud already resident in HBM.
  e2e       the same step through the C ABI with HOST buffers: pinned cloud uploaded every
            step, each batch's counts + FNV digests downloaded (BatchResult's default content).
  e2e_csr   the same with the whole CSR (u64 offsets + u32 indices) downloaded every step.
  knn       kNN batches on the resident structure (device) and knn.e2e (host cloud in, sorted
            (index, dist_sq) rows + digests out).

Multi-GPU (torchrun, one rank per GPU): rank 0 reorders + builds, the structure is broadcast
over NCCL (timed as its own stage), each rank searches its contiguous SFC slice of the queries
(strong scaling: the total work is the config's fixed batch).  Time = max over ranks of
CUDA-event time.

`--impl reference` times the reference's own CPU implementation (oracle/_ref: the unmodified
reference sources compiled by oracle/Makefile) on this host with all its threads, same config /
metric / unit.  Inputs come from the oracle's generators (no repo library is loaded).  The
full-size reorder_cloud + LinearOctree run once; each step then runs run_batch_loop's radius
query (neighbours_lin + FNV digests, dynamic OpenMP) over a bounded sample of centres: many
contiguous SFC slices spread evenly over the whole cloud, rotated every step.  A step's time
is the sample's measured search time plus its per-query share of the measured reorder + build.
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
DEFAULT_CONFIG = "cfg3"


def generate(cfg):
    """Product-arm input: the library's host generators (bit-identical to the oracle's)."""
    from paper_2603_06771_b200 import linoct as lo
    if cfg["kind"] == "uniform":
        return lo.generate_uniform(cfg["n"], cfg["seed"], cfg["extent"])
    if cfg["kind"] == "terrain":
        return lo.generate_terrain(cfg["n"], cfg["seed"], cfg["extent"])
    return lo.generate_mixed(cfg["n"], cfg["seed"])


def generate_oracle(cfg):
    """Reference-arm input: the oracle's C generators (rng.hpp draw order; no repo library)."""
    from oracle.oracle_py import Oracle
    o = Oracle()
    if cfg["kind"] == "uniform":
        return o.gen_uniform(cfg["n"], cfg["seed"], cfg["extent"])
    if cfg["kind"] == "terrain":
        return o.gen_terrain(cfg["n"], cfg["seed"], cfg["extent"])
    return o.gen_mixed(cfg["n"], cfg["seed"])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (every LO_BENCH_CLOCK_MS,
    default 100 ms; 0 disables it)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        interval = int(os.environ.get("LO_BENCH_CLOCK_MS", "100"))
        if interval <= 0:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(interval)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)  # let the first samples land before the (possibly short) timed region
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.1)
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


def host_info():
    """CPU model / sockets / cores of this host (lscpu), for the CPU baseline's record."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=20).stdout
    except (OSError, subprocess.SubprocessError):
        return info
    keys = {"Model name": "model", "Socket(s)": "sockets", "Core(s) per socket": "cores_per_socket",
            "Thread(s) per core": "threads_per_core", "NUMA node(s)": "numa_nodes", "CPU(s)": "cpus"}
    for ln in out.splitlines():
        k, _, v = ln.partition(":")
        k = k.strip()
        if k in keys and keys[k] not in info:
            v = v.strip()
            info[keys[k]] = int(v) if v.isdigit() else v
    return info


# ---- reference arm / CPU baseline -----------------------------------------------------------
def spread_centres(n: int, total: int, slices: int, step: int) -> np.ndarray:
    """`slices` contiguous runs of sorted (SFC-ordered) centres, evenly spread over [0, n),
    together ~`total` centres; the run positions rotate with `step` so successive steps sample
    different parts of each stride.  Contiguous runs keep the batch loop's cache behaviour
    (Full mode walks the sorted cloud in order); the spread covers every region of the cloud
    (cfg3's clusters, terrain and noise) in proportion."""
    total = min(total, n)
    slices = max(1, min(slices, total))
    per = max(1, total // slices)
    stride = n // slices
    room = max(1, stride - per + 1)
    off = (step * 7919 * per) % room
    starts = np.arange(slices, dtype=np.int64) * stride + off
    c = (starts[:, None] + np.arange(per, dtype=np.int64)[None, :]).ravel()
    return c[c < n].astype(np.uint32)


class RefRun:
    """The unmodified reference library (oracle/_ref) on this host's cores: reorder_cloud +
    LinearOctree at full size once (reference's own steady_clock, ref_driver.cpp), then
    bounded search samples."""

    def __init__(self, cfg, xyz, threads=None):
        from oracle.oracle_py import Ref
        self.cfg = cfg
        self.ref = Ref()
        self.threads = threads or self.ref.max_threads()
        self.p = self.ref.pipeline(xyz, cfg["curve"], cfg["n_max"], threads=self.threads)
        # LinearOctree timed after one warm-up build: the first build pays page faults
        self.t_reorder = float(self.p.timings[0])
        self.t_build = float(self.p.rebuild(cfg["n_max"], self.threads))

    @property
    def t_setup(self):
        return self.t_reorder + self.t_build

    def radius_step(self, step: int, sample: int, slices: int):
        n = self.cfg["n"]
        c = spread_centres(n, sample, slices, step)
        walls, mus = [], []
        for r in self.cfg["radii"]:
            wall, counts, _ = self.p.radius_centres(r, c, threads=self.threads)
            walls.append(wall)
            mus.append(float(counts.mean()))
        s = len(c)
        t_search = sum(walls)
        t_step = t_search + self.t_setup * s / n  # the sample's share of the full-size build
        return dict(value=len(self.cfg["radii"]) * s / t_step, t_step=t_step, t_search=t_search,
                    walls=walls, mu=mus, sample=s)

    def knn_qps(self, sample: int, slices: int):
        out = {}
        c = spread_centres(self.cfg["n"], sample, slices, 0)
        for k in self.cfg["ks"]:
            wall, _ = self.p.knn_centres(k, c, threads=self.threads)
            out[str(k)] = len(c) / wall
        return out

    def close(self):
        del self.p


def cfg0_figures(threads: int):
    """cfg0 (1M uniform, Morton, leaf 32, r = 2.5) through the reference's stock
    run_radius_batch (Full mode, fingerprints on) at `threads` and at 1 thread."""
    from oracle.oracle_py import Ref
    cfg = CONFIGS["cfg0"]
    ref = Ref()
    xyz = ref.gen_uniform(cfg["n"], cfg["seed"], cfg["extent"])  # the reference's own gen_uniform
    out = {}
    for th in sorted({threads, 1}, reverse=True):
        p = ref.pipeline(xyz, cfg["curve"], cfg["n_max"], threads=th)
        t_build = float(p.rebuild(cfg["n_max"], th))  # after one warm-up build
        wall = p.radius(cfg["radii"][0], threads=th)["wall"]  # run_radius_batch's own wall_seconds
        t = float(p.timings[0]) + t_build + wall
        out[f"threads_{th}"] = {"queries_per_s": cfg["n"] / t, "step_s": t, "reorder_s": float(p.timings[0]),
                                "build_s": t_build, "radius_s": wall, "mode": "Full (every point), stock run_radius_batch"}
        del p
    return out


def reference_baseline(cfg, xyz, steps, warmup, sample, slices, threads=None, with_cfg0=True):
    t0 = time.perf_counter()
    rr = RefRun(cfg, xyz, threads)
    st = []
    for i in range(warmup + steps):
        s = rr.radius_step(i, sample, slices)
        if i >= warmup:
            st.append(s)
    knn = rr.knn_qps(max(1, sample // 2), slices) if cfg["ks"] else {}
    res = dict(
        value=statistics.median(s["value"] for s in st),
        ms_per_step=statistics.median(s["t_step"] for s in st) * 1e3,
        threads=rr.threads, sample=st[0]["sample"], slices=slices,
        t_reorder=rr.t_reorder, t_build=rr.t_build,
        t_search=statistics.median(s["t_search"] for s in st),
        mu=st[0]["mu"], knn_qps=knn, step_values=[s["value"] for s in st])
    res["full_step_s_estimate"] = rr.t_setup + res["t_search"] * cfg["n"] / res["sample"]
    rr.close()
    if with_cfg0:
        res["cfg0"] = cfg0_figures(rr.threads)
    res["wall_s"] = time.perf_counter() - t0
    return res


def baseline_desc(cfg, b, steps):
    return (f"oracle/_ref (unmodified reference sources): full-size reorder_cloud + LinearOctree once "
            f"({b['t_reorder']:.2f} s + {b['t_build']:.3f} s), then per step run_batch_loop's radius query "
            f"(neighbours_lin + FNV digests, dynamic OpenMP) over {b['sample']} sorted centres = {b['slices']} "
            f"contiguous SFC slices spread over the whole cloud (rotated per step) at each radius; step time = "
            f"sample search time + the sample's {b['sample']}/{cfg['n']} share of reorder + build; median of "
            f"{steps} steps; the reference radix sort is single-threaded at every thread count "
            f"(reorder.cpp:38-62)")


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    t0 = time.perf_counter()
    xyz = generate_oracle(cfg)
    t_gen = time.perf_counter() - t0
    b = reference_baseline(cfg, xyz, args.steps, args.warmup, args.cpu_sample, args.cpu_slices)
    wall = time.perf_counter() - t0
    line = {
        "impl": "reference", "metric": metric_name(cfg), "value": b["value"], "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": b["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY.md §8d; oracle generators, rng.hpp draw order)",
        "config": config_block(args, cfg),
        "cpu_baseline": {"value": b["value"], "unit": "queries/s", "cores": b["threads"], "kind": "reference",
                         "sample": baseline_desc(cfg, b, args.steps), "host": host_info()},
        "e2e": {"value": b["value"], "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "stages_s": {"reorder": b["t_reorder"], "build": b["t_build"], "search_per_step": b["t_search"]},
        "full_step_s_estimate": b["full_step_s_estimate"],
        "step_values": b["step_values"],
        "mu": b["mu"],
        "knn_qps": b["knn_qps"],
        "cfg0": b["cfg0"],
        "consistency": {"wall_s": wall, "generate_s": t_gen,
                        "timed_s": (args.steps + args.warmup) * b["ms_per_step"] * 1e-3,
                        "fits_in_wall": (args.steps + args.warmup) * b["ms_per_step"] * 1e-3 <= wall},
    }
    print(json.dumps(line), flush=True)
    return 0


def metric_name(cfg):
    return ("radius queries/s per hot-path step (reorder + octree build + full radius batch with FNV "
            "digests at each radius; " + cfg["desc"] + ")")


def config_block(args, cfg, workload=None):
    return {"workload": workload or args.config, "points": cfg["n"], "cloud": cfg["kind"],
            "curve": "hilbert" if cfg["curve"] else "morton", "leaf_bucket": cfg["n_max"],
            "radii": cfg["radii"], "knn_k": cfg["ks"], "queries_per_step": len(cfg["radii"]) * cfg["n"],
            "parallelism": (f"query-shard x{args.gpus} (" + ("structure built on every rank"
                                                            if os.environ.get("LO_BENCH_REPLICATE") == "1"
                                                            else "structure broadcast from rank 0") + ")")
            if args.gpus > 1 else "1 GPU",
            "l2": "inputs larger than L2 (cloud 24 B/pt + multi-GB CSR per step)"}


# ---- our arm --------------------------------------------------------------------------------
class Arm:
    """The product path through the C ABI (liblinoct_b200.so) for one config on this rank."""

    def __init__(self, args, cfg, ctx, L, world, rank, local, replicate):
        import torch
        self.torch = torch
        self.args, self.cfg, self.ctx, self.L = args, cfg, ctx, L
        self.world, self.rank, self.local, self.replicate = world, rank, local, replicate
        self.builds = rank == 0 or replicate
        self.n = cfg["n"]
        self.stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{local}")
        self.xyz_host = generate(cfg) if self.builds else None
        self.xyz_dev = C.c_void_p()
        from paper_2603_06771_b200 import _lib
        self._lib = _lib
        if self.builds:
            _lib.check(L.lo_device_alloc(ctx.h, 24 * self.n, C.byref(self.xyz_dev)))
            _lib.check(L.lo_memcpy_h2d(ctx.h, self.xyz_dev, self.xyz_host.ctypes.data, 24 * self.n))
        from paper_2603_06771_b200 import distributed as D
        self.D = D
        # N > 1 over NCCL: the library's own communicator (lo_comm, C ABI) broadcasts the structure
        # and shards the searches; the gloo test hook (several ranks on one device, where NCCL
        # refuses duplicate GPUs) keeps the torch.distributed plumbing
        self.comm = None
        if world > 1 and not replicate and os.environ.get("LO_BENCH_DIST_BACKEND", "nccl") == "nccl":
            self.comm = D.Comm(ctx, rank, world)
        self.b0, self.b1 = self.comm.shard(self.n) if self.comm else D.shard_range(self.n, rank, world)
        self.totals = {}
        self.global_totals = {}
        self.bcast_last_ms = 0.0

    def check(self, rc):
        self._lib.check(rc)

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(self, v):
        if self.world == 1:
            return v
        import torch.distributed as dist
        t = self.torch.tensor([v], device=f"cuda:{self.local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def build_structure(self, xyz_dev=None):
        L, ctx, cfg = self.L, self.ctx, self.cfg
        coded = tree = None
        if self.builds:
            coded = C.c_void_p()
            self.check(L.lo_reorder_device(ctx.h, xyz_dev or self.xyz_dev, self.n, cfg["curve"], 21, C.byref(coded)))
            tree = C.c_void_p()
            self.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))
        if self.comm is not None:
            coded, tree = self.comm.broadcast_structure(coded, tree, root=0)
        elif self.world > 1 and not self.replicate:
            torch = self.torch
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
            coded, tree, _, _ = self.D.broadcast_structure(self.ctx, coded, tree, src=0)
            e1.record(self.stream)
            e1.synchronize()
            self.bcast_last_ms = e0.elapsed_time(e1)
        return coded, tree

    def free(self, coded, tree):
        self.L.lo_octree_destroy(tree)
        self.L.lo_coded_destroy(coded)

    def radius(self, coded, tree, r, fingerprint=1):
        if self.comm is not None:
            csr, _, _, total = self.comm.radius(tree, coded, r, fingerprint=fingerprint)
            self.global_totals[r] = total
            return csr
        csr = C.c_void_p()
        self.check(self.L.lo_radius_range(self.ctx.h, tree, coded, 1, 0, r, self.b0, self.b1, fingerprint,
                                          C.byref(csr)))
        return csr

    def step(self):
        coded, tree = self.build_structure()
        for r in self.cfg["radii"]:
            csr = self.radius(coded, tree, r)
            info = self._lib.CsrInfo()
            self.check(self.L.lo_csr_info_get(csr, C.byref(info)))
            self.totals[r] = int(info.total)
            self.L.lo_csr_destroy(csr)
        self.free(coded, tree)

    def timed(self, fn, steps):
        """K calls of fn bracketed by barrier + synchronize, CUDA events on the library stream;
        returns max-over-ranks ms per call."""
        torch = self.torch
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        self.barrier()
        torch.cuda.synchronize()
        e0.record(self.stream)
        per = [] if os.environ.get("LO_BENCH_STEP_TIMES") else None  # diagnostics: per-call device times
        for _ in range(steps):
            fn()
            if per is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(self.stream)
                per.append(ev)
        self.check(self.L.lo_context_join(self.ctx.h))  # side-stream work (aux digests, downloads) inside e1
        e1.record(self.stream)
        torch.cuda.synchronize()
        self.barrier()
        if per:
            prev, out = e0, []
            for ev in per:
                out.append(round(prev.elapsed_time(ev), 2))
                prev = ev
            sys.stderr.write(f"[bench] per-call device ms: {out}\n")
        return self.max_over_ranks(e0.elapsed_time(e1) / steps)

    def main_region(self, steps, warmup):
        for _ in range(warmup):
            self.step()
        self.ctx.synchronize()
        if os.environ.get("LO_DEBUG_ALLOC"):
            sys.stderr.write("== timed region\n")
        l0 = self.L.lo_launch_count()
        with ClockSampler(self.local) as clocks:
            ms = self.timed(self.step, steps)
        if os.environ.get("LO_DEBUG_ALLOC"):
            sys.stderr.write("== end of timed region\n")
        return ms, self.L.lo_launch_count() - l0, clocks.summary()

    def stages(self, reps):
        """Per-stage device times (CUDA events on the context stream) over instrumented steps."""
        ctx, L = self.ctx, self.L
        ctx.set_timing(True)
        acc: dict[str, list[float]] = {}
        tinfo = self._lib.OctreeInfo()
        for _ in range(reps):
            t0 = time.perf_counter()
            coded, tree = self.build_structure()
            if self.world > 1 and not self.replicate and self.comm is None:
                acc.setdefault("broadcast", []).append(self.bcast_last_ms)
            for name, t in ctx.stage_times():
                acc.setdefault(name, []).append(t)
            for r in self.cfg["radii"]:
                csr = self.radius(coded, tree, r)
                for name, t in ctx.stage_times():
                    acc.setdefault(f"{name}@r={r}", []).append(t)
                L.lo_csr_destroy(csr)
            self.check(L.lo_octree_info_get(tree, C.byref(tinfo)))
            self.free(coded, tree)
        ctx.set_timing(False)
        self.tinfo = tinfo
        return {k: statistics.mean(v) for k, v in acc.items()}

    def knn_device(self, reps):
        out = {}
        if not self.cfg["ks"]:
            return out
        coded, tree = self.build_structure()
        for k in self.cfg["ks"]:
            def one():
                if self.comm is not None:
                    res, _ = self.comm.knn(tree, coded, k)
                else:
                    res = C.c_void_p()
                    self.check(self.L.lo_knn_range(self.ctx.h, tree, coded, k, self.b0, self.b1, 1, C.byref(res)))
                self.L.lo_knn_destroy(res)
            one()  # warm
            kms = self.timed(one, reps)
            qps = self.n / (kms * 1e-3)
            out[str(k)] = {"ms": kms, "queries_per_s": qps, "neighbours_per_s": qps * k,
                           "hbm_frac": self.n * (24 + 12 * k) / (kms * 1e-3) / (PEAKS["hbm_gbs"] * 1e9 * self.world),
                           "digests": True}
        self.free(coded, tree)
        return out

    # -- end to end: host buffers, copies inside the timed region --------------------------------
    def _pinned(self, nbytes):
        p = C.c_void_p()
        self.check(self.L.lo_host_alloc_pinned(max(16, nbytes), C.byref(p)))
        return p

    def e2e(self, steps, warm, mode):
        """mode "digests": per radius counts + FNV digests (double-buffered host results);
        "csr": counts + digests + u64 offsets + u32 indices (single host buffer set, the caller
        consumes step s-1's rows while step s computes); "knn": kNN rows (index, dist_sq) + digests.
        Step s+1's cloud uploads (lo_h2d_begin) while step s computes."""
        L, ctx, n, cfg = self.L, self.ctx, self.n, self.cfg
        rows = self.b1 - self.b0
        pinned = None
        dev_in = [C.c_void_p(), C.c_void_p()]
        if self.builds:
            pinned = self._pinned(24 * n)
            C.memmove(pinned, self.xyz_host.ctypes.data, 24 * n)
            for d in dev_in:
                self.check(L.lo_device_alloc(ctx.h, 24 * n, C.byref(d)))
        nbuf = 2 if mode == "digests" else 1
        keys = cfg["radii"] if mode != "knn" else cfg["ks"][:1]
        host = []
        d2h = 0
        for b in range(nbuf):
            per = []
            for key in keys:
                bufs = {"counts": self._pinned(4 * rows), "fps": self._pinned(8 * rows)}
                if b == 0:
                    d2h += 12 * rows
                if mode == "csr":
                    tot = self.totals[key]
                    bufs["offsets"] = self._pinned(8 * (rows + 1))
                    bufs["indices"] = self._pinned(4 * tot)
                    if b == 0:
                        d2h += 8 * (rows + 1) + 4 * tot
                if mode == "knn":
                    del bufs["counts"]
                    bufs["idx"] = self._pinned(4 * rows * key)
                    bufs["dist"] = self._pinned(8 * rows * key)
                    if b == 0:
                        d2h += 12 * rows * key - 4 * rows
                per.append(bufs)
            host.append(per)

        def run(nsteps):
            if self.builds:
                self.check(L.lo_h2d_begin(ctx.h, dev_in[0], pinned, 24 * n, 0))
            for s in range(nsteps):
                cur = s % 2
                slot = s % nbuf
                coded = tree = None
                if self.builds:
                    if s + 1 < nsteps:
                        self.check(L.lo_h2d_begin(ctx.h, dev_in[1 - cur], pinned, 24 * n, 1 - cur))
                    self.check(L.lo_h2d_wait(ctx.h, cur))
                coded, tree = self.build_structure(dev_in[cur] if self.builds else None)
                results = []
                for key in keys:
                    if mode == "knn" and self.comm is not None:
                        res, _ = self.comm.knn(tree, coded, key)
                    elif mode == "knn":
                        res = C.c_void_p()
                        self.check(L.lo_knn_range(ctx.h, tree, coded, key, self.b0, self.b1, 1, C.byref(res)))
                    else:
                        res = self.radius(coded, tree, key)
                    results.append(res)
                # the caller has consumed the results that last used these host buffers
                if s >= nbuf:
                    self.check(L.lo_d2h_wait(ctx.h, slot))
                for key, res, bufs in zip(keys, results, host[slot]):
                    if mode == "knn":
                        self.check(L.lo_knn_download_async(ctx.h, res, bufs["idx"], bufs["dist"], bufs["fps"]))
                        L.lo_knn_destroy(res)
                    else:
                        self.check(L.lo_csr_download_async(ctx.h, res, bufs["counts"], bufs["fps"],
                                                           bufs.get("offsets"), bufs.get("indices")))
                        L.lo_csr_destroy(res)
                self.check(L.lo_d2h_fence(ctx.h, slot))
                self.free(coded, tree)
            self.check(L.lo_context_synchronize(ctx.h))  # every step's results are on the host

        run(warm)
        dbg = os.environ.get("LO_DEBUG_ALLOC")
        if dbg:
            sys.stderr.write(f"== e2e {mode} timed region\n")
        ems = self.timed(lambda: run(steps), 1) / steps
        if dbg:
            sys.stderr.write(f"== end of e2e {mode} timed region: {ems:.2f} ms per step\n")
        if self.builds:
            L.lo_host_free_pinned(pinned)
            for d in dev_in:
                L.lo_device_free(ctx.h, d)
        for per in host:
            for bufs in per:
                for p in bufs.values():
                    L.lo_host_free_pinned(p)
        h2d = 24 * n * (self.world if self.replicate else 1)
        q = len(keys) * n
        return {"value": q / (ems * 1e-3), "unit": "queries/s", "ms_per_step": ems, "steps": steps,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h * self.world}


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2603_06771_b200 import _lib, linoct as lo

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
    # N > 1: rank 0 builds and broadcasts the structure (north star);
    # LO_BENCH_REPLICATE=1 has every rank build the (deterministic, bit-identical) structure from
    # its own copy of the cloud instead (§8e's alternative, no communication)
    replicate = world > 1 and os.environ.get("LO_BENCH_REPLICATE") == "1"
    arm = Arm(args, cfg, ctx, L, world, rank, local, replicate)
    arm.bcast_last_ms = 0.0
    n = cfg["n"]
    radii = cfg["radii"]

    ms, launches, clocks = arm.main_region(args.steps, args.warmup)
    value = len(radii) * n / (ms * 1e-3)
    nbrs = sum(arm.totals.values())
    if arm.comm is not None:
        nbrs = sum(arm.global_totals.values())
    elif world > 1:
        _, nbrs = arm.D.global_row_base(nbrs, device=f"cuda:{local}")
    stages = arm.stages(max(2, min(args.steps, 4)))
    tinfo = arm.tinfo
    knn_out = arm.knn_device(max(1, min(args.steps, 3))) if not args.no_knn else {}

    e2e = e2e_csr = None
    if not args.no_e2e:
        # warm-ups reach the steady state of the result buffers: a step's results are parked behind their
        # download while the next step allocates, so the cache settles after two or three steps
        e2e = arm.e2e(args.steps, max(3, args.warmup), "digests")
        e2e["path"] = ("lo_h2d_begin(pinned cloud, next step's upload overlapped) -> lo_reorder_device -> "
                       "lo_octree_build -> lo_radius_range(+FNV) -> lo_csr_download_async(counts, digests; "
                       "overlapped with the next radius and step; host buffers double-buffered behind "
                       "lo_d2h_fence/lo_d2h_wait) -> lo_context_synchronize")
        k_e2e = max(2, min(args.steps, 5))
        e2e_csr = arm.e2e(k_e2e, 3, "csr")
        e2e_csr["path"] = ("as e2e, plus every row of the CSR (u64 offsets + u32 indices) downloaded each step "
                           "(BatchResult::results, collect_results = true, search.hpp:115,125)")
        if cfg["ks"] and not args.no_knn:
            ke = arm.e2e(k_e2e, 3, "knn")
            ke["unit"] = f"queries/s (k={cfg['ks'][0]})"
            ke["path"] = ("lo_h2d_begin -> lo_reorder_device -> lo_octree_build -> lo_knn_range(+FNV) -> "
                          "lo_knn_download_async(index + dist_sq rows, digests) -> lo_context_synchronize")
            knn_out["e2e"] = ke

    # roofline of the dominant work: the radius search unit (count -> scan -> fill) at the largest
    # radius, against SURVEY.md §8d's algorithmic bytes per query (24 + 8 + 4 mu)
    q = arm.b1 - arm.b0
    mus = {r: arm.totals[r] / max(1, q) for r in radii}

    def algo_bytes(stage):
        name, _, rtag = stage.partition("@r=")
        if name == "radius_fill":
            return q * (24 + 8 + 4 * mus[float(rtag)])
        if name == "radius_count":
            return q * (24 + 4)
        if name == "radius_scan":
            return q * (4 + 8)
        if name == "radius_digest":
            return q * (8 + 8) + 4 * q * mus[float(rtag)]
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

    r_top = max(radii)
    unit_stages = [f"radius_count@r={r_top}", f"radius_scan@r={r_top}", f"radius_fill@r={r_top}"]
    unit_ms = sum(stages.get(s, 0.0) for s in unit_stages)
    unit_bytes = q * (24 + 8 + 4 * mus[r_top])
    achieved = unit_bytes / (unit_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": f"radius search unit @ r={r_top} (radius_pt_kernel count + u64 scan "
                                          f"+ replay fill)",
                "achieved": achieved, "peak": PEAKS["hbm_gbs"], "unit": "GB/s", "frac": achieved / PEAKS["hbm_gbs"],
                "traffic": None, "peak_source": PEAK_SRC, "algorithmic_bytes_per_launch": unit_bytes,
                "launch_ms": unit_ms,
                "note": "bytes per query = 24 + 8 + 4*mu (SURVEY.md §8d: coordinates, u64 offset, u32 indices) "
                        "over the event-timed count + scan + fill; the count kernel alone is instruction-issue "
                        "bound (issue_active from ncu), the fill is the HBM-moving kernel; roofline.stages "
                        "has every stage on the same basis"}
    traffic = {}
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        try:
            tr = json.load(open(traffic_file))
            if tr.get("config") == args.config:
                traffic = tr.get("stages", {})
        except (OSError, ValueError):
            traffic = {}
    tb = [traffic[s]["dram_bytes_per_launch"] for s in unit_stages if s in traffic]
    if len(tb) == len(unit_stages):
        roofline["traffic"] = sum(tb)
        roofline["traffic_source"] = traffic[unit_stages[0]].get("source")
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
                rec["traffic_bytes"] = traffic[st]["dram_bytes_per_launch"]
                rec["traffic_gbs"] = round(traffic[st]["dram_bytes_per_launch"] / (st_ms * 1e-3) / 1e9, 1)
                if traffic[st].get("issue_active_pct") is not None:
                    rec["issue_active"] = round(traffic[st]["issue_active_pct"] / 100.0, 3)
            per_stage[st] = rec
    roofline["stages"] = per_stage

    # the rest of the configs at N = 1: cfg1 (+ cfg2's kNN) on the same device, device-timed
    extra = {}
    if world == 1 and not args.no_extra:
        for name in args.extra:
            if name == args.config:
                continue
            ecfg = CONFIGS[name]
            if arm is not None:
                if arm.builds:
                    L.lo_device_free(ctx.h, arm.xyz_dev)
                arm = None
            sub = Arm(args, ecfg, ctx, L, world, rank, local, replicate)
            sub.bcast_last_ms = 0.0
            ems, _, eclk = sub.main_region(args.steps, args.warmup)
            est = sub.stages(2)
            ek = sub.knn_device(max(1, min(args.steps, 3))) if not args.no_knn else {}
            en = ecfg["n"]
            extra[name] = {"config": config_block(args, ecfg, workload=name), "value": len(ecfg["radii"]) * en / (ems * 1e-3),
                           "unit": "queries/s", "ms_per_step": ems, "clocks": eclk,
                           "mu": {str(r): sub.totals[r] / en for r in ecfg["radii"]},
                           "neighbours_per_s": sum(sub.totals.values()) / (ems * 1e-3),
                           "stages_ms": est, "knn": ek}
            L.lo_device_free(ctx.h, sub.xyz_dev)
            sub = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            xyz = generate_oracle(cfg)
            b = reference_baseline(cfg, xyz, 2, 0, args.cpu_sample, args.cpu_slices)
            del xyz
            cpu = {"value": b["value"], "unit": "queries/s", "cores": b["threads"], "kind": "reference",
                   "sample": baseline_desc(cfg, b, 2), "host": host_info(),
                   "ms_per_step": b["ms_per_step"], "full_step_s_estimate": b["full_step_s_estimate"],
                   "stages_s": {"reorder": b["t_reorder"], "build": b["t_build"], "search_per_step": b["t_search"]},
                   "knn_queries_per_s": b["knn_qps"], "cfg0": b["cfg0"]}
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
            "e2e_csr": e2e_csr,
            "gpu_launches": launches,
            "clocks": clocks,
            "stages_ms": stages,
            "knn": knn_out,
            "extra": extra,
        }
        print(json.dumps(line), flush=True)
    if arm is not None and arm.builds:
        L.lo_device_free(ctx.h, arm.xyz_dev)
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
    ap.add_argument("--config", choices=sorted(CONFIGS), default=DEFAULT_CONFIG)
    ap.add_argument("--extra", nargs="*", default=["cfg1"], help="further configs timed on the device at N = 1")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=2_000_000, help="centres per CPU sample step")
    ap.add_argument("--cpu-slices", type=int, default=200, help="contiguous SFC slices per CPU sample")
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
