"""cfg4 reordering ablation (BASELINE configs[4]): 50M uniform points in
[0,500]^3, original random order vs Morton vs Hilbert.  Per order: encode / sort / gather /
build times (keys/s), radius r=3 and kNN k=16 search times, the exact kNN locality histogram
(log2 bins + mean / G1 / quartiles) and -- from a separate ncu pass -- the L2 hit rate of the
search kernels.

"Original order" follows the reference (cli.cpp:230-238, locality.hpp:36-40): the structure is
the Hilbert-sorted tree, queries are issued in the file's storage order (centre i = original
point i, i.e. the inverse permutation), and locality distances are measured between mapped
(original) indices.  Our coordinates stay in sorted storage, so the original-order line isolates
the query-order effect; the reference itself has no linear-octree search in original order
(--sfc none supports only the pointer octree, which is out of scope).

    python profiles/cfg4_ablation.py [--n 50000000] [--out profiles/r1/cfg4_ablation.json]
    python profiles/cfg4_ablation.py --searches-only --order hilbert   # the ncu target
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2603_06771_b200 import _lib, linoct as lo  # noqa: E402


KNN_STORAGE_CENTRES = 2_000_000  # kNN in true storage order is bounded to a prefix of the queries


def run_order(L, ctx, xyz, n, order, stats=True):
    """order: "morton" / "hilbert" (Full mode, sorted queries); "original" (queries in storage
    order, searched along the curve by the library and scattered back -- the default mitigation);
    "original_storage" (the same queries searched in storage order: LO_OPT_CENTRE_ORDER = 0)."""
    curve = 0 if order == "morton" else 1
    storage = order == "original_storage"
    _lib.check(L.lo_context_set_option(ctx.h, 1, 0 if storage else 1))
    ctx.set_timing(True)
    coded = C.c_void_p()
    _lib.check(L.lo_reorder(ctx.h, xyz.ctypes.data, n, curve, 21, C.byref(coded)))
    tree = C.c_void_p()
    _lib.check(L.lo_octree_build(ctx.h, coded, 32, C.byref(tree)))
    st = dict(ctx.stage_times())
    ctx.set_timing(False)
    rec = {"curve": "hilbert" if curve else "morton"}
    for k in ("encode", "sort", "gather", "build"):
        if k in st:
            rec[f"{k}_ms"] = st[k]
            rec[f"{k}_keys_per_s"] = n / (st[k] * 1e-3)
    centres = None
    if order.startswith("original"):
        perm = np.empty(n, np.uint32)
        _lib.check(L.lo_coded_download(ctx.h, coded, None, None, perm.ctypes.data))
        inv = np.empty(n, np.uint32)
        inv[perm] = np.arange(n, dtype=np.uint32)
        centres = inv  # query i = original point i
    cp = None if centres is None else centres.ctypes.data
    m = 0 if centres is None else n
    # radius r = 3 (Lin, digests on) and kNN k = 16, each timed on its second run
    for rep in range(2):
        h = C.c_void_p()
        t0 = time.perf_counter()
        _lib.check(L.lo_radius(ctx.h, tree, coded, 1, 0, 3.0, cp, m, 1, C.byref(h)))
        wall = time.perf_counter() - t0
        info = _lib.CsrInfo()
        _lib.check(L.lo_csr_info_get(h, C.byref(info)))
        L.lo_csr_destroy(h)
    rec["radius_r3_ms"] = info.device_ms
    rec["radius_r3_wall_ms"] = wall * 1e3
    rec["radius_mu"] = info.mean_count
    km = m
    if order.startswith("original"):
        km = min(m, KNN_STORAGE_CENTRES)  # the same bounded prefix for both original-order rows
        rec["knn16_centres"] = km
    for rep in range(2):
        kh = C.c_void_p()
        _lib.check(L.lo_knn(ctx.h, tree, coded, 16, cp, km, 1, C.byref(kh)))
        rows, keff, ms = C.c_uint64(), C.c_uint32(), C.c_double()
        _lib.check(L.lo_knn_info_get(kh, C.byref(rows), C.byref(keff), C.byref(ms)))
        L.lo_knn_destroy(kh)
    rec["knn16_ms"] = ms.value
    if stats and not storage:  # (the storage-order row shares the "original" histogram)
        # exact locality histogram over every centre (sorted-order kNN result), mapped through
        # the permutation for the original order
        perm = None
        if order.startswith("original"):
            perm = np.empty(n, np.uint32)
            _lib.check(L.lo_coded_download(ctx.h, coded, None, None, perm.ctypes.data))
        full = C.c_void_p()
        _lib.check(L.lo_knn(ctx.h, tree, coded, 16, None, 0, 0, C.byref(full)))
        nb = C.c_uint64()
        pm = None if perm is None else perm.ctypes.data
        _lib.check(L.lo_locality_histogram(ctx.h, full, coded, None, pm, C.byref(nb), None, None, 0))
        d = np.empty(nb.value, np.uint32)
        c = np.empty(nb.value, np.uint64)
        _lib.check(L.lo_locality_histogram(ctx.h, full, coded, None, pm, C.byref(nb), d.ctypes.data,
                                           c.ctypes.data, nb.value))
        L.lo_knn_destroy(full)
        hist = lo.LocalityHistogram(16, n, n, d, c)
        log2 = np.zeros(33, np.uint64)
        b = np.where(d == 0, 0, np.floor(np.log2(np.maximum(d, 1))).astype(np.int64) + 1)
        np.add.at(log2, b, c)
        q = lo.histogram_quantiles(hist)
        rec["locality"] = {"mean": hist.mean(), "stddev": hist.stddev(), "G1": lo.fisher_pearson_skewness(hist),
                           "Q1": q[0], "Q2": q[1], "Q3": q[2], "distinct_d": int(nb.value),
                           "log2_bins": [int(x) for x in log2]}
    L.lo_octree_destroy(tree)
    L.lo_coded_destroy(coded)
    _lib.check(L.lo_context_set_option(ctx.h, 1, 1))
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=50_000_000)
    ap.add_argument("--out", default=None)
    ap.add_argument("--order", nargs="*", default=["original_storage", "original", "morton", "hilbert"])
    ap.add_argument("--searches-only", action="store_true")
    a = ap.parse_args()
    cfg = dict(bench.CONFIGS["cfg4"])
    cfg["n"] = a.n
    L = _lib.lib()
    ctx = lo.Context(0)
    xyz = bench.generate(cfg)
    out = {"config": "cfg4", "n": a.n, "leaf_bucket": 32, "orders": {}}
    for order in a.order:
        run_order(L, ctx, xyz, a.n, order, stats=False)  # warm-up: pool growth, lazy module loads
        rec = run_order(L, ctx, xyz, a.n, order, stats=not a.searches_only)
        out["orders"][order] = rec
        print(order, json.dumps({k: v for k, v in rec.items() if k != "locality"}), flush=True)
        if "locality" in rec:
            print("  locality", json.dumps({k: v for k, v in rec["locality"].items() if k != "log2_bins"}),
                  flush=True)
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
