"""Work-weighted vs equal query shards on one B200: for G = 2, 4, 8 ranks, each rank's
slice of the config's Full radius batch (count + scan + fill + digests) is timed alone with the library's
stage events, for equal slices (lo_shard_range) and for lo_radius_work_bounds (one radius batch over the
first query tile of every 2048 centres).  The max over ranks is the radius stage's critical path at G GPUs
(no interconnect in it: the structure is broadcast before, and the rows need no exchange).

    python profiles/shard_balance.py [--config cfg3] [--reps 2]
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_06771_b200 import _lib, distributed as D, linoct as lo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--stride", type=int, default=2048)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
L = _lib.lib()
ctx = lo.Context(0)
xyz = bench.generate(cfg)
n = cfg["n"]
r = cfg["radii"][-1]
coded, tree = C.c_void_p(), C.c_void_p()
_lib.check(L.lo_reorder(ctx.h, xyz.ctypes.data, n, cfg["curve"], 21, C.byref(coded)))
_lib.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))


def slice_ms(b, e):
    ts = []
    for rep in range(a.reps + 1):
        ctx.set_timing(True)
        csr = C.c_void_p()
        _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, b, e, 1, C.byref(csr)))
        st = ctx.stage_times()
        ctx.set_timing(False)
        info = _lib.CsrInfo()
        _lib.check(L.lo_csr_info_get(csr, C.byref(info)))
        L.lo_csr_destroy(csr)
        if rep:
            ts.append(sum(t for _, t in st))
    return statistics.mean(ts), int(info.total)


out = {"config": a.config, "radius": r, "stride": a.stride, "ranks": {}}
full_ms, full_nb = slice_ms(0, n)
out["single_gpu_ms"] = round(full_ms, 3)
for g in (2, 4, 8):
    rec = {}
    ctx.set_timing(True)
    bw = D.radius_work_bounds(ctx, tree, coded, r, g, stride=a.stride)
    st = ctx.stage_times()
    ctx.set_timing(False)
    rec["work_bounds_ms"] = round(sum(t for _, t in st), 3)
    for name, bounds in (("equal", [D.shard_range(n, k, g) for k in range(g)]),
                         ("weighted", [(int(bw[k]), int(bw[k + 1])) for k in range(g)])):
        per = [slice_ms(b, e) for b, e in bounds]
        ms = [p[0] for p in per]
        nb = [p[1] for p in per]
        rec[name] = {"slices": bounds, "ms": [round(x, 3) for x in ms], "neighbours": nb,
                     "max_ms": round(max(ms), 3), "max_over_mean_ms": round(max(ms) / (sum(ms) / g), 3),
                     "max_over_mean_neighbours": round(max(nb) / (sum(nb) / g), 3)}
    rec["critical_path_gain"] = round(rec["equal"]["max_ms"] / (rec["weighted"]["max_ms"] + rec["work_bounds_ms"]), 3)
    out["ranks"][g] = rec
    sys.stderr.write(f"G={g}: equal max {rec['equal']['max_ms']} ms, weighted max {rec['weighted']['max_ms']} + "
                     f"{rec['work_bounds_ms']} ms bounds\n")
print(json.dumps(out))
