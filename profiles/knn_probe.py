"""kNN timing probe: one structure, lo_knn_range over every point for each k, under the kernel
variants selected by environment knobs (read per call); device ms from the result's own events.

    python profiles/knn_probe.py [--config cfg1] [--k 8 16 32 64] [--reps 3] [--variants select heaps]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_06771_b200 import _lib, linoct as lo  # noqa: E402

VARIANTS = {"select": {"LO_KNN_SELECT": "1"}, "heaps": {"LO_KNN_SELECT": "0"},
            "win2": {"LO_KNN_SELECT": "1", "LO_KNN_WIN": "2"}, "win8": {"LO_KNN_SELECT": "1", "LO_KNN_WIN": "8"},
            "cap4": {"LO_KNN_SELECT": "1", "LO_KNN_CAP": "4"}, "cap16": {"LO_KNN_SELECT": "1", "LO_KNN_CAP": "16"}}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg1")
ap.add_argument("--k", type=int, nargs="*", default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--variants", nargs="*", default=["select", "heaps"])
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
ks = a.k or cfg["ks"]
L = _lib.lib()
ctx = lo.Context(0)
xyz = bench.generate(cfg)
coded, tree = C.c_void_p(), C.c_void_p()
_lib.check(L.lo_reorder(ctx.h, xyz.ctypes.data, cfg["n"], cfg["curve"], 21, C.byref(coded)))
_lib.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))
out = {"config": a.config, "lib": os.environ.get("LO_LIB_PATH", "in-tree"), "n": cfg["n"], "ms": {}, "fps_equal": {}}
ref_fps = {}
for v in a.variants:
    for key in ("LO_KNN_SELECT", "LO_KNN_WIN", "LO_KNN_CAP"):
        os.environ.pop(key, None)
    os.environ.update(VARIANTS[v])
    for k in ks:
        times = []
        for _ in range(a.reps):
            res = C.c_void_p()
            _lib.check(L.lo_knn_range(ctx.h, tree, coded, k, 0, cfg["n"], 1, C.byref(res)))
            rows, keff, ms = C.c_uint64(), C.c_uint32(), C.c_double()
            _lib.check(L.lo_knn_info_get(res, C.byref(rows), C.byref(keff), C.byref(ms)))
            times.append(ms.value)
            import numpy as np
            fps = np.empty(cfg["n"], dtype=np.uint64)
            _lib.check(L.lo_knn_download(ctx.h, res, None, None, fps.ctypes.data))
            L.lo_knn_destroy(res)
        h = int(np.bitwise_xor.reduce(fps))
        if k not in ref_fps:
            ref_fps[k] = h
        out["fps_equal"][f"{v}@{k}"] = h == ref_fps[k]
        out.setdefault("fps_xor", {})[f"{v}@{k}"] = f"{h:016x}"
        out["ms"][f"{v}@{k}"] = [round(t, 2) for t in times]
        sys.stderr.write(f"{v} k={k}: {[round(t, 2) for t in times]} ms\n")
print(json.dumps(out))
