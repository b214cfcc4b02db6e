"""Octree-build probe: one reordered cloud, lo_octree_build timed per stage over reps (LO_LIB_PATH selects a
side build), then one radius batch on the last tree whose counts + digests fingerprint the tight node boxes the
walk prunes with.

    python profiles/build_probe.py [--config cfg3] [--reps 5]
"""
import argparse
import ctypes as C
import hashlib
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_06771_b200 import _lib, linoct as lo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
L = _lib.lib()
ctx = lo.Context(0)
xyz = bench.generate(cfg)
n = cfg["n"]
coded = C.c_void_p()
_lib.check(L.lo_reorder(ctx.h, xyz.ctypes.data, n, cfg["curve"], 21, C.byref(coded)))
acc = []
tree = C.c_void_p()
for rep in range(a.reps + 1):
    if tree.value:
        L.lo_octree_destroy(tree)
    tree = C.c_void_p()
    ctx.set_timing(True)
    _lib.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))
    st = dict(ctx.stage_times())
    ctx.set_timing(False)
    if rep:
        acc.append(st.get("build", sum(st.values())))
r = cfg["radii"][-1]
csr = C.c_void_p()
_lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, 0, n, 1, C.byref(csr)))
cnt = np.empty(n, np.uint32)
fps = np.empty(n, np.uint64)
_lib.check(L.lo_csr_download(ctx.h, csr, cnt.ctypes.data, fps.ctypes.data, None, None))
print(json.dumps({"config": a.config, "lib": os.environ.get("LO_LIB_PATH", "in-tree"), "build_ms": round(statistics.mean(acc), 4),
                  "sha": hashlib.sha1(cnt.tobytes() + fps.tobytes()).hexdigest()[:16]}))
