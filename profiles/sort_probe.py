"""Reorder-stage probe: lo_reorder_device on a config's cloud, per-stage device times (bbox / encode /
sort / gather) averaged over reps; LO_LIB_PATH selects a side build (tuning variants).

    python profiles/sort_probe.py [--config cfg3] [--reps 5]
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
dev = C.c_void_p()
_lib.check(L.lo_device_alloc(ctx.h, 24 * n, C.byref(dev)))
_lib.check(L.lo_memcpy_h2d(ctx.h, dev, xyz.ctypes.data, 24 * n))
acc = {}
perm0 = None
for rep in range(a.reps + 1):
    ctx.set_timing(True)
    coded = C.c_void_p()
    _lib.check(L.lo_reorder_device(ctx.h, dev, n, cfg["curve"], 21, C.byref(coded)))
    st = ctx.stage_times()
    ctx.set_timing(False)
    if rep == 0:
        import numpy as np
        perm0 = np.empty(n, np.uint32)
        _lib.check(L.lo_coded_download(ctx.h, coded, None, None, perm0.ctypes.data))
    else:
        for name, t in st:
            acc.setdefault(name, []).append(t)
    L.lo_coded_destroy(coded)
import hashlib
print(json.dumps({"lib": os.environ.get("LO_LIB_PATH", "in-tree"), "config": a.config,
                  "perm_sha": hashlib.sha1(perm0.tobytes()).hexdigest()[:16],
                  "ms": {k: round(statistics.mean(v), 4) for k, v in acc.items()}}))
