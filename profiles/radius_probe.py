"""Radius-stage probe: one structure, full radius batches at the config's radii, per-stage device
times (count / scan / fill / digest) averaged over reps.  Tuning knobs are read from the
environment by the library (LO_COARSE, LO_COMPACT_MUL, LO_REPLAY_ROW_MAJOR_MIN, ...).

    python profiles/radius_probe.py [--config cfg3] [--reps 3] [--radius 1.0 ...]
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
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--radius", type=float, nargs="*", default=None)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
radii = a.radius or cfg["radii"]
L = _lib.lib()
ctx = lo.Context(0)
xyz = bench.generate(cfg)
n = cfg["n"]
coded, tree = C.c_void_p(), C.c_void_p()
_lib.check(L.lo_reorder(ctx.h, xyz.ctypes.data, n, cfg["curve"], 21, C.byref(coded)))
_lib.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))
acc = {}
sha = {}
import hashlib
import numpy as np
for rep in range(a.reps + 1):
    ctx.set_timing(True)
    for r in radii:
        csr = C.c_void_p()
        _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, 0, n, 1, C.byref(csr)))
        if rep == 0:  # result fingerprint (counts + row digests) to compare variants
            cnt = np.empty(n, np.uint32)
            fps = np.empty(n, np.uint64)
            _lib.check(L.lo_csr_download(ctx.h, csr, cnt.ctypes.data, fps.ctypes.data, None, None))
            sha[str(r)] = hashlib.sha1(cnt.tobytes() + fps.tobytes()).hexdigest()[:16]
        if rep:
            for name, t in ctx.stage_times():
                acc.setdefault(f"{name}@{r}", []).append(t)
        L.lo_csr_destroy(csr)
    ctx.set_timing(False)
knobs = {k: v for k, v in os.environ.items() if k.startswith("LO_")}
print(json.dumps({"config": a.config, "lib": os.environ.get("LO_LIB_PATH", "in-tree"), "sha": sha, "knobs": knobs, "ms": {k: round(statistics.mean(v), 3) for k, v in acc.items()}}))
