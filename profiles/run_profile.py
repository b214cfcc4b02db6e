"""Small driver for ncu captures: one cfg1-sized pipeline and one radius / kNN batch.

    python profiles/run_profile.py [--config cfg1] [--radius 3.0] [--k 16] [--reps 2]
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2603_06771_b200 import _lib, linoct as lo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--radius", type=float, nargs="*", default=[3.0])
    ap.add_argument("--k", type=int, nargs="*", default=[])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--fingerprint", action="store_true", help="also compute the FNV row digests")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    L = _lib.lib()
    ctx = lo.Context(0)
    xyz = bench.generate(cfg)
    for _ in range(a.reps):
        coded = C.c_void_p()
        _lib.check(L.lo_reorder(ctx.h, xyz.ctypes.data, cfg["n"], cfg["curve"], 21, C.byref(coded)))
        tree = C.c_void_p()
        _lib.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))
        for r in a.radius:
            csr = C.c_void_p()
            _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, 0, cfg["n"], int(a.fingerprint),
                                         C.byref(csr)))
            L.lo_csr_destroy(csr)
        for k in a.k:
            res = C.c_void_p()
            _lib.check(L.lo_knn_range(ctx.h, tree, coded, k, 0, cfg["n"], 0, C.byref(res)))
            L.lo_knn_destroy(res)
        L.lo_octree_destroy(tree)
        L.lo_coded_destroy(coded)
    ctx.synchronize()
    print("profile run ok")


if __name__ == "__main__":
    main()
