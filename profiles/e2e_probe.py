"""Timing probe for the end-to-end (host buffers) step: synchronous vs asynchronous result
downloads, wall clock per step and per phase.

    python profiles/e2e_probe.py [--config cfg1] [--steps 4]
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2603_06771_b200 import _lib, linoct as lo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--steps", type=int, default=4)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    L = _lib.lib()
    ctx = lo.Context(0)
    xyz = bench.generate(cfg)
    n = cfg["n"]
    radii = cfg["radii"]
    pinned = C.c_void_p()
    _lib.check(L.lo_host_alloc_pinned(24 * n, C.byref(pinned)))
    C.memmove(pinned, xyz.ctypes.data, 24 * n)
    hc = [C.c_void_p() for _ in radii]
    hf = [C.c_void_p() for _ in radii]
    for x, y in zip(hc, hf):
        _lib.check(L.lo_host_alloc_pinned(4 * n, C.byref(x)))
        _lib.check(L.lo_host_alloc_pinned(8 * n, C.byref(y)))
    for mode in ("sync", "async", "nofp", "sync", "async"):
        for it in range(a.steps):
            t = [time.perf_counter()]
            coded = C.c_void_p()
            _lib.check(L.lo_reorder(ctx.h, pinned, n, cfg["curve"], 21, C.byref(coded)))
            t.append(time.perf_counter())
            tree = C.c_void_p()
            _lib.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))
            t.append(time.perf_counter())
            for i, r in enumerate(radii):
                csr = C.c_void_p()
                fp = 0 if mode == "nofp" else 1
                _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, 0, n, fp, C.byref(csr)))
                t.append(time.perf_counter())
                if mode == "async":
                    _lib.check(L.lo_csr_download_async(ctx.h, csr, hc[i], hf[i], None, None))
                else:
                    _lib.check(L.lo_csr_download(ctx.h, csr, hc[i], hf[i] if fp else None, None, None))
                L.lo_csr_destroy(csr)
                t.append(time.perf_counter())
            L.lo_octree_destroy(tree)
            L.lo_coded_destroy(coded)
            _lib.check(L.lo_context_synchronize(ctx.h))
            t.append(time.perf_counter())
            d = [1e3 * (t[i + 1] - t[i]) for i in range(len(t) - 1)]
            print(f"{mode:5s} total {1e3 * (t[-1] - t[0]):7.2f} ms  reorder {d[0]:.2f} build {d[1]:.2f} "
                  f"radius/download {' '.join(f'{x:.2f}' for x in d[2:-1])} sync {d[-1]:.2f}", flush=True)


if __name__ == "__main__":
    main()
