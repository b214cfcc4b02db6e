"""Per-phase device times inside the bench's e2e loop (pipelined upload, async downloads, double-
buffered host results): where the e2e step spends the time the device-only step does not.

    python profiles/e2e_phases.py [--config cfg1] [--steps 6] [--no-fp]
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
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--no-fp", action="store_true")
    ap.add_argument("--no-dl", action="store_true", help="no result downloads")
    ap.add_argument("--no-h2d", action="store_true", help="reorder the resident cloud (no uploads)")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    L = _lib.lib()
    ctx = lo.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream, device="cuda:0")
    xyz = bench.generate(cfg)
    n, radii = cfg["n"], cfg["radii"]
    pinned = C.c_void_p()
    _lib.check(L.lo_host_alloc_pinned(24 * n, C.byref(pinned)))
    C.memmove(pinned, xyz.ctypes.data, 24 * n)
    hc = [[C.c_void_p() for _ in radii] for _ in range(2)]
    hf = [[C.c_void_p() for _ in radii] for _ in range(2)]
    for x, y in zip(hc[0] + hc[1], hf[0] + hf[1]):
        _lib.check(L.lo_host_alloc_pinned(4 * n, C.byref(x)))
        _lib.check(L.lo_host_alloc_pinned(8 * n, C.byref(y)))
    dev_in = [C.c_void_p(), C.c_void_p()]
    for d in dev_in:
        _lib.check(L.lo_device_alloc(ctx.h, 24 * n, C.byref(d)))
    fp = 0 if a.no_fp else 1
    marks = []
    host_calls = {}

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    _lib.check(L.lo_h2d_begin(ctx.h, dev_in[0], pinned, 24 * n, 0))
    t0 = time.perf_counter()
    for s in range(a.steps):
        cur = s % 2
        row = [("start", ev(), time.perf_counter())]
        if s + 1 < a.steps and not a.no_h2d:
            _lib.check(L.lo_h2d_begin(ctx.h, dev_in[1 - cur], pinned, 24 * n, 1 - cur))
        if not a.no_h2d:
            _lib.check(L.lo_h2d_wait(ctx.h, cur))
        row.append(("h2d_wait", ev(), time.perf_counter()))
        coded = C.c_void_p()
        _lib.check(L.lo_reorder_device(ctx.h, dev_in[0 if a.no_h2d else cur], n, cfg["curve"], 21, C.byref(coded)))
        tree = C.c_void_p()
        _lib.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))
        row.append(("reorder+build", ev(), time.perf_counter()))
        if s >= 2:
            _lib.check(L.lo_d2h_wait(ctx.h, cur))
        for i, r in enumerate(radii):
            csr = C.c_void_p()
            _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, 0, n, fp, C.byref(csr)))
            h0 = time.perf_counter()
            if not a.no_dl:
                _lib.check(L.lo_csr_download_async(ctx.h, csr, hc[cur][i], hf[cur][i] if fp else None, None,
                                                   None))
            h1 = time.perf_counter()
            L.lo_csr_destroy(csr)
            h2 = time.perf_counter()
            host_calls.setdefault("download_async", []).append((h1 - h0) * 1e3)
            host_calls.setdefault("destroy", []).append((h2 - h1) * 1e3)
            row.append((f"r={r}", ev(), time.perf_counter()))
        _lib.check(L.lo_d2h_fence(ctx.h, cur))
        L.lo_octree_destroy(tree)
        L.lo_coded_destroy(coded)
        marks.append(row)
    _lib.check(L.lo_context_synchronize(ctx.h))
    wall = (time.perf_counter() - t0) * 1e3 / a.steps
    torch.cuda.synchronize()
    for s, row in enumerate(marks):
        parts = []
        for (name, e, h), (_, e0, h0) in zip(row[1:], row[:-1]):
            parts.append(f"{name} {e0.elapsed_time(e):.2f}/{(h - h0) * 1e3:.2f}")
        nxt = marks[s + 1][0][1] if s + 1 < len(marks) else None
        tot = row[0][1].elapsed_time(nxt) if nxt is not None else float("nan")
        print(f"step {s}: device/host ms  " + "  ".join(parts) + f"  | step {tot:.2f}")
    print("host ms per call:", {k: round(sum(v) / len(v), 3) for k, v in host_calls.items()})
    print(f"wall per step {wall:.2f} ms (fingerprints {'off' if a.no_fp else 'on'}, downloads "
          f"{'off' if a.no_dl else 'on'}, uploads {'off' if a.no_h2d else 'on'})")


if __name__ == "__main__":
    main()
