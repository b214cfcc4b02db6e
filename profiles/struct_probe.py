"""Struct (RangedResult) radius batches on a bench config: device time per radius and the
output size against the Lin CSR.

    python profiles/struct_probe.py [--config cfg1] [--reps 3]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2603_06771_b200 import _lib, linoct as lo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    L = _lib.lib()
    ctx = lo.Context(0)
    xyz = bench.generate(cfg)
    n = cfg["n"]
    coded = C.c_void_p()
    _lib.check(L.lo_reorder(ctx.h, xyz.ctypes.data, n, cfg["curve"], 21, C.byref(coded)))
    tree = C.c_void_p()
    _lib.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))
    out = {}
    for r in cfg["radii"]:
        rec = {}
        for method, name in ((1, "lin"), (3, "struct")):
            best = None
            for _ in range(a.reps):
                ctx.set_timing(True)
                csr = C.c_void_p()
                _lib.check(L.lo_radius_range(ctx.h, tree, coded, method, 0, r, 0, n, 1, C.byref(csr)))
                info = _lib.CsrInfo()
                _lib.check(L.lo_csr_info_get(csr, C.byref(info)))
                best = info.device_ms if best is None else min(best, info.device_ms)
                if method == 3:
                    tr, ts = C.c_uint64(), C.c_uint64()
                    _lib.check(L.lo_csr_struct_info(csr, C.byref(tr), C.byref(ts)))
                    rec["ranges"], rec["singles"] = tr.value, ts.value
                    rec["struct_bytes"] = 8 * tr.value + 4 * ts.value + 16 * (n + 1)
                else:
                    rec["members"] = info.total
                    rec["lin_bytes"] = 4 * info.total + 8 * (n + 1)
                L.lo_csr_destroy(csr)
                rec[f"{name}_stages"] = {k: round(v, 3) for k, v in ctx.stage_times()}
                ctx.set_timing(False)
            rec[f"{name}_ms"] = best
        out[str(r)] = rec
        print(r, rec, flush=True)
    print(json.dumps({"config": a.config, "struct": out}))


if __name__ == "__main__":
    main()
