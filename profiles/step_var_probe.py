"""Step-time variance probe for the bench's main region (cfg3 by default).

Runs the exact bench step (bench.Arm.step pieces: reorder, build, radius with digests, destroys) in
blocks of K back-to-back steps, with CUDA events between the API calls on the library stream, the
library's stage events on, and host perf_counter times around every call. For each step it reports
the device time of each API call, the sum of the stages inside it, and the host time of the call,
so a slow step can be attributed to (a) a slower kernel (stage grows), (b) device idle between
kernels while the host is inside the library (call time > stage sum), or (c) the host outside the
library (gap between calls).

    python profiles/step_var_probe.py [--config cfg3] [--steps 20] [--blocks 3]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_06771_b200 import _lib, linoct as lo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--blocks", type=int, default=3)
ap.add_argument("--timing", type=int, default=1, help="library stage events on")
a = ap.parse_args()

import torch  # noqa: E402

cfg = bench.CONFIGS[a.config]
L = _lib.lib()
ctx = lo.Context(0)
args = argparse.Namespace(steps=a.steps, warmup=5)
arm = bench.Arm(args, cfg, ctx, L, 1, 0, 0, False)
stream = arm.stream


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


def step(marks, host):
    t0 = time.perf_counter()
    coded = C.c_void_p()
    _lib.check(L.lo_reorder_device(ctx.h, arm.xyz_dev, arm.n, cfg["curve"], 21, C.byref(coded)))
    t1 = time.perf_counter()
    marks.append(("reorder", ev()))
    tree = C.c_void_p()
    _lib.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))
    t2 = time.perf_counter()
    marks.append(("build", ev()))
    hs = [("reorder", t1 - t0), ("build", t2 - t1)]
    for r in cfg["radii"]:
        t3 = time.perf_counter()
        csr = arm.radius(coded, tree, r)
        t4 = time.perf_counter()
        marks.append((f"radius@{r}", ev()))
        info = _lib.CsrInfo()
        _lib.check(L.lo_csr_info_get(csr, C.byref(info)))
        L.lo_csr_destroy(csr)
        t5 = time.perf_counter()
        marks.append((f"csr_destroy@{r}", ev()))
        hs += [(f"radius@{r}", t4 - t3), (f"csr_destroy@{r}", t5 - t4)]
    t6 = time.perf_counter()
    arm.free(coded, tree)
    t7 = time.perf_counter()
    marks.append(("free", ev()))
    hs.append(("free", t7 - t6))
    host.append({k: round(v * 1e3, 2) for k, v in hs})


for _ in range(5):
    step([], [])
ctx.synchronize()
out = {"config": a.config, "timing": a.timing, "blocks": []}
for b in range(a.blocks):
    if a.timing:
        ctx.set_timing(True)
    torch.cuda.synchronize()
    e0 = ev()
    per_marks, host = [], []
    for _ in range(a.steps):
        m = []
        step(m, host)
        per_marks.append(m)
    torch.cuda.synchronize()
    st = ctx.stage_times() if a.timing else []
    ctx.set_timing(False)
    nst = len(st) // a.steps if st else 0
    rows = []
    prev = e0
    for i, m in enumerate(per_marks):
        row = {"call_ms": {}, "host_ms": host[i]}
        s0 = prev
        for name, e in m:
            row["call_ms"][name] = round(prev.elapsed_time(e), 2)
            prev = e
        row["step_ms"] = round(s0.elapsed_time(prev), 2)
        if nst:
            chunk = st[i * nst:(i + 1) * nst]
            row["stages"] = {k: round(t, 2) for k, t in chunk}
            row["stage_sum"] = round(sum(t for _, t in chunk), 2)
        rows.append(row)
    out["blocks"].append({"mean_step_ms": round(e0.elapsed_time(prev) / a.steps, 2), "steps": rows})
    sys.stderr.write(f"block {b}: mean {out['blocks'][-1]['mean_step_ms']} ms; steps "
                     f"{[r['step_ms'] for r in rows]}\n")
print(json.dumps(out))
