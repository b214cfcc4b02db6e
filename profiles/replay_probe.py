"""Fill (replay) stage time per radius for a config, e.g. to place the buffer-major / row-major
switch:  LO_REPLAY_ROW_MAJOR_MIN=0 python profiles/replay_probe.py --config cfg4"""
import argparse, ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_06771_b200 import _lib, linoct as lo
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="cfg4"); ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
cfg = dict(bench.CONFIGS[a.config]); cfg["n"] = a.n or cfg["n"]
L = _lib.lib(); ctx = lo.Context(0); xyz = bench.generate(cfg); n = cfg["n"]
coded = C.c_void_p(); _lib.check(L.lo_reorder(ctx.h, xyz.ctypes.data, n, cfg["curve"], 21, C.byref(coded)))
tree = C.c_void_p(); _lib.check(L.lo_octree_build(ctx.h, coded, cfg["n_max"], C.byref(tree)))
for r in cfg["radii"]:
    for rep in range(3):
        ctx.set_timing(True)
        h = C.c_void_p(); _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, 0, n, 0, C.byref(h)))
        L.lo_csr_destroy(h); st = dict(ctx.stage_times()); ctx.set_timing(False)
    print(a.config, "r", r, {k: round(v, 3) for k, v in st.items()}, flush=True)
