"""Wall-clock breakdown of a radius batch with an explicit (shuffled) centre list."""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_06771_b200 import _lib, linoct as lo
from oracle.oracle_py import Oracle
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
L = _lib.lib(); ctx = lo.Context(0)
pts = Oracle().gen_uniform(n, 5, 500.0)
coded = lo.reorder_cloud(pts, lo.Curve.Hilbert); tree = lo.LinearOctree(coded, 32)
perm = np.random.default_rng(1).permutation(n).astype(np.uint32)
for rep in range(3):
    ctx.set_timing(True)
    t0 = time.perf_counter()
    h = C.c_void_p()
    _lib.check(L.lo_radius(ctx.h, tree.h, coded.h, 1, 0, 3.0, perm.ctypes.data, n, 1, C.byref(h)))
    t1 = time.perf_counter()
    L.lo_csr_destroy(h)
    st = ctx.stage_times()
    ctx.set_timing(False)
    print(f"rep {rep} wall {1e3*(t1-t0):.1f} ms", {k: round(v, 2) for k, v in st}, flush=True)
