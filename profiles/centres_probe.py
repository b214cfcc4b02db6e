"""kNN / radius with explicit centre lists vs Full mode (device time of the search)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_06771_b200 import _lib, linoct as lo
from oracle.oracle_py import Oracle
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
L = _lib.lib(); ctx = lo.Context(0)
pts = Oracle().gen_uniform(n, 5, 100.0 * (n / 1e6) ** (1 / 3))
coded = lo.reorder_cloud(pts, lo.Curve.Hilbert); tree = lo.LinearOctree(coded, 32)
rng = np.random.default_rng(1)
for name, c in [("full", None), ("arange", np.arange(n, dtype=np.uint32)), ("perm", rng.permutation(n).astype(np.uint32)),
                ("subset", np.sort(rng.choice(n, n // 10, replace=False)).astype(np.uint32))]:
    for rep in range(2):
        kh = C.c_void_p()
        _lib.check(L.lo_knn(ctx.h, tree.h, coded.h, 16, None if c is None else c.ctypes.data, 0 if c is None else len(c), 1, C.byref(kh)))
        rows, keff, ms = C.c_uint64(), C.c_uint32(), C.c_double()
        _lib.check(L.lo_knn_info_get(kh, C.byref(rows), C.byref(keff), C.byref(ms)))
        L.lo_knn_destroy(kh)
        h = C.c_void_p()
        _lib.check(L.lo_radius(ctx.h, tree.h, coded.h, 1, 0, 2.5, None if c is None else c.ctypes.data, 0 if c is None else len(c), 1, C.byref(h)))
        info = _lib.CsrInfo(); _lib.check(L.lo_csr_info_get(h, C.byref(info))); L.lo_csr_destroy(h)
    print(f"{name:7s} knn16 {ms.value:9.2f} ms  radius {info.device_ms:8.2f} ms  mu {info.mean_count:.1f}", flush=True)
