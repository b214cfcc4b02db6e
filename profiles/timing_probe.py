import ctypes as C, time, sys, os
sys.path.insert(0, os.getcwd())
import bench
from paper_2603_06771_b200 import _lib, linoct as lo
L=_lib.lib(); ctx=lo.Context(0)
cfg=bench.CONFIGS['cfg1']; xyz=bench.generate(cfg); n=cfg['n']
d=C.c_void_p(); _lib.check(L.lo_device_alloc(ctx.h, 24*n, C.byref(d))); _lib.check(L.lo_memcpy_h2d(ctx.h, d, xyz.ctypes.data, 24*n))
for it in range(4):
    t0=time.perf_counter()
    coded=C.c_void_p(); _lib.check(L.lo_reorder_device(ctx.h, d, n, 1, 21, C.byref(coded)))
    tree=C.c_void_p(); _lib.check(L.lo_octree_build(ctx.h, coded, 32, C.byref(tree)))
    t1=time.perf_counter(); ts=[]
    for r in cfg['radii']:
        a=time.perf_counter(); csr=C.c_void_p(); _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, 0, n, 0, C.byref(csr))); L.lo_csr_destroy(csr); ts.append(time.perf_counter()-a)
    L.lo_octree_destroy(tree); L.lo_coded_destroy(coded)
    print(f"it{it} build {1e3*(t1-t0):.1f} ms radius", [f"{1e3*x:.1f}" for x in ts], flush=True)
