"""Asynchronous result downloads (lo_csr_download_async): results destroyed while their copy is
in flight must still arrive intact, and equal the synchronous download."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

lo = pytest.importorskip("paper_2603_06771_b200.linoct")
from paper_2603_06771_b200 import _lib  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    return lo.default_context(0)


def test_async_download_overlaps_and_matches(ctx, oracle):
    pts = oracle.gen_terrain(400000, 3, 200.0)
    coded = lo.reorder_cloud(pts, lo.Curve.Hilbert)
    tree = lo.LinearOctree(coded, 32)
    L = _lib.lib()
    n = coded.n
    radii = [0.5, 1.0, 2.0, 3.0]
    want = [lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, r, lo.BatchOptions())
            for r in radii]
    bufs = []
    for rep in range(2):
        got = []
        for r in radii:
            counts = np.zeros(n, np.uint32)
            fps = np.zeros(n, np.uint64)
            h = C.c_void_p()
            _lib.check(L.lo_radius_range(ctx.h, tree.h, coded.h, 1, 0, r, 0, n, 1, C.byref(h)))
            _lib.check(L.lo_csr_download_async(ctx.h, h, counts.ctypes.data, fps.ctypes.data, None, None))
            L.lo_csr_destroy(h)  # before the copy is known to be done
            got.append((counts, fps))
            bufs.append((counts, fps))
        _lib.check(L.lo_context_synchronize(ctx.h))
        for (counts, fps), w in zip(got, want):
            assert np.array_equal(counts, w.counts) and np.array_equal(fps, w.fingerprints)
