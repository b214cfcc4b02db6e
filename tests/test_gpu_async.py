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


def test_pipelined_steps_with_d2h_fences(ctx, oracle):
    """Three steps whose results trail into the next step (digests on the aux stream, copies on the
    copy stream, result buffers parked in the context cache), host buffers double-buffered behind
    lo_d2h_fence / lo_d2h_wait: every step's counts and digests equal the synchronous ones."""
    pts = oracle.gen_terrain(300000, 5, 200.0)
    coded = lo.reorder_cloud(pts, lo.Curve.Hilbert)
    tree = lo.LinearOctree(coded, 32)
    L = _lib.lib()
    n = coded.n
    radii = [1.0, 3.0]
    want = [lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, r, lo.BatchOptions())
            for r in radii]
    host = [[(np.zeros(n, np.uint32), np.zeros(n, np.uint64)) for _ in radii] for _ in range(2)]
    seen = 0
    for s in range(4):
        cur = s % 2
        if s >= 2:
            _lib.check(L.lo_d2h_wait(ctx.h, cur))
            for (counts, fps), w in zip(host[cur], want):
                assert np.array_equal(counts, w.counts) and np.array_equal(fps, w.fingerprints)
                counts[:] = 0
                fps[:] = 0
            seen += 1
        for (counts, fps), r in zip(host[cur], radii):
            h = C.c_void_p()
            _lib.check(L.lo_radius_range(ctx.h, tree.h, coded.h, 1, 0, r, 0, n, 1, C.byref(h)))
            _lib.check(L.lo_csr_download_async(ctx.h, h, counts.ctypes.data, fps.ctypes.data, None, None))
            L.lo_csr_destroy(h)
        _lib.check(L.lo_d2h_fence(ctx.h, cur))
    _lib.check(L.lo_context_synchronize(ctx.h))
    for buf in host:
        for (counts, fps), w in zip(buf, want):
            assert np.array_equal(counts, w.counts) and np.array_equal(fps, w.fingerprints)
    assert seen == 2
    with pytest.raises(Exception):
        _lib.check(L.lo_d2h_fence(ctx.h, 4))


def test_concurrent_host_threads_share_a_context(ctx, oracle):
    """Calls on one context are serialized by its lock: two host threads issuing radius
    and kNN batches on the same context and structure get the sequential results."""
    import threading
    pts = oracle.gen_terrain(200000, 7, 150.0)
    coded = lo.reorder_cloud(pts, lo.Curve.Hilbert)
    tree = lo.LinearOctree(coded, 32)
    want_r = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, 2.0, lo.BatchOptions())
    want_k = lo.run_knn_batch(tree, coded, 16, lo.BatchOptions())
    errors = []

    def work(kind):
        try:
            for _ in range(3):
                if kind == "radius":
                    got = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, 2.0,
                                              lo.BatchOptions())
                    assert np.array_equal(got.counts, want_r.counts)
                    assert np.array_equal(got.fingerprints, want_r.fingerprints)
                else:
                    got = lo.run_knn_batch(tree, coded, 16, lo.BatchOptions())
                    assert np.array_equal(got.fingerprints, want_k.fingerprints)
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(k,)) for k in ("radius", "knn", "radius")]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
