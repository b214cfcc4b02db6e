"""Context / handle robustness on the device:

- lo_locality_histogram with an index map that is not a permutation (any u32 is a legal map value,
  locality.cpp:47-49): dense bins over the map's value span, or sort + run-length encoding when
  the span is huge -- checked against a numpy histogram of the reference's own kNN lists;
- destroying a context while handles created on it are alive is a LO_LOGIC_ERROR, not a
  use-after-free;
- two contexts on one device sharing read-only handles, used from two host threads: lazily built
  device data (Struct octant boxes) is published complete, results equal the single-context ones.
"""
import ctypes as C
import threading

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


def brute_hist(idx, centres, imap):
    d = np.abs(imap[centres][:, None].astype(np.int64) - imap[idx].astype(np.int64)).ravel()
    u, c = np.unique(d, return_counts=True)
    return u.astype(np.uint32), c.astype(np.uint64)


@pytest.mark.parametrize("kind", ["permutation", "offset", "huge_span"])
def test_locality_non_permutation_map(ctx, ref, oracle, kind):
    pts = oracle.gen_uniform(30_000, 3, 40.0)
    p = ref.pipeline(pts, 1, 32)
    coded = lo.reorder_cloud(pts, lo.Curve.Hilbert)
    tree = lo.LinearOctree(coded, 32)
    n = coded.n
    rng = np.random.default_rng(11)
    if kind == "permutation":
        imap = rng.permutation(n).astype(np.uint32)
    elif kind == "offset":  # values >= n (the dense array must cover the span, not n)
        imap = (rng.permutation(n) * 3 + 1_000_000).astype(np.uint32)
    else:  # span ~2^32: sort + run-length path
        imap = rng.integers(0, 2 ** 32 - 1, n, dtype=np.uint64).astype(np.uint32)
        imap[0], imap[1] = 0, 2 ** 32 - 1
    k = 8
    want_idx = p.knn(k, collect=True)["idx"]
    wd, wc = brute_hist(want_idx, np.arange(n), imap)
    h = lo.locality_histogram(tree, coded, k, index_map=imap)
    assert np.array_equal(h.d, wd) and np.array_equal(h.count, wc)
    # a subset of centres through the same paths
    sub = lo.sample_indices(n, 3000, 5)
    h2 = lo.locality_histogram_approx(tree, coded, k, 3000, 5, index_map=imap)
    sd, sc = brute_hist(want_idx[sub], sub, imap)
    assert np.array_equal(h2.d, sd) and np.array_equal(h2.count, sc)


def test_context_destroy_with_live_handles(ctx, oracle):
    L = _lib.lib()
    c2 = lo.Context(0)
    pts = oracle.gen_uniform(5000, 1, 10.0)
    coded = lo.reorder_cloud(pts, lo.Curve.Morton, ctx=c2)
    tree = lo.LinearOctree(coded, 16)
    rc = L.lo_context_destroy(c2.h)
    assert rc == _lib.LOGIC_ERROR
    assert b"still alive" in L.lo_last_error()
    # the context still works
    res = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, 1.0, lo.BatchOptions())
    assert res.counts.sum() > 0
    del res, tree, coded
    import gc
    gc.collect()
    assert L.lo_context_destroy(c2.h) == _lib.OK
    c2.h = None


def _radius_digests(L, ctx_h, tree, coded, method, r):
    csr = C.c_void_p()
    _lib.check(L.lo_radius(ctx_h, tree.h, coded.h, method, 0, r, None, 0, 1, C.byref(csr)))
    info = _lib.CsrInfo()
    _lib.check(L.lo_csr_info_get(csr, C.byref(info)))
    counts = np.empty(info.rows, np.uint32)
    fps = np.empty(info.rows, np.uint64)
    _lib.check(L.lo_csr_download(ctx_h, csr, counts.ctypes.data_as(C.c_void_p), fps.ctypes.data_as(C.c_void_p),
                                 None, None))
    L.lo_csr_destroy(csr)
    return counts, fps


def test_two_contexts_share_handles_across_threads(ctx, ref, oracle):
    L = _lib.lib()
    pts = oracle.gen_mixed(200_000, 21)
    p = ref.pipeline(pts, 1, 64)
    ca, cb = lo.Context(0), lo.Context(0)
    coded = lo.reorder_cloud(pts, lo.Curve.Hilbert, ctx=ca)
    tree = lo.LinearOctree(coded, 64)
    want_lin = p.radius(2.0, method=1)
    want_struct = p.radius(2.0, method=3)
    out = {}
    errors = []

    def worker(name, c, method):
        try:
            for rep in range(3):
                out[(name, rep)] = _radius_digests(L, c.h, tree, coded, method, 2.0)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    # the Struct boxes are built lazily by whichever context asks first; both threads ask at once
    th = [threading.Thread(target=worker, args=("a", ca, 3)), threading.Thread(target=worker, args=("b", cb, 3)),
          threading.Thread(target=worker, args=("c", cb, 1))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for (name, rep), (counts, fps) in out.items():
        want = want_lin if name == "c" else want_struct
        assert np.array_equal(counts, want["counts"]), (name, rep)
        assert np.array_equal(fps, want["fps"]), (name, rep)
    del tree, coded
    import gc
    gc.collect()
    cb.close()
    ca.close()
