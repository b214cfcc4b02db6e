"""GPU parity of the paths the fast kernels fall back to, each forced deterministically and
compared with the reference library itself (oracle/_ref, search.cpp:316-388):

- the exact FP64 kernels (radius_kernel, radius_struct_kernel, knn_kernel), taken when the FP32
  filter disables itself (radius d >= 0.01 r: r below ~2.4e-5 x the cube side, the
  paper's own sg27 r = 0.05 regime) or under LO_FORCE_FP64=1;
- the record-overflow fill walk (tiles with more count-pass records than LO_REC_CAP);
- the two-walk radius path without records (LO_RADIUS_NO_FUSE=1).

Counts and FNV-1a digests (search.cpp:263-271) are compared for every centre (Full mode)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

lo = pytest.importorskip("paper_2603_06771_b200.linoct")


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    return lo.default_context(0)


def pipeline(points, curve, n_max):
    coded = lo.reorder_cloud(points, lo.Curve(curve))
    return coded, lo.LinearOctree(coded, n_max)


def far_patch_cloud(n=120_000, seed=7):
    """A dense 1 m patch plus two far corner points: cube side ~3000 m (cfg3's extent), so r = 0.05
    leaves the FP32 filter disabled (d = 2^-22 * 3000 = 7.2e-4 > 0.01 r) while mu stays ~10-20."""
    rng = np.random.default_rng(seed)
    pts = rng.uniform(0.0, 1.0, (n, 3)) + np.array([1500.0, 1500.0, 20.0])
    pts[0] = (0.0, 0.0, 0.0)
    pts[1] = (3000.0, 3000.0, 60.0)
    return pts


def check_radius(tree, coded, p, r, shape=0, method=1):
    want = p.radius(r, method=method, shape=shape)
    got = lo.run_radius_batch(tree, coded, lo.RadiusMethod(method), lo.KernelShape(shape), r, lo.BatchOptions())
    assert np.array_equal(got.counts, want["counts"]), (r, shape, method)
    assert np.array_equal(got.fingerprints, want["fps"]), (r, shape, method)
    return got


def check_knn(tree, coded, p, k):
    want = p.knn(k)
    got = lo.run_knn_batch(tree, coded, k, lo.BatchOptions())
    assert np.array_equal(got.fingerprints, want["fps"]), k


def test_filter_disables_itself_at_small_radius(ctx, ref):
    """r = 0.05 on a 3 km cube: the FP32 filter is off by its own error bound, every test is FP64."""
    pts = far_patch_cloud()
    p = ref.pipeline(pts, 1, 64)
    coded, tree = pipeline(pts, 1, 64)
    side = coded.disc_box[3] - coded.disc_box[0]
    u = 2.0 ** -23
    for r in (0.05, 0.03):
        assert 2 * u * side + 2 * u * r >= 0.01 * r  # make_float_test's disable condition
        got = check_radius(tree, coded, p, r)
        assert got.mean_count > 3
        for shape in (1, 2, 3):
            check_radius(tree, coded, p, r, shape=shape)
        check_radius(tree, coded, p, r, method=3)  # Struct digests: ranges, separator, singles
        check_radius(tree, coded, p, r, shape=2, method=3)


@pytest.mark.parametrize("curve", [0, 1])
def test_forced_fp64_kernels(ctx, ref, oracle, monkeypatch, curve):
    """LO_FORCE_FP64=1: radius_kernel, radius_struct_kernel and knn_kernel on a normal cloud."""
    pts = oracle.gen_terrain(60_000, 41 + curve, 300.0)
    p = ref.pipeline(pts, curve, 32)
    coded, tree = pipeline(pts, curve, 32)
    monkeypatch.setenv("LO_FORCE_FP64", "1")
    for r in (0.7, 2.0):
        for shape in range(4):
            check_radius(tree, coded, p, r, shape=shape)
        check_radius(tree, coded, p, r, method=3)
    for k in (1, 8, 16, 33, 64, 100):
        check_knn(tree, coded, p, k)
    monkeypatch.delenv("LO_FORCE_FP64")
    check_knn(tree, coded, p, 16)  # and the filtered kernel agrees with both


@pytest.mark.parametrize("cap", [1, 3])
def test_record_overflow_fill_walk(ctx, ref, oracle, monkeypatch, cap):
    """LO_REC_CAP: tiles with more processed buffers than the cap are not recorded and are filled
    by the second walk over a tile list (radius_pt_kernel<SHAPE, true>), Lin and Struct."""
    pts = oracle.gen_terrain(150_000, 5, 120.0)
    p = ref.pipeline(pts, 1, 32)
    coded, tree = pipeline(pts, 1, 32)
    monkeypatch.setenv("LO_REC_CAP", str(cap))
    for r in (1.0, 3.0):
        got = check_radius(tree, coded, p, r)
        assert got.mean_count > 10
        check_radius(tree, coded, p, r, shape=2)
        check_radius(tree, coded, p, r, method=3)


def test_two_walk_radius_path(ctx, ref, oracle, monkeypatch):
    """LO_RADIUS_NO_FUSE=1: count walk, u64 scan, fill walk (no records)."""
    pts = oracle.gen_mixed(80_000, 9)
    p = ref.pipeline(pts, 1, 64)
    coded, tree = pipeline(pts, 1, 64)
    monkeypatch.setenv("LO_RADIUS_NO_FUSE", "1")
    for r in (0.5, 2.0, 6.0):
        for shape in (0, 1):
            check_radius(tree, coded, p, r, shape=shape)


def test_fused_digest_pass(ctx, ref, oracle, monkeypatch):
    """LO_DIGEST_FUSED=1: row digests hashed by the count pass as members are found (in row order)
    instead of the stand-alone radius_digest kernel over the CSR; both equal the reference."""
    pts = oracle.gen_mixed(90_000, 13)
    p = ref.pipeline(pts, 1, 64)
    coded, tree = pipeline(pts, 1, 64)
    for r in (0.7, 3.0):
        check_radius(tree, coded, p, r)
        monkeypatch.setenv("LO_DIGEST_FUSED", "1")
        check_radius(tree, coded, p, r)
        check_radius(tree, coded, p, r, shape=1)
        monkeypatch.delenv("LO_DIGEST_FUSED")


KNN_VARIANTS = {
    "select": {"LO_KNN_SELECT": "1"},                        # bound + collect + warp select
    "select_overflow": {"LO_KNN_SELECT": "1", "LO_KNN_CAP": "1", "LO_KNN_WIN": "1"},  # 32-entry lists
    "select_chunked": {"LO_KNN_SELECT": "1", "LO_KNN_LIST_MB": "1"},  # 32k-query chunks
    "heaps": {"LO_KNN_SELECT": "0"},                         # per-lane heaps (knn_float.cuh, default)
    "warp": {"LO_KNN_WARP": "1"},                            # warp-cooperative heaps (knn_warp.cuh)
}


@pytest.mark.parametrize("variant", sorted(KNN_VARIANTS))
def test_knn_kernels_k_up_to_64(ctx, ref, oracle, monkeypatch, variant):
    """Every kNN kernel path for k <= 64: the candidate-selection path (knn_select.cuh),
    with most queries overflowing into the heap fallback, in small chunks, the per-lane heaps and
    the warp-cooperative heaps.  Full mode and RandomSubset (per-query seed windows)."""
    pts = oracle.gen_mixed(70_000, 17)
    p = ref.pipeline(pts, 1, 64)
    coded, tree = pipeline(pts, 1, 64)
    for key, val in KNN_VARIANTS[variant].items():
        monkeypatch.setenv(key, val)
    for k in (1, 2, 8, 16, 31, 32, 33, 48, 64):
        check_knn(tree, coded, p, k)
        want = p.knn(k, mode=1, subset=3000, seed=k)
        got = lo.run_knn_batch(tree, coded, k, lo.BatchOptions(mode=lo.BatchMode.RandomSubset, subset_size=3000,
                                                               seed=k))
        assert np.array_equal(got.fingerprints, want["fps"]), k


@pytest.mark.parametrize("jitter", [0.0, 1e-9])
def test_knn_select_ties(ctx, ref, monkeypatch, jitter):
    """A lattice: many candidates at exactly equal distances (order by index) or, with a 1e-9
    jitter, at distances equal in their FP32 round-up but not in FP64 (the selection re-sorts those
    runs by the exact (dist_sq, index))."""
    g = np.arange(36, dtype=np.float64)
    pts = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3) + 100.0
    if jitter:
        pts = pts + np.random.default_rng(5).uniform(-jitter, jitter, pts.shape)
    p = ref.pipeline(pts, 1, 32)
    coded, tree = pipeline(pts, 1, 32)
    for sel in ("1", "0"):
        monkeypatch.setenv("LO_KNN_SELECT", sel)
        for k in (7, 8, 19, 27, 33, 64):
            check_knn(tree, coded, p, k)


def test_knobs_off_again(ctx, ref, oracle):
    """The knobs are read per call: with none set the default (filtered, fused) path runs and agrees."""
    pts = oracle.gen_uniform(50_000, 12, 60.0)
    p = ref.pipeline(pts, 0, 32)
    coded, tree = pipeline(pts, 0, 32)
    check_radius(tree, coded, p, 2.5)
    check_knn(tree, coded, p, 16)
