"""Locality statistics: the exact kNN index-distance histogram
(locality.cpp:41-97) computed on the device, and its statistics (mean, stddev, Fisher-Pearson
G1, quartiles; locality.cpp:13-140) -- bins equal the reference's, statistics bit-equal."""
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


def stats(h):
    q = lo.histogram_quantiles(h)
    return np.array([h.mean(), h.stddev(), lo.fisher_pearson_skewness(h), *q])


@pytest.mark.parametrize("curve,k,perm", [(0, 8, False), (1, 16, False), (1, 16, True), (0, 5, True)])
def test_locality_exact_vs_reference(ctx, ref, oracle, curve, k, perm):
    pts = oracle.gen_uniform(60000, 40 + k, 100.0)
    rp = ref.pipeline(pts, curve, 32, threads=8)
    coded = lo.reorder_cloud(pts, lo.Curve(curve))
    tree = lo.LinearOctree(coded, 32)
    d, c, want = rp.locality_stats(k, use_perm_map=perm, threads=8)
    h = lo.locality_histogram(tree, coded, k, index_map=coded.permutation if perm else None)
    assert np.array_equal(h.d, d) and np.array_equal(h.count, c)
    assert h.total() == k * len(pts) and h.count_at(0) == len(pts)
    assert np.array_equal(stats(h).view(np.uint64), want.view(np.uint64))


def test_locality_approx_vs_reference(ctx, ref, oracle):
    pts = oracle.gen_terrain(80000, 12, 100.0)
    rp = ref.pipeline(pts, 1, 32, threads=8)
    coded = lo.reorder_cloud(pts, lo.Curve.Hilbert)
    tree = lo.LinearOctree(coded, 32)
    d, c, want = rp.locality_stats(16, sample=5000, seed=77, threads=8)
    h = lo.locality_histogram_approx(tree, coded, 16, 5000, 77)
    assert np.array_equal(h.d, d) and np.array_equal(h.count, c)
    assert np.array_equal(stats(h).view(np.uint64), want.view(np.uint64))
    with pytest.raises(lo.InvalidArgument, match="k exceeds cloud size"):
        lo.locality_histogram(tree, coded, 80001)
    with pytest.raises(lo.InvalidArgument, match="sample size exceeds"):
        lo.locality_histogram_approx(tree, coded, 4, 80001, 1)
    with pytest.raises(lo.InvalidArgument, match="index map size mismatch"):
        lo.locality_histogram(tree, coded, 4, index_map=np.arange(5, dtype=np.uint32))


def test_memory_report(ctx, oracle):
    pts = oracle.gen_uniform(50000, 3, 100.0)
    coded = lo.reorder_cloud(pts, lo.Curve.Morton)
    tree = lo.LinearOctree(coded, 32)
    rep = lo.measure_structure(tree)
    la = tree.leaves()
    assert rep.bytes_total == la.boundaries.nbytes + la.offsets.nbytes + 56 * tree.internal_count()
    assert rep.node_count == tree.leaf_count() + tree.internal_count() and rep.point_count == 50000
    p = lo.linear_octree_cost_params(rep.rho())
    assert p.node_bytes == (7 * 12 + 56) / 8 and lo.expected_overhead(p) == rep.rho() * p.node_bytes / 32.0
