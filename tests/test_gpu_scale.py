"""Full-size parity on the BASELINE configs against the reference library itself
(oracle/_ref, the unmodified reference sources), every point a centre (BatchMode::Full):

- cfg1 / cfg2: 10M terrain, Hilbert, leaf 32: r = 0.5 / 1 / 2 / 3 and k = 8 / 16 / 32 / 64;
- cfg4: 50M uniform, Hilbert, leaf 32: r = 3, k = 16;
- cfg3: 100M mixed, Hilbert, leaf 64: r = 1, k = 16 (6.4 G neighbours, u64 CSR offsets);
- cfg3 RandomSubset (the reference's sample_indices) with 250k centres.

Structure (sorted codes, permutation, reordered coordinates, LeafArray, InternalNode table) is
compared bit for bit; radius rows by count + FNV-1a digest per centre and kNN rows by the
(index, dist_sq) digest per centre (search.cpp:263-271, :345-347, :376-381) -- the reference
digests instead of keeping 25 GB of rows at 100M points, and so do these tests.  cfg0 is covered
in full by test_gpu_parity.py::test_cfg0_full_vs_reference.  Inputs come from the oracle's
generators (rng.hpp draw order)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

lo = pytest.importorskip("paper_2603_06771_b200.linoct")

CFGS = {
    "cfg1": dict(kind="terrain", n=10_000_000, seed=1001, extent=1000.0, curve=1, n_max=32,
                 radii=[0.5, 1.0, 2.0, 3.0], ks=[8, 16, 32, 64]),
    "cfg4": dict(kind="uniform", n=50_000_000, seed=1004, extent=500.0, curve=1, n_max=32, radii=[3.0], ks=[16]),
    "cfg3": dict(kind="mixed", n=100_000_000, seed=1003, curve=1, n_max=64, radii=[1.0], ks=[16]),
}


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    return lo.default_context(0)


def generate(oracle, cfg):
    if cfg["kind"] == "uniform":
        return oracle.gen_uniform(cfg["n"], cfg["seed"], cfg["extent"])
    if cfg["kind"] == "terrain":
        return oracle.gen_terrain(cfg["n"], cfg["seed"], cfg["extent"])
    return oracle.gen_mixed(cfg["n"], cfg["seed"])


def structure_equal(coded, tree, p):
    xs, codes, perm = p.coded()
    assert np.array_equal(coded.codes, codes)
    assert np.array_equal(coded.permutation, perm)
    assert np.array_equal(coded.cloud.points.view(np.uint64), xs.view(np.uint64))
    del xs, codes, perm
    b, o, nodes = p.tree()
    la = tree.leaves()
    assert np.array_equal(la.boundaries, b) and np.array_equal(la.offsets, o)
    assert tree.internal_nodes().tobytes() == nodes.tobytes() and tree.root() == p.root


@pytest.fixture(scope="module")
def cfg3(ctx, ref, oracle):
    cfg = CFGS["cfg3"]
    pts = generate(oracle, cfg)
    p = ref.pipeline(pts, cfg["curve"], cfg["n_max"])
    coded = lo.reorder_cloud(pts, lo.Curve(cfg["curve"]))
    del pts
    tree = lo.LinearOctree(coded, cfg["n_max"])
    return cfg, p, coded, tree


@pytest.mark.parametrize("name", ["cfg1", "cfg4"])
def test_full_size_parity(ctx, ref, oracle, name):
    cfg = CFGS[name]
    pts = generate(oracle, cfg)
    p = ref.pipeline(pts, cfg["curve"], cfg["n_max"])
    coded = lo.reorder_cloud(pts, lo.Curve(cfg["curve"]))
    del pts
    tree = lo.LinearOctree(coded, cfg["n_max"])
    structure_equal(coded, tree, p)
    for r in cfg["radii"]:
        want = p.radius(r, method=1)
        got = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, r, lo.BatchOptions())
        assert np.array_equal(got.counts, want["counts"]), r
        assert np.array_equal(got.fingerprints, want["fps"]), r
    for k in cfg["ks"]:
        want = p.knn(k)
        got = lo.run_knn_batch(tree, coded, k, lo.BatchOptions())
        assert np.array_equal(got.fingerprints, want["fps"]), k


def test_cfg3_full_structure(cfg3):
    cfg, p, coded, tree = cfg3
    structure_equal(coded, tree, p)


def test_cfg3_full_radius(cfg3):
    cfg, p, coded, tree = cfg3
    want = p.radius(1.0, method=1)
    got = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, 1.0, lo.BatchOptions())
    assert np.array_equal(got.counts, want["counts"])
    assert np.array_equal(got.fingerprints, want["fps"])
    assert got.counts.astype(np.uint64).sum() > 2 ** 32  # u64 CSR offsets are exercised


def test_cfg3_full_knn(cfg3):
    cfg, p, coded, tree = cfg3
    want = p.knn(16)
    got = lo.run_knn_batch(tree, coded, 16, lo.BatchOptions())
    assert np.array_equal(got.fingerprints, want["fps"])


def test_cfg3_random_subset(cfg3):
    """RandomSubset (sample_indices, rng.hpp:46-58) of 250k centres: scattered centres are searched in
    curve order and scattered back (centres.cu); counts, digests and kNN digests vs the reference."""
    cfg, p, coded, tree = cfg3
    for method in (1, 3):
        want = p.radius(1.0, method=method, mode=1, subset=250_000, seed=2026)
        got = lo.run_radius_batch(tree, coded, lo.RadiusMethod(method), lo.KernelShape.Sphere, 1.0,
                                  lo.BatchOptions(mode=lo.BatchMode.RandomSubset, subset_size=250_000, seed=2026))
        assert np.array_equal(got.centers, want["centers"])
        assert np.array_equal(got.counts, want["counts"])
        assert np.array_equal(got.fingerprints, want["fps"])
    want = p.knn(16, mode=1, subset=250_000, seed=2027)
    got = lo.run_knn_batch(tree, coded, 16, lo.BatchOptions(mode=lo.BatchMode.RandomSubset, subset_size=250_000,
                                                           seed=2027))
    assert np.array_equal(got.centers, want["centers"])
    assert np.array_equal(got.fingerprints, want["fps"])
