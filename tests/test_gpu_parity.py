"""GPU parity: the B200 path (through the C ABI) against the golden vectors produced by the
reference, the C restatement (oracle/) and, where it was built, the reference library itself
(oracle/_ref).  Bit-exact for codes, permutations, coordinates, tree tables, radius index
sets and kNN (index, dist_sq) lists -- the tolerance is zero."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases

pytestmark = pytest.mark.gpu

lo = pytest.importorskip("paper_2603_06771_b200.linoct")


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    return lo.default_context(0)


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def pipeline(points, curve, n_max, level=21):
    coded = lo.reorder_cloud(points, lo.Curve(curve), level)
    return coded, lo.LinearOctree(coded, n_max)


# ---- golden vectors (reference output, tests/golden) -----------------------------------
@pytest.mark.parametrize("name", golden_cases())
def test_golden_pipeline(ctx, name):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    curve, level, n_max = int(g["curve"]), int(g["level"]), int(g["n_max"])
    coded, tree = pipeline(g["points"], curve, n_max, level)
    assert np.array_equal(coded.codes, g["codes"])
    assert np.array_equal(coded.permutation, g["perm"])
    assert np.array_equal(bits(coded.cloud.points), bits(g["sorted_points"]))
    assert np.array_equal(coded.disc_box, g["disc_box"])
    if level == 21:
        assert np.array_equal(lo.compute_codes(g["points"], lo.Curve(curve)), g["raw_codes"])
    la = tree.leaves()
    assert np.array_equal(la.boundaries, g["boundaries"])
    assert np.array_equal(la.offsets, g["offsets"])
    assert tree.internal_nodes().view(np.uint8).reshape(-1, 56).tobytes() == g["nodes"].tobytes()
    assert tree.root() == int(g["root"])

    opts = lo.BatchOptions(collect_results=True)
    res = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape(int(g["shape"])),
                              float(g["radius"]), opts)
    assert np.array_equal(res.offsets, g["radius_offsets"])
    assert np.array_equal(res.indices, g["radius_indices"])
    assert np.array_equal(res.counts, g["radius_counts"])
    assert np.array_equal(res.fingerprints, g["radius_fps"])

    k = int(g["k"])
    kr = lo.run_knn_batch(tree, coded, k, opts)
    ke = min(k, len(g["points"]))
    assert np.array_equal(kr.indices.reshape(-1, ke), g["knn_idx"])
    assert np.array_equal(bits(kr.distances.reshape(-1, ke)), bits(g["knn_dist"]))
    assert np.array_equal(kr.fingerprints, g["knn_fps"])


# ---- oracle (C restatement) on fresh seeds ---------------------------------------------
CASES = [
    ("uniform", 20000, 11, 0, 32), ("uniform", 20000, 12, 1, 1), ("terrain", 30000, 13, 1, 32),
    ("mixed", 40000, 14, 1, 64), ("mixed", 25000, 15, 0, 7), ("terrain", 12000, 16, 0, 128),
]


def gen(oracle, kind, n, seed):
    if kind == "uniform":
        return oracle.gen_uniform(n, seed, 100.0)
    if kind == "terrain":
        return oracle.gen_terrain(n, seed, 200.0)
    return oracle.gen_mixed(n, seed)


@pytest.mark.parametrize("kind,n,seed,curve,n_max", CASES)
def test_structure_vs_oracle(ctx, oracle, kind, n, seed, curve, n_max):
    pts = gen(oracle, kind, n, seed)
    coded, tree = pipeline(pts, curve, n_max)
    xs, codes, perm, box = oracle.reorder(pts, curve)
    assert np.array_equal(coded.codes, codes)
    assert np.array_equal(coded.permutation, perm)
    assert np.array_equal(bits(coded.cloud.points), bits(xs))
    b, o = oracle.build_leaves(codes, n_max)
    nodes, root = oracle.link(b, o)
    assert np.array_equal(tree.leaves().boundaries, b) and np.array_equal(tree.leaves().offsets, o)
    assert tree.internal_nodes().tobytes() == nodes.tobytes() and tree.root() == root


@pytest.mark.parametrize("shape", [0, 1, 2, 3])
@pytest.mark.parametrize("kind,n,seed,curve,n_max", CASES[:4])
def test_radius_vs_bruteforce(ctx, oracle, kind, n, seed, curve, n_max, shape):
    pts = gen(oracle, kind, n, seed)
    coded, tree = pipeline(pts, curve, n_max)
    xs = coded.cloud.points
    rng = np.random.default_rng(seed * 10 + shape)
    for r in (0.8, 3.0, 11.0):
        res = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape(shape), r,
                                  lo.BatchOptions(collect_results=True))
        for q in rng.choice(len(xs), 40, replace=False):
            want = oracle.radius_brute(xs, xs[q], r, shape)
            got = res.indices[res.offsets[q]:res.offsets[q + 1]]
            assert np.array_equal(got, want), (r, q)
            assert int(res.fingerprints[q]) == oracle.fnv_radius(want)


@pytest.mark.parametrize("k", [1, 8, 16, 33, 64, 200])
@pytest.mark.parametrize("kind,n,seed,curve,n_max", CASES[:4])
def test_knn_vs_bruteforce(ctx, oracle, kind, n, seed, curve, n_max, k):
    pts = gen(oracle, kind, n, seed)
    coded, tree = pipeline(pts, curve, n_max)
    xs = coded.cloud.points
    res = lo.run_knn_batch(tree, coded, k, lo.BatchOptions(collect_results=True))
    rng = np.random.default_rng(seed + k)
    for q in rng.choice(len(xs), 40, replace=False):
        i, d = oracle.knn_brute(xs, xs[q], k)
        assert np.array_equal(res.indices[q * k:(q + 1) * k], i), q
        assert np.array_equal(bits(res.distances[q * k:(q + 1) * k]), bits(d))
        assert int(res.fingerprints[q]) == oracle.fnv_knn(i, d)


def test_knn_large_k_global_heap(ctx, oracle):
    pts = oracle.gen_uniform(6000, 21, 100.0)
    coded, tree = pipeline(pts, 1, 32)
    xs = coded.cloud.points
    k = 700  # beyond the shared-memory heap budget
    idx, dist = lo.knn_points(tree, coded, xs[::500], k)
    for row, q in enumerate(range(0, len(xs), 500)):
        i, d = oracle.knn_brute(xs, xs[q], k)
        assert np.array_equal(idx[row], i) and np.array_equal(bits(dist[row]), bits(d))


def test_grid_ties_offcloud_centres(ctx, oracle):
    g = np.arange(12, dtype=float)
    pts = np.array([[x, y, z] for x in g for y in g for z in g])
    coded, tree = pipeline(pts, 0, 16)
    xs = coded.cloud.points
    rng = np.random.default_rng(37)
    centres = np.concatenate([xs[rng.choice(len(xs), 30)], rng.uniform(-2, 14, (30, 3)),
                              np.floor(rng.uniform(0, 12, (20, 3))) + 0.5])
    for k in (1, 6, 27, 100):
        idx, dist = lo.knn_points(tree, coded, centres, k)
        for row, c in enumerate(centres):
            i, d = oracle.knn_brute(xs, c, k)
            assert np.array_equal(idx[row], i) and np.array_equal(bits(dist[row]), bits(d))
    rows = lo.radius_points(tree, coded, lo.KernelShape.Sphere, 1.0, centres)
    for row, c in zip(rows, centres):
        assert np.array_equal(row, oracle.radius_brute(xs, c, 1.0, 0))


@pytest.mark.parametrize("shape", [0, 1, 2, 3])
def test_boundary_band_exact(ctx, oracle, shape):
    """Points placed within a few ulps of the kernel boundary: the FP32 filter must hand
    them to the exact FP64 predicate (strict '<' of geometry.hpp:127-140)."""
    rng = np.random.default_rng(77 + shape)
    centres = rng.uniform(200, 800, (64, 3))
    r = 2.75
    pts = [rng.uniform(0, 1000, (20000, 3))]
    for c in centres:
        d = rng.normal(size=(200, 3))
        if shape in (1, 3):
            d[:, 2] = 0.0
        if shape in (0, 1):
            d /= np.linalg.norm(d, axis=1, keepdims=True)
        else:
            d /= np.abs(d).max(axis=1, keepdims=True)
        scale = r * (1.0 + rng.choice([-1, 0, 1], 200)[:, None] * rng.uniform(0, 4e-16, (200, 1)))
        shell = c + d * scale
        if shape in (1, 3):
            shell[:, 2] = c[2] + rng.uniform(-5, 5, 200)
        pts.append(shell)
        pts.append(c[None, :])
    pts = np.concatenate(pts)
    coded, tree = pipeline(pts, 1, 32)
    xs = coded.cloud.points
    inv = lo.invert_permutation(coded.permutation)
    base = 20000
    qidx = [int(inv[base + i * 201 + 200]) for i in range(len(centres))]
    res = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape(shape), r,
                              lo.BatchOptions(collect_results=True))
    for q in qidx:
        want = oracle.radius_brute(xs, xs[q], r, shape)
        assert np.array_equal(res.indices[res.offsets[q]:res.offsets[q + 1]], want)


# ---- edge cases the reference tests -------------------------------------------------------
def test_edge_cases(ctx, oracle):
    with pytest.raises(lo.InvalidArgument):
        lo.reorder_cloud(np.zeros((0, 3)), lo.Curve.Morton)
    with pytest.raises(lo.InvalidArgument):
        lo.compute_codes(np.zeros((0, 3)), lo.Curve.Hilbert)
    with pytest.raises(lo.InvalidArgument):
        lo.build_leaves(np.array([3, 2, 1], np.uint64), 8)
    with pytest.raises(lo.InvalidArgument):
        lo.build_leaves(np.zeros(0, np.uint64), 8)
    with pytest.raises(lo.InvalidArgument):
        lo.build_leaves(np.array([1, 2, 3], np.uint64), 0)
    with pytest.raises(lo.InvalidArgument):
        lo.build_leaves(np.array([1, 2, 1 << 63], np.uint64), 8)
    bad = np.array([[0.0, 0.0, 0.0], [1.0, np.inf, 2.0]])
    with pytest.raises(lo.InvalidArgument, match="non-finite coordinate at point 1"):
        lo._lib.check(lo._lib.lib().lo_reorder(lo.default_context().h, lo._p(bad), 2, 0, 21,
                                               lo.C.byref(lo.C.c_void_p())))
    with pytest.raises(lo.DomainError):
        lo.compute_codes(np.array([[9.0, 0.0, 0.0]]), lo.Curve.Morton,
                         disc_box=np.array([0, 0, 0, 8, 8, 8.0]))
    # single point, root leaf, k > N
    coded, tree = pipeline(np.array([[1.0, 2.0, 3.0]]), 1, 128)
    assert tree.leaf_count() == 1 and tree.internal_count() == 0 and tree.root() == -1
    assert list(tree.leaves().boundaries) == [0, 1 << 63]
    res = lo.run_knn_batch(tree, coded, 5, lo.BatchOptions(collect_results=True))
    assert list(res.indices) == [0] and res.distances[0] == 0.0
    with pytest.raises(lo.InvalidArgument):
        lo.run_knn_batch(tree, coded, 0, lo.BatchOptions())
    with pytest.raises(lo.InvalidArgument):
        lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, 0.0, lo.BatchOptions())
    with pytest.raises(lo.InvalidArgument):
        lo.run_radius_batch(tree, coded, lo.RadiusMethod.Ptr, lo.KernelShape.Sphere, 1.0, lo.BatchOptions())
    with pytest.raises(lo.InvalidArgument):
        lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, 1.0,
                            lo.BatchOptions(mode=lo.BatchMode.RandomSubset, subset_size=2))
    # all-inclusive and disjoint kernels (test_search.cpp:41-49)
    pts = oracle.gen_uniform(2000, 1, 100.0)
    coded, tree = pipeline(pts, 0, 64)
    assert len(lo.neighbours_lin(tree, coded, lo.SearchKernel(lo.KernelShape.Sphere, (-900, 0, 0), 2))) == 0
    allp = lo.neighbours_lin(tree, coded, lo.SearchKernel(lo.KernelShape.Sphere, (50, 50, 50), 1e5))
    assert np.array_equal(allp, np.arange(2000))
    # coincident points stop at single cells; self first with lowest index
    pts = np.array([[5, 5, 5], [1, 1, 1], [1, 1, 1], [9, 9, 9], [1, 1, 1]], float)
    coded, tree = pipeline(pts, 0, 2)
    nb = lo.knn_lin_oct(tree, coded, (1, 1, 1), 1)
    xs = coded.cloud.points
    lowest = min(i for i in range(5) if tuple(xs[i]) == (1, 1, 1))
    assert nb[0].index == lowest and nb[0].dist_sq == 0.0
    # reorder of an already sorted cloud is the identity (test_reorder.cpp:41-50)
    pts = oracle.gen_uniform(2000, 7, 100.0)
    once = lo.reorder_cloud(pts, lo.Curve.Hilbert)
    twice = lo.reorder_cloud(once.cloud.points, lo.Curve.Hilbert)
    assert np.array_equal(twice.permutation, np.arange(2000))
    assert np.array_equal(twice.codes, once.codes)
    inv = lo.invert_permutation(once.permutation)
    assert np.array_equal(once.cloud.points[inv], pts)


def test_codecs_vs_golden(ctx):
    g = np.load(os.path.join(GOLDEN, "kat_cells.npz"))
    assert np.array_equal(lo.sfc_encode(lo.Curve.Morton, g["cells"]), g["morton"])
    assert np.array_equal(lo.sfc_encode(lo.Curve.Hilbert, g["cells"]), g["hilbert"])
    assert np.array_equal(lo.sfc_decode(lo.Curve.Hilbert, g["hilbert"]), g["cells"])
    assert lo.morton_encode((3, 7, 2), 3) == 190
    assert [lo.hilbert_encode(c, 2) for c in [(3, 0, 0), (0, 3, 0), (2, 1, 3)]] == [63, 29, 50]


def test_node_bounds_vs_oracle(ctx, oracle):
    pts = oracle.gen_mixed(20000, 21)
    for curve in (0, 1):
        coded, tree = pipeline(pts, curve, 32)
        box = coded.disc_box
        refs = np.concatenate([np.arange(tree.internal_count()), ~np.arange(tree.leaf_count())]).astype(np.int32)
        got = tree.node_bounds(refs)
        xs = coded.cloud.points
        for row, ref_ in enumerate(refs[::37]):
            ref_ = int(ref_)
            depth = tree.node_depth(ref_)
            prefix = tree.node_prefix(ref_)
            top = prefix >> (3 * (21 - depth))
            h = oracle.hilbert_decode(top, depth) if curve else (
                tuple(int(v) for v in lo.sfc_decode(lo.Curve.Morton, [top], depth)[0]))
            want = oracle.octant_bounds(box, *h, depth)
            assert np.array_equal(bits(got[row * 37]), bits(want))
            b, e = tree.points_in_node(ref_)
            if e > b:  # every node's box contains its points (test_linear_octree.cpp:230-251)
                p = xs[b:e]
                assert (p >= want[:3]).all() and (p <= want[3:]).all()


# ---- the reference itself (oracle/_ref), full cfg0 ----------------------------------------
def test_cfg0_full_vs_reference(ctx, ref):
    pts = lo.generate_uniform(1_000_000, 1000, 100.0)
    p = ref.pipeline(pts, 0, 32)
    xs, codes, perm = p.coded()
    b, o, nodes = p.tree()
    coded, tree = pipeline(pts, 0, 32)
    assert np.array_equal(coded.codes, codes) and np.array_equal(coded.permutation, perm)
    assert np.array_equal(bits(coded.cloud.points), bits(xs))
    assert np.array_equal(tree.leaves().boundaries, b) and np.array_equal(tree.leaves().offsets, o)
    assert tree.internal_nodes().tobytes() == nodes.tobytes()
    want = p.radius(2.5, method=1)
    got = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, 2.5, lo.BatchOptions())
    assert np.array_equal(got.counts, want["counts"])
    assert np.array_equal(got.fingerprints, want["fps"])
    assert abs(got.mean_count - 64.61) < 0.5
    sub = p.knn(16, mode=1, subset=20000, seed=5)
    kr = lo.run_knn_batch(tree, coded, 16, lo.BatchOptions(mode=lo.BatchMode.RandomSubset,
                                                           subset_size=20000, seed=5))
    assert np.array_equal(kr.centers, sub["centers"])
    assert np.array_equal(kr.fingerprints, sub["fps"])


def test_random_subset_and_points_vs_reference(ctx, ref, oracle):
    pts = oracle.gen_mixed(60000, 31)
    p = ref.pipeline(pts, 1, 64)
    coded, tree = pipeline(pts, 1, 64)
    for method in (1, 2):
        want = p.radius(1.5, method=method, mode=1, subset=5000, seed=424242)
        got = lo.run_radius_batch(tree, coded, lo.RadiusMethod(method), lo.KernelShape.Sphere, 1.5,
                                  lo.BatchOptions(mode=lo.BatchMode.RandomSubset, subset_size=5000,
                                                  seed=424242))
        assert np.array_equal(got.centers, want["centers"])
        assert np.array_equal(got.counts, want["counts"])
        assert np.array_equal(got.fingerprints, want["fps"])
    rng = np.random.default_rng(4)
    centres = rng.uniform(coded.disc_box[:3] - 5, coded.disc_box[3:] + 5, (200, 3))
    idx, dist = lo.knn_points(tree, coded, centres, 12)
    for row, c in enumerate(centres):
        i, d = p.knn_point(c, 12)
        assert np.array_equal(idx[row], i) and np.array_equal(bits(dist[row]), bits(d))
    rows = lo.radius_points(tree, coded, lo.KernelShape.Cube, 4.0, centres)
    for row, c in zip(rows, centres):
        assert np.array_equal(row, p.radius_point(c, 4.0, shape=2))
