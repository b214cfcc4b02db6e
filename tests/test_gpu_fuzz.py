"""Randomised parity sweep (seeded, deterministic): many small clouds with random shape, size,
level, curve, leaf bucket, kernel shape, radius, k and query mode, each checked against the C
restatement (brute-force radius / kNN, the Struct traversal) -- bit for bit.  A second sweep runs
mid-size clouds (50k-400k points) through the reference library itself (oracle/_ref, Full mode:
every point a centre, counts + FNV digests of every row, kNN digests).

LO_FUZZ_CASES / LO_FUZZ_REF_CASES scale the sweeps (defaults 120 / 8) for longer campaigns."""
import os

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


def cloud(rng, kind, n):
    if kind == "uniform":
        return rng.random((n, 3)) * rng.choice([1e-3, 1.0, 100.0, 1e4])
    if kind == "clusters":
        c = rng.random((max(1, n // 50), 3)) * 100.0
        return c[rng.integers(0, len(c), n)] + rng.normal(0, 0.5, (n, 3))
    if kind == "coincident":
        base = rng.random((max(1, n // 20), 3)) * 10.0
        return base[rng.integers(0, len(base), n)]
    if kind == "grid":
        m = max(2, int(round(n ** (1 / 3))))
        g = np.arange(m, dtype=float)
        return np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)[:n]
    # flat: all points in a plane (zero-extent axis)
    p = rng.random((n, 3)) * 50.0
    p[:, 2] = 7.0
    return p


@pytest.mark.parametrize("case", range(int(os.environ.get("LO_FUZZ_CASES", "120"))))
def test_fuzz_against_oracle(ctx, oracle, case):
    rng = np.random.default_rng(1000 + case)
    kind = ["uniform", "clusters", "coincident", "grid", "flat"][case % 5]
    n = int(rng.integers(1, 4000))
    pts = cloud(rng, kind, n)
    n = len(pts)
    curve = int(rng.integers(0, 2))
    level = int(rng.choice([1, 2, 5, 10, 21, 21, 21]))
    n_max = int(rng.choice([1, 2, 7, 32, 128, 1000]))
    coded = lo.reorder_cloud(pts, lo.Curve(curve), level)
    tree = lo.LinearOctree(coded, n_max)
    xs, codes, perm, box = oracle.reorder(pts, curve, level)
    assert np.array_equal(coded.codes, codes) and np.array_equal(coded.permutation, perm)
    b, o = oracle.build_leaves(codes, n_max, level)
    la = tree.leaves()
    assert np.array_equal(la.boundaries, b) and np.array_equal(la.offsets, o)
    nodes, root = oracle.link(b, o, level)
    assert tree.internal_nodes().tobytes() == nodes.tobytes() and tree.root() == root
    ext = float(np.ptp(xs, axis=0).max()) or 1.0
    shape = int(rng.integers(0, 4))
    r = float(ext * rng.choice([1e-4, 0.01, 0.05, 0.2, 2.0]))
    # radius (Full) + Struct rows on a few centres
    res = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape(shape), r,
                              lo.BatchOptions(collect_results=True))
    qs = rng.integers(0, n, min(n, 40))
    for q in qs:
        want = oracle.radius_brute(xs, xs[q], r, shape)
        assert np.array_equal(res.results[q], want), (kind, n, shape, r)
        assert res.fingerprints[q] == oracle.fnv_radius(want)
    st = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Struct, lo.KernelShape(shape), r,
                             lo.BatchOptions(mode=lo.BatchMode.RandomSubset, subset_size=min(n, 60), seed=case))
    for i, c in enumerate(st.centers):
        cnt, ranges, singles = oracle.radius_struct(xs, b, o, nodes, root, box, curve, xs[c], r, shape, level)
        e = st.extra
        assert np.array_equal(e["ranges"][e["range_offsets"][i]:e["range_offsets"][i + 1]], ranges)
        assert np.array_equal(e["singles"][e["single_offsets"][i]:e["single_offsets"][i + 1]], singles)
        assert st.counts[i] == cnt
    # kNN: Full mode and off-cloud points
    k = int(rng.choice([1, 3, 8, 16, 33, 64, n + 5]))
    kr = lo.run_knn_batch(tree, coded, k, lo.BatchOptions(collect_results=True), collect_distances=True)
    ke = min(k, n)
    for q in qs[:15]:
        i, d = oracle.knn_brute(xs, xs[q], k)
        assert np.array_equal(kr.indices.reshape(-1, ke)[q], i), (kind, n, k)
        assert np.array_equal(kr.distances.reshape(-1, ke)[q].view(np.uint64), d.view(np.uint64))
    off = xs.min(0) + rng.random((10, 3)) * (np.ptp(xs, axis=0) + ext * 0.3) - ext * 0.15
    idx, dist = lo.knn_points(tree, coded, off, k)
    for j, c in enumerate(off):
        i, d = oracle.knn_brute(xs, c, k)
        assert np.array_equal(idx[j], i) and np.array_equal(dist[j].view(np.uint64), d.view(np.uint64))
    rows = lo.radius_points(tree, coded, lo.KernelShape(shape), r, off)
    for j, c in enumerate(off):
        assert np.array_equal(rows[j], oracle.radius_brute(xs, c, r, shape))


def midsize_cloud(rng, oracle, kind, n):
    seed = int(rng.integers(1, 1 << 30))
    if kind == "uniform":
        return oracle.gen_uniform(n, seed, float(rng.choice([10.0, 100.0, 1000.0])))
    if kind == "terrain":
        return oracle.gen_terrain(n, seed, float(rng.choice([100.0, 300.0, 1000.0])))
    if kind == "mixed":
        return oracle.gen_mixed(n, seed)
    # dense clusters in a large empty cube (sparse tiles, long curve jumps)
    c = rng.random((max(1, n // 2000), 3)) * 5000.0
    return c[rng.integers(0, len(c), n)] + rng.normal(0, float(rng.choice([0.3, 2.0])), (n, 3))


@pytest.mark.parametrize("case", range(int(os.environ.get("LO_FUZZ_REF_CASES", "8"))))
def test_fuzz_midsize_against_reference(ctx, oracle, ref, case):
    rng = np.random.default_rng(77_000 + case)
    kind = ["uniform", "terrain", "mixed", "clusters"][case % 4]
    n = int(rng.integers(50_000, 400_000))
    pts = midsize_cloud(rng, oracle, kind, n)
    curve = int(rng.integers(0, 2))
    n_max = int(rng.choice([8, 32, 64, 200]))
    p = ref.pipeline(pts, curve, n_max)
    coded = lo.reorder_cloud(pts, lo.Curve(curve))
    tree = lo.LinearOctree(coded, n_max)
    # a radius that gives ~mu neighbours on average: from the k-th neighbour distance of a sample
    from scipy.spatial import cKDTree
    mu = int(rng.choice([4, 16, 64, 200]))
    xs = coded.cloud.points
    d, _ = cKDTree(xs).query(xs[rng.integers(0, len(xs), 256)], k=mu + 1)
    r = float(np.median(d[:, -1])) or 1.0
    shape = int(rng.integers(0, 4))
    want = p.radius(r, shape=shape)
    got = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape(shape), r, lo.BatchOptions())
    assert np.array_equal(got.counts, want["counts"]), (kind, n, curve, n_max, shape, r)
    assert np.array_equal(got.fingerprints, want["fps"]), (kind, n, curve, n_max, shape, r)
    k = int(rng.choice([1, 8, 16, 32, 64]))
    kw = p.knn(k)
    kg = lo.run_knn_batch(tree, coded, k, lo.BatchOptions())
    assert np.array_equal(kg.fingerprints, kw["fps"]), (kind, n, curve, n_max, k)
