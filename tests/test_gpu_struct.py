"""GPU parity of RadiusMethod::Struct (neighbours_struct, search.cpp:76-135; RangedResult,
search.hpp:18-56): the coalesced contained ranges and the singles must be the reference's
exactly -- they depend on the reference's padded octant boxes, not only on the index set --
and the Struct digests (search.cpp:325-336) must match.  Checked against the golden vectors
(reference output), the C restatement (oracle/) and, when built, the reference library."""
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


def pipeline(points, curve, n_max, level=21):
    coded = lo.reorder_cloud(points, lo.Curve(curve), level)
    return coded, lo.LinearOctree(coded, n_max)


def rows(res, i):
    e = res.extra
    return (e["ranges"][e["range_offsets"][i]:e["range_offsets"][i + 1]],
            e["singles"][e["single_offsets"][i]:e["single_offsets"][i + 1]])


@pytest.mark.parametrize("name", golden_cases())
def test_struct_golden(ctx, name):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    curve, level, n_max = int(g["curve"]), int(g["level"]), int(g["n_max"])
    coded, tree = pipeline(g["points"], curve, n_max, level)
    res = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Struct, lo.KernelShape(int(g["shape"])),
                              float(g["radius"]), lo.BatchOptions(collect_results=True))
    assert np.array_equal(res.counts, g["struct_counts"])
    assert np.array_equal(res.fingerprints, g["struct_fps"])
    # expansion == the Lin rows
    assert np.array_equal(res.offsets, g["radius_offsets"])
    assert np.array_equal(res.indices, g["radius_indices"])
    ro, rg, so, sg = (g["struct_range_offsets"], g["struct_ranges"], g["struct_single_offsets"],
                      g["struct_singles"])
    for q in range(len(ro) - 1):
        ranges, singles = rows(res, q)
        assert np.array_equal(ranges, rg[ro[q]:ro[q + 1]])
        assert np.array_equal(singles, sg[so[q]:so[q + 1]])


CASES = [("uniform", 30000, 21, 0, 32), ("uniform", 30000, 22, 1, 8), ("terrain", 40000, 23, 1, 32),
         ("mixed", 40000, 24, 1, 64), ("terrain", 20000, 25, 0, 1)]


def gen(oracle, kind, n, seed):
    if kind == "uniform":
        return oracle.gen_uniform(n, seed, 100.0)
    if kind == "terrain":
        return oracle.gen_terrain(n, seed, 200.0)
    return oracle.gen_mixed(n, seed)


@pytest.mark.parametrize("kind,n,seed,curve,n_max", CASES)
def test_struct_points_vs_oracle(ctx, oracle, kind, n, seed, curve, n_max):
    pts = gen(oracle, kind, n, seed)
    coded, tree = pipeline(pts, curve, n_max)
    xs = coded.cloud.points
    la = tree.leaves()
    nodes, root = tree.internal_nodes(), tree.root()
    rng = np.random.default_rng(seed)
    lo_b, hi_b = xs.min(0), xs.max(0)
    on_cloud = xs[rng.integers(0, n, 24)]
    off_cloud = lo_b + rng.random((8, 3)) * (hi_b - lo_b) * 1.2 - 0.1 * (hi_b - lo_b)
    centres = np.concatenate([on_cloud, off_cloud])
    ext = float((hi_b - lo_b).max())
    for shape in range(4):
        for r in (0.004 * ext, 0.03 * ext, 0.12 * ext):
            got = lo.struct_points(tree, coded, lo.KernelShape(shape), r, centres)
            for c, rr in zip(centres, got):
                cnt, ranges, singles = oracle.radius_struct(xs, la.boundaries, la.offsets, nodes, root,
                                                            coded.disc_box, curve, c, r, shape)
                assert np.array_equal(rr.ranges, ranges), (shape, r)
                assert np.array_equal(rr.singles, singles), (shape, r)
                assert rr.count() == cnt
                assert np.array_equal(rr.expand(), oracle.radius_brute(xs, c, r, shape))


@pytest.mark.parametrize("curve,shape", [(0, 0), (1, 0), (1, 1), (0, 2), (1, 3)])
def test_struct_batch_vs_reference(ctx, oracle, ref, curve, shape):
    pts = oracle.gen_uniform(50000, 31 + curve, 100.0)
    p = ref.pipeline(pts, curve, 32, threads=4)
    coded, tree = pipeline(pts, curve, 32)
    for r in (1.5, 4.0):
        want = p.radius(r, method=3, shape=shape, threads=8)
        got = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Struct, lo.KernelShape(shape), r,
                                  lo.BatchOptions())
        assert np.array_equal(got.counts, want["counts"])
        assert np.array_equal(got.fingerprints, want["fps"])
        sub = p.radius(r, method=3, shape=shape, mode=1, subset=3000, seed=5, threads=8)
        gs = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Struct, lo.KernelShape(shape), r,
                                 lo.BatchOptions(mode=lo.BatchMode.RandomSubset, subset_size=3000, seed=5))
        assert np.array_equal(gs.centers, sub["centers"])
        assert np.array_equal(gs.fingerprints, sub["fps"])
    xs = coded.cloud.points
    for i in range(0, 50000, 4999):
        cnt, ranges, singles = p.radius_struct_point(xs[i], 2.5, shape)
        rr = lo.neighbours_struct(tree, coded, lo.SearchKernel(lo.KernelShape(shape), tuple(xs[i]), 2.5))
        assert np.array_equal(rr.ranges, ranges) and np.array_equal(rr.singles, singles)


def test_struct_degenerate(ctx, oracle):
    # coincident points (leaves beyond n_max at max depth) and a single-leaf tree
    pts = np.repeat(oracle.gen_uniform(40, 3, 10.0), 50, axis=0)
    for n_max in (8, 4096):
        coded, tree = pipeline(pts, 1, n_max)
        xs = coded.cloud.points
        la = tree.leaves()
        for r in (0.01, 2.0, 50.0):
            got = lo.struct_points(tree, coded, lo.KernelShape.Sphere, r, xs[::97])
            for c, rr in zip(xs[::97], got):
                cnt, ranges, singles = oracle.radius_struct(xs, la.boundaries, la.offsets,
                                                            tree.internal_nodes(), tree.root(),
                                                            coded.disc_box, 1, c, r, 0)
                assert np.array_equal(rr.ranges, ranges) and np.array_equal(rr.singles, singles)
