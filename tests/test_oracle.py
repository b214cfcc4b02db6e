"""The C restatement (oracle/) pinned against the reference's known answers and golden
vectors (tests/golden, produced by the reference library itself)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases

NODE = np.dtype([("prefix", "<u8"), ("children", "<i4", (8,)), ("begin", "<u4"), ("end", "<u4"),
                 ("depth", "u1"), ("child_mask", "u1"), ("pad_", "u1", (6,))])


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def test_kat_codes(oracle):
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))
    for x, y, z, level, want in kat["morton"]:
        assert oracle.morton(x, y, z) == want
    assert kat["morton"][0][-1] == 190  # test_sfc.cpp:62-65
    for x, y, z, level, want in kat["hilbert_l2"]:
        assert oracle.hilbert(x, y, z, level) == want
    assert [v[-1] for v in kat["hilbert_l2"]] == [0, 63, 29, 9, 45, 50, 31, 48]  # test_sfc.cpp:106-113
    assert [list(oracle.hilbert_decode(c, 1)) for c in range(8)] == kat["hilbert_l1_path"]


def test_kat_random_cells(oracle):
    g = np.load(os.path.join(GOLDEN, "kat_cells.npz"))
    for c, m, h in zip(g["cells"][:1024], g["morton"][:1024], g["hilbert"][:1024]):
        assert oracle.morton(*map(int, c)) == int(m)
        assert oracle.hilbert(*map(int, c)) == int(h)
        assert oracle.hilbert_decode(int(h)) == tuple(int(v) for v in c)


def test_stepper_tables(oracle):
    d, n = oracle.stepper(1)
    assert len(d) == 24
    d0, _ = oracle.stepper(0)
    assert len(d0) == 1


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_matches_golden(oracle, name):
    g = load(name)
    pts, curve, level, n_max = g["points"], int(g["curve"]), int(g["level"]), int(g["n_max"])
    xs, codes, perm, box = oracle.reorder(pts, curve, level)
    assert np.array_equal(codes, g["codes"])
    assert np.array_equal(perm, g["perm"])
    assert np.array_equal(xs.view(np.uint64), g["sorted_points"].view(np.uint64))
    assert np.array_equal(box, g["disc_box"])
    if level == 21:
        raw, _ = oracle.compute_codes(pts, curve)
        assert np.array_equal(raw, g["raw_codes"])
    b, o = oracle.build_leaves(codes, n_max, level)
    assert np.array_equal(b, g["boundaries"]) and np.array_equal(o, g["offsets"])
    nodes, root = oracle.link(b, o, level)
    assert nodes.view(np.uint8).reshape(-1, 56).tobytes() == g["nodes"].tobytes()
    assert root == int(g["root"])
    # radius rows (brute force) and digests on a spread of centres
    r, shape = float(g["radius"]), int(g["shape"])
    offs, idx = g["radius_offsets"], g["radius_indices"]
    for q in range(0, len(xs), max(1, len(xs) // 97)):
        want = idx[offs[q]:offs[q + 1]]
        assert np.array_equal(oracle.radius_brute(xs, xs[q], r, shape), want)
        assert oracle.fnv_radius(want) == int(g["radius_fps"][q])
    k = int(g["k"])
    for q in range(0, len(xs), max(1, len(xs) // 97)):
        i, d = oracle.knn_brute(xs, xs[q], k)
        assert np.array_equal(i, g["knn_idx"][q])
        assert np.array_equal(d.view(np.uint64), g["knn_dist"][q].view(np.uint64))
        assert oracle.fnv_knn(i, d) == int(g["knn_fps"][q])
    # RadiusMethod::Struct: the reference's RangedResult rows and Struct digests
    ro, rg, so, sg = (g["struct_range_offsets"], g["struct_ranges"], g["struct_single_offsets"],
                      g["struct_singles"])
    for q in range(len(ro) - 1):
        cnt, ranges, singles = oracle.radius_struct(xs, b, o, nodes, root, box, curve, xs[q], r, shape,
                                                    level)
        assert np.array_equal(ranges, rg[ro[q]:ro[q + 1]])
        assert np.array_equal(singles, sg[so[q]:so[q + 1]])
        assert cnt == int(g["struct_counts"][q]) == int(g["radius_counts"][q])
        assert oracle.fnv_struct(ranges, singles) == int(g["struct_fps"][q])


def test_generators_match_reference(oracle, ref):
    assert np.array_equal(oracle.gen_uniform(5000, 42, 100.0), ref.gen_uniform(5000, 42, 100.0))
    assert np.array_equal(oracle.sample_indices(10000, 500, 9), ref.sample_indices(10000, 500, 9))


def test_octant_bounds_match_reference(oracle, ref):
    rng = np.random.default_rng(3)
    box = np.array([-1.7, 2.3, -9.1, -1.7 + 12.4, 2.3 + 12.4, -9.1 + 12.4])
    for _ in range(500):
        depth = int(rng.integers(0, 22))
        h = rng.integers(0, 1 << depth, 3) if depth else np.zeros(3, int)
        a = oracle.octant_bounds(box, *map(int, h), depth)
        b = ref.octant_bounds(box, *map(int, h), depth)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_oracle_pipeline_vs_reference_random(oracle, ref):
    """Restatement vs the live reference on fresh seeds (not only the frozen fixtures)."""
    for seed, curve, n_max in [(101, 0, 8), (102, 1, 32), (103, 1, 1)]:
        pts = oracle.gen_mixed(4000, seed)
        p = ref.pipeline(pts, curve, n_max, threads=2)
        xs, codes, perm = p.coded()
        b, o, nodes = p.tree()
        xs2, codes2, perm2, _ = oracle.reorder(pts, curve)
        assert np.array_equal(codes, codes2) and np.array_equal(perm, perm2)
        b2, o2 = oracle.build_leaves(codes2, n_max)
        assert np.array_equal(b, b2) and np.array_equal(o, o2)
        n2, root = oracle.link(b2, o2)
        assert n2.tobytes() == nodes.tobytes() and root == p.root
