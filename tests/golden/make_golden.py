"""Generates tests/golden/*.npz + kat.json from the UNMODIFIED reference library.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It builds oracle/_ref/libref_linoct.so from /root/reference/proj/src (oracle/Makefile) and
records, for a handful of small seeded clouds, everything the hot path produces: codes,
permutation, reordered points, LeafArray, InternalNode table, radius CSR + FNV digests, kNN
lists + digests.  The known-answer values of kat.json are the reference's own test
constants (proj/tests/test_sfc.cpp:62-125, test_linear_octree.cpp:26-34), re-evaluated
through the reference library.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle import oracle_py  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def grid12():
    g = np.arange(12, dtype=np.float64)
    return np.array([[x, y, z] for x in g for y in g for z in g])


def coincident():
    return np.array([[1.0, 1.0, 1.0]] * 10 + [[5.0, 5.0, 5.0]])


def cases(o: oracle_py.Oracle):
    # name, points, curve, n_max, radius, shape, k
    return [
        ("uniform2k_morton", o.gen_uniform(2000, 1, 100.0), 0, 32, 8.0, 0, 10),
        ("uniform3k_hilbert_cube", o.gen_uniform(3000, 7, 100.0), 1, 16, 6.0, 2, 7),
        ("terrain3k_hilbert", o.gen_terrain(3000, 2, 100.0), 1, 16, 3.0, 0, 16),
        ("mixed5k_hilbert", o.gen_mixed(5000, 3), 1, 64, 40.0, 1, 32),
        ("grid12_morton", grid12(), 0, 16, 1.5, 0, 27),
        ("coincident_morton", coincident(), 0, 2, 1.0, 0, 3),
        ("uniform1k_square_level10", o.gen_uniform(1000, 11, 50.0), 1, 8, 4.0, 3, 5),
    ]


def main():
    oracle_py.build(ref=True)
    o = oracle_py.Oracle()
    r = oracle_py.Ref()
    kat = {
        "morton": [[3, 7, 2, 3, int(r.morton(3, 7, 2, 3))], [0, 0, 0, 3, int(r.morton(0, 0, 0, 3))],
                   [1, 1, 1, 3, int(r.morton(1, 1, 1, 3))]],
        "hilbert_l2": [[x, y, z, 2, int(r.hilbert(x, y, z, 2))] for (x, y, z) in
                       [(0, 0, 0), (3, 0, 0), (0, 3, 0), (0, 0, 3), (3, 3, 3), (2, 1, 3), (1, 2, 0),
                        (3, 1, 2)]],
        "hilbert_l1_path": [list(r.hilbert_decode(c, 1)) for c in range(8)],
        "root_leaf_boundaries": [0, 1 << 63],
    }
    rng = np.random.default_rng(20260303)
    cells = rng.integers(0, 1 << 21, size=(4096, 3), dtype=np.uint32)
    kat_cells = {"cells": cells,
                 "morton": np.array([r.morton(*map(int, c), 21) for c in cells], np.uint64),
                 "hilbert": np.array([r.hilbert(*map(int, c), 21) for c in cells], np.uint64)}
    with open(os.path.join(OUT, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)
    np.savez_compressed(os.path.join(OUT, "kat_cells.npz"), **kat_cells)

    for name, pts, curve, n_max, radius, shape, k in cases(o):
        level = 10 if "level10" in name else 21
        p = r.pipeline(pts, curve, n_max, level=level, threads=4)
        xs, codes, perm = p.coded()
        b, off, nodes = p.tree()
        rad = p.radius(radius, method=1, shape=shape, collect=True, threads=4)
        knn = p.knn(k, collect=True, threads=4)
        # RadiusMethod::Struct: batch digests (search.cpp:325-336) and, for the first centres,
        # the RangedResult rows themselves (neighbours_struct, search.cpp:122-135)
        st = p.radius(radius, method=3, shape=shape, threads=4)
        s_ro, s_rg, s_so, s_sg = [0], [], [0], []
        for i in range(min(64, len(xs))):
            _, rg, sg = p.radius_struct_point(xs[i], radius, shape)
            s_rg.append(rg.reshape(-1, 2))
            s_sg.append(sg)
            s_ro.append(s_ro[-1] + len(rg))
            s_so.append(s_so[-1] + len(sg))
        raw_codes = r.compute_codes(pts, curve) if level == 21 else np.zeros(0, np.uint64)
        np.savez_compressed(
            os.path.join(OUT, f"{name}.npz"), points=pts, curve=curve, level=level, n_max=n_max,
            radius=radius, shape=shape, k=k, disc_box=p.disc_box(), raw_codes=raw_codes,
            sorted_points=xs, codes=codes, perm=perm, boundaries=b, offsets=off,
            nodes=nodes.view(np.uint8).reshape(-1, 56), root=p.root, radius_offsets=rad["offsets"],
            radius_indices=rad["indices"], radius_counts=rad["counts"], radius_fps=rad["fps"],
            knn_idx=knn["idx"], knn_dist=knn["dist"], knn_fps=knn["fps"],
            struct_counts=st["counts"], struct_fps=st["fps"],
            struct_range_offsets=np.array(s_ro, np.uint64), struct_ranges=np.concatenate(s_rg).astype(np.uint32),
            struct_single_offsets=np.array(s_so, np.uint64), struct_singles=np.concatenate(s_sg).astype(np.uint32))
        print(f"{name}: n={len(pts)} leaves={p.leaves} internal={p.internal} "
              f"nbrs={int(rad['counts'].sum())}")


if __name__ == "__main__":
    main()
