"""Full-size parity of the B200 path against the reference library (oracle/_ref) on every
BASELINE config (cfg0..cfg4).  Run on a GPU box:

    python tests/scale_parity.py [--configs cfg0 cfg1 ...] [--centres 20000] [--full cfg0 cfg1 ...] \
        > profiles/r1/scale_parity.txt

For each config the whole structure is compared bit for bit (sorted codes, permutation,
reordered coordinates, LeafArray, InternalNode table); radius counts and FNV-1a digests are
compared on `--centres` seeded random centres (RandomSubset, the reference's own sampler) and
kNN digests on a quarter of that.  cfg0 is compared on ALL centres.  At 100M points the
reference cannot hold every CSR row in memory, which is exactly why it digests them
(search.cpp:263-271).  The same comparisons run in the driver's GPU suite as
tests/test_gpu_scale.py (cfg1 / cfg4 / cfg3 in Full mode and a 250k-centre cfg3 RandomSubset).
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle.oracle_py import Ref  # noqa: E402
from paper_2603_06771_b200 import linoct as lo  # noqa: E402


def check(cfg_name: str, centres: int, full_cfgs=("cfg0",)) -> list[str]:
    cfg = bench.CONFIGS[cfg_name]
    out = []
    t0 = time.time()
    xyz = bench.generate(cfg)
    ref = Ref()
    p = ref.pipeline(xyz, cfg["curve"], cfg["n_max"])
    t_ref = time.time() - t0
    coded = lo.reorder_cloud(xyz, lo.Curve(cfg["curve"]))
    tree = lo.LinearOctree(coded, cfg["n_max"])
    xs, codes, perm = p.coded()
    ok = np.array_equal(coded.codes, codes) and np.array_equal(coded.permutation, perm)
    ok &= np.array_equal(coded.cloud.points.view(np.uint64), xs.view(np.uint64))
    out.append(f"{cfg_name}: n={cfg['n']} codes/perm/coords bit-exact: {ok}")
    del xs, codes, perm
    b, o, nodes = p.tree()
    la = tree.leaves()
    ok_t = np.array_equal(la.boundaries, b) and np.array_equal(la.offsets, o)
    ok_t &= tree.internal_nodes().tobytes() == nodes.tobytes() and tree.root() == p.root
    out.append(f"{cfg_name}: leaves={len(b) - 1} internal={len(nodes)} LeafArray + InternalNode table "
               f"bit-exact: {ok_t}")
    del b, o, nodes
    full = cfg_name in full_cfgs
    for r in cfg["radii"]:
        if full:
            want = p.radius(r, method=1)
            got = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, r,
                                      lo.BatchOptions())
        else:
            want = p.radius(r, method=1, mode=1, subset=centres, seed=1000 + int(10 * r))
            got = lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, r,
                                      lo.BatchOptions(mode=lo.BatchMode.RandomSubset, subset_size=centres,
                                                      seed=1000 + int(10 * r)))
        okr = (np.array_equal(got.centers, want["centers"]) and np.array_equal(got.counts, want["counts"])
               and np.array_equal(got.fingerprints, want["fps"]))
        out.append(f"{cfg_name}: radius r={r} on {len(got.centers)} centres: counts + FNV digests equal: "
                   f"{okr} (mu={got.counts.mean():.2f})")
    for k in cfg["ks"]:
        if full:
            want = p.knn(k)
            got = lo.run_knn_batch(tree, coded, k, lo.BatchOptions())
            m = len(got.centers)
        else:
            m = max(1000, centres // 4)
            want = p.knn(k, mode=1, subset=m, seed=77 + k)
            got = lo.run_knn_batch(tree, coded, k, lo.BatchOptions(mode=lo.BatchMode.RandomSubset,
                                                                   subset_size=m, seed=77 + k))
        okk = np.array_equal(got.centers, want["centers"]) and np.array_equal(got.fingerprints, want["fps"])
        out.append(f"{cfg_name}: kNN k={k} on {m} centres: (index, dist_sq) FNV digests equal: {okk}")
    out.append(f"{cfg_name}: reference build {t_ref:.1f}s, total {time.time() - t0:.1f}s")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="*", default=["cfg0", "cfg1", "cfg4", "cfg3"])
    ap.add_argument("--centres", type=int, default=20000)
    ap.add_argument("--full", nargs="*", default=["cfg0"],
                    help="configs compared on every point as a centre (Full mode) instead of a subset")
    a = ap.parse_args()
    allok = True
    for c in a.configs:
        for line in check(c, a.centres, tuple(a.full)):
            print(line, flush=True)
            allok &= ": False" not in line
    print("ALL EQUAL" if allok else "MISMATCH")
    return 0 if allok else 1


if __name__ == "__main__":
    sys.exit(main())
