"""Small end-to-end run for compute-sanitizer (racecheck / memcheck / synccheck): every kernel
family of the path on a 20k-point cloud -- reorder (bbox, encode, onesweep sort, gather), build,
radius (count + replay fill, Struct, explicit centres, forced FP64), kNN (filtered and FP64),
locality.  The tools replay every launch, so the cloud is small."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_06771_b200 import linoct as lo  # noqa: E402

pts = lo.generate_mixed(20000, 3)
for curve in (lo.Curve.Morton, lo.Curve.Hilbert):
    coded = lo.reorder_cloud(pts, curve)
    tree = lo.LinearOctree(coded, 32)
    for r in (0.5, 3.0):
        for m in (lo.RadiusMethod.Lin, lo.RadiusMethod.Struct):
            lo.run_radius_batch(tree, coded, m, lo.KernelShape.Sphere, r, lo.BatchOptions(collect_results=True))
    lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Cube, 2.0,
                        lo.BatchOptions(mode=lo.BatchMode.RandomSubset, subset_size=3000, seed=1, collect_results=True))
    for k in (8, 16, 40):
        lo.run_knn_batch(tree, coded, k, lo.BatchOptions(collect_results=True))
    os.environ["LO_FORCE_FP64"] = "1"
    lo.run_radius_batch(tree, coded, lo.RadiusMethod.Lin, lo.KernelShape.Sphere, 2.0, lo.BatchOptions())
    lo.run_knn_batch(tree, coded, 16, lo.BatchOptions())
    del os.environ["LO_FORCE_FP64"]
    lo.locality_histogram(tree, coded, 8, index_map=coded.permutation)
lo.default_context().synchronize()
print("sanitizer run ok")
