"""ctypes bindings for the parity oracle (TEST INFRASTRUCTURE ONLY).

`Oracle` wraps oracle/liboracle.so (the plain-C restatement); `Ref` wraps
oracle/_ref/libref_linoct.so (the unmodified reference library compiled from
/root/reference/proj/src by oracle/Makefile).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_linoct.so")
REF_SRC = "/root/reference/proj"

P = C.c_void_p
u32, u64, i32, i64, f64 = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_double

NODE_DTYPE = np.dtype(
    [("prefix", "<u8"), ("children", "<i4", (8,)), ("begin", "<u4"), ("end", "<u4"),
     ("depth", "u1"), ("child_mask", "u1"), ("pad_", "u1", (6,))]
)
assert NODE_DTYPE.itemsize == 56


def _ptr(a):
    return None if a is None else a.ctypes.data_as(P)


def build(ref: bool = True) -> None:
    """Compile the restatement and, when the reference tree is present, oracle/_ref."""
    targets = ["all"]
    if ref and os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


class Oracle:
    """The C restatement (oracle/linoct_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.L = C.CDLL(path)
        L.or_gen_uniform.argtypes = [u64, u64, f64, P]
        L.or_gen_terrain.argtypes = [u64, u64, f64, P]
        L.or_gen_mixed.argtypes = [u64, u64, P]
        L.or_bbox.argtypes = [P, u64, P]
        L.or_bbox.restype = i64
        L.or_cubify.argtypes = [P, P]
        L.or_morton_encode.argtypes = [u32, u32, u32]
        L.or_morton_encode.restype = u64
        L.or_hilbert_encode.argtypes = [u32, u32, u32, C.c_int]
        L.or_hilbert_encode.restype = u64
        L.or_hilbert_decode.argtypes = [u64, C.c_int, P]
        L.or_stepper.argtypes = [C.c_int, P, P, C.c_int]
        L.or_octant_bounds.argtypes = [P, u32, u32, u32, C.c_int, P]
        L.or_compute_codes.argtypes = [P, u64, C.c_int, C.c_int, P, P, P]
        L.or_reorder.argtypes = [P, u64, C.c_int, C.c_int, P, P, P, P]
        L.or_build_leaves.argtypes = [P, u64, u32, C.c_int, P, P, u64]
        L.or_build_leaves.restype = i64
        L.or_link.argtypes = [P, P, u64, C.c_int, P, u64, P]
        L.or_link.restype = i64
        L.or_radius_brute.argtypes = [P, u64, P, f64, C.c_int, P]
        L.or_radius_brute.restype = u64
        L.or_knn_brute.argtypes = [P, u64, P, u32, P, P]
        L.or_knn_brute.restype = u32
        L.or_fnv_radius_row.argtypes = [P, u64]
        L.or_fnv_radius_row.restype = u64
        L.or_fnv_knn_row.argtypes = [P, P, u64]
        L.or_fnv_knn_row.restype = u64
        L.or_sample_indices.argtypes = [u32, u32, u64, P]
        L.or_radius_struct.argtypes = [P, P, P, P, C.c_int32, P, C.c_int, C.c_int, P, f64, C.c_int,
                                       P, u64, P, u64, P, P]
        L.or_radius_struct.restype = i64
        L.or_fnv_struct_row.argtypes = [P, u64, P, u64]
        L.or_fnv_struct_row.restype = u64

    # generators -------------------------------------------------------------------------
    def gen_uniform(self, n, seed, extent=100.0):
        a = np.empty((n, 3), np.float64)
        self.L.or_gen_uniform(n, seed, extent, _ptr(a))
        return a

    def gen_terrain(self, n, seed, extent_xy=1000.0):
        a = np.empty((n, 3), np.float64)
        self.L.or_gen_terrain(n, seed, extent_xy, _ptr(a))
        return a

    def gen_mixed(self, n, seed):
        a = np.empty((n, 3), np.float64)
        self.L.or_gen_mixed(n, seed, _ptr(a))
        return a

    def sample_indices(self, n, k, seed):
        out = np.empty(min(n, k), np.uint32)
        self.L.or_sample_indices(n, k, seed, _ptr(out))
        return out

    # sfc --------------------------------------------------------------------------------
    def morton(self, x, y, z):
        return self.L.or_morton_encode(x, y, z)

    def hilbert(self, x, y, z, level=21):
        return self.L.or_hilbert_encode(x, y, z, level)

    def hilbert_decode(self, code, level=21):
        out = np.zeros(3, np.uint32)
        self.L.or_hilbert_decode(code, level, _ptr(out))
        return tuple(int(v) for v in out)

    def stepper(self, curve):
        d = np.zeros((128, 8), np.uint8)
        nx = np.zeros((128, 8), np.uint8)
        s = self.L.or_stepper(curve, _ptr(d), _ptr(nx), 128)
        assert s > 0
        return d[:s].copy(), nx[:s].copy()

    def octant_bounds(self, box, hx, hy, hz, depth):
        b = np.ascontiguousarray(box, np.float64)
        out = np.zeros(6, np.float64)
        self.L.or_octant_bounds(_ptr(b), hx, hy, hz, depth, _ptr(out))
        return out

    def bbox(self, xyz):
        xyz = np.ascontiguousarray(xyz, np.float64)
        box = np.zeros(6)
        rc = self.L.or_bbox(_ptr(xyz), len(xyz), _ptr(box))
        return rc, box

    # reorder ----------------------------------------------------------------------------
    def compute_codes(self, xyz, curve, level=21):
        xyz = np.ascontiguousarray(xyz, np.float64)
        codes = np.empty(len(xyz), np.uint64)
        box = np.zeros(6)
        rc = self.L.or_compute_codes(_ptr(xyz), len(xyz), curve, level, _ptr(codes), _ptr(box), None)
        if rc != 0:
            raise ValueError("compute_codes failed")
        return codes, box

    def reorder(self, xyz, curve, level=21):
        xyz = np.ascontiguousarray(xyz, np.float64)
        n = len(xyz)
        xs = np.empty((n, 3), np.float64)
        codes = np.empty(n, np.uint64)
        perm = np.empty(n, np.uint32)
        box = np.zeros(6)
        rc = self.L.or_reorder(_ptr(xyz), n, curve, level, _ptr(xs), _ptr(codes), _ptr(perm), _ptr(box))
        if rc != 0:
            raise ValueError("reorder failed")
        return xs, codes, perm, box

    # octree -----------------------------------------------------------------------------
    def build_leaves(self, codes, n_max, level=21):
        codes = np.ascontiguousarray(codes, np.uint64)
        need = self.L.or_build_leaves(_ptr(codes), len(codes), n_max, level, None, None, 0)
        if need < 0:
            raise ValueError("build_leaves: invalid argument")
        b = np.empty(need + 1, np.uint64)
        o = np.empty(need + 1, np.uint32)
        self.L.or_build_leaves(_ptr(codes), len(codes), n_max, level, _ptr(b), _ptr(o), need + 1)
        return b, o

    def link(self, b, o, level=21):
        L = len(b) - 1
        nodes = np.zeros(L // 7 + 8, NODE_DTYPE)
        root = np.zeros(1, np.int32)
        cnt = self.L.or_link(_ptr(b), _ptr(o), L, level, _ptr(nodes), len(nodes), _ptr(root))
        if cnt < 0:
            raise ValueError("link: malformed leaves")
        return nodes[:cnt].copy(), int(root[0])

    # search -----------------------------------------------------------------------------
    def radius_brute(self, xyz, c, r, shape=0):
        xyz = np.ascontiguousarray(xyz, np.float64)
        c = np.ascontiguousarray(c, np.float64)
        cnt = self.L.or_radius_brute(_ptr(xyz), len(xyz), _ptr(c), r, shape, None)
        out = np.empty(cnt, np.uint32)
        self.L.or_radius_brute(_ptr(xyz), len(xyz), _ptr(c), r, shape, _ptr(out))
        return out

    def knn_brute(self, xyz, c, k):
        xyz = np.ascontiguousarray(xyz, np.float64)
        c = np.ascontiguousarray(c, np.float64)
        take = min(k, len(xyz))
        idx = np.empty(take, np.uint32)
        dist = np.empty(take, np.float64)
        self.L.or_knn_brute(_ptr(xyz), len(xyz), _ptr(c), k, _ptr(idx), _ptr(dist))
        return idx, dist

    def radius_struct(self, xs, b, o, nodes, root, disc_box, curve, c, r, shape=0, level=21):
        """neighbours_struct restated over the oracle's own tree arrays (sorted cloud xs):
        (count, ranges (k, 2) u32, singles u32)."""
        xs = np.ascontiguousarray(xs, np.float64)
        c = np.ascontiguousarray(c, np.float64)
        box = np.ascontiguousarray(disc_box, np.float64)
        cap_r, cap_s = max(1, len(xs)), max(1, len(xs))
        ranges = np.empty((cap_r, 2), np.uint32)
        singles = np.empty(cap_s, np.uint32)
        nr = np.zeros(1, np.uint64)
        ns = np.zeros(1, np.uint64)
        nodes = np.ascontiguousarray(nodes) if len(nodes) else np.zeros(1, NODE_DTYPE)
        cnt = self.L.or_radius_struct(_ptr(xs), _ptr(b), _ptr(o), _ptr(nodes), root, _ptr(box), level,
                                      curve, _ptr(c), r, shape, _ptr(ranges), cap_r, _ptr(singles),
                                      cap_s, _ptr(nr), _ptr(ns))
        if cnt < 0:
            raise ValueError("radius_struct: capacity exceeded")
        return int(cnt), ranges[: int(nr[0])].copy(), singles[: int(ns[0])].copy()

    def fnv_struct(self, ranges, singles):
        ranges = np.ascontiguousarray(ranges, np.uint32)
        singles = np.ascontiguousarray(singles, np.uint32)
        return self.L.or_fnv_struct_row(_ptr(ranges), len(ranges), _ptr(singles), len(singles))

    def fnv_radius(self, idx):
        idx = np.ascontiguousarray(idx, np.uint32)
        return self.L.or_fnv_radius_row(_ptr(idx), len(idx))

    def fnv_knn(self, idx, dist):
        idx = np.ascontiguousarray(idx, np.uint32)
        dist = np.ascontiguousarray(dist, np.float64)
        return self.L.or_fnv_knn_row(_ptr(idx), _ptr(dist), len(idx))


class RefPipeline:
    """reorder_cloud + LinearOctree held by the reference library (oracle/_ref)."""

    def __init__(self, ref: "Ref", xyz, curve, n_max, level=21, threads=None):
        self.ref = ref
        L = ref.L
        xyz = np.ascontiguousarray(xyz, np.float64)
        self.threads = threads or L.ref_max_threads()
        h = P()
        self.timings = np.zeros(2)
        rc = L.ref_pipeline_create(_ptr(xyz), len(xyz), curve, level, n_max, self.threads,
                                   C.byref(h), _ptr(self.timings))
        if rc != 0:
            raise ValueError(L.ref_last_error().decode())
        self.h = h
        s = np.zeros(4, np.int64)
        L.ref_pipeline_sizes(h, _ptr(s))
        self.n, self.leaves, self.internal, self.root = (int(v) for v in s)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.ref.L.ref_pipeline_destroy(h)
            self.h = None

    def disc_box(self):
        b = np.zeros(6)
        self.ref.L.ref_pipeline_disc(self.h, _ptr(b))
        return b

    def coded(self):
        xyz = np.empty((self.n, 3))
        codes = np.empty(self.n, np.uint64)
        perm = np.empty(self.n, np.uint32)
        self.ref.L.ref_pipeline_coded(self.h, _ptr(xyz), _ptr(codes), _ptr(perm))
        return xyz, codes, perm

    def tree(self):
        b = np.empty(self.leaves + 1, np.uint64)
        o = np.empty(self.leaves + 1, np.uint32)
        nodes = np.zeros(self.internal, NODE_DTYPE)
        self.ref.L.ref_pipeline_tree(self.h, _ptr(b), _ptr(o), _ptr(nodes))
        return b, o, nodes

    def rebuild(self, n_max, threads=None):
        return self.ref.L.ref_pipeline_rebuild(self.h, n_max, threads or self.threads)

    def radius(self, r, method=1, shape=0, mode=0, subset=0, seed=0, threads=None,
               fingerprint=True, collect=False):
        L = self.ref.L
        th = threads or self.threads
        m = self.n if mode == 0 else subset
        centers = np.empty(m, np.uint32)
        counts = np.empty(m, np.uint32)
        fps = np.zeros(m, np.uint64)
        mean = np.zeros(1)
        if not collect:
            wall = L.ref_radius(self.h, method, shape, r, mode, subset, seed, th, int(fingerprint),
                                _ptr(centers), _ptr(counts), _ptr(fps), None, None, _ptr(mean))
            if wall < 0:
                raise ValueError(L.ref_last_error().decode())
            return dict(centers=centers, counts=counts, fps=fps, wall=wall, mean=float(mean[0]))
        wall = L.ref_radius(self.h, method, shape, r, mode, subset, seed, th, int(fingerprint),
                            _ptr(centers), _ptr(counts), _ptr(fps), None, None, _ptr(mean))
        if wall < 0:
            raise ValueError(L.ref_last_error().decode())
        offs = np.empty(m + 1, np.uint64)
        idx = np.empty(int(counts.astype(np.uint64).sum()), np.uint32)
        wall = L.ref_radius(self.h, method, shape, r, mode, subset, seed, th, int(fingerprint),
                            _ptr(centers), _ptr(counts), _ptr(fps), _ptr(offs), _ptr(idx), _ptr(mean))
        return dict(centers=centers, counts=counts, fps=fps, wall=wall, mean=float(mean[0]),
                    offsets=offs, indices=idx)

    def knn(self, k, mode=0, subset=0, seed=0, threads=None, fingerprint=True, collect=False):
        L = self.ref.L
        th = threads or self.threads
        m = self.n if mode == 0 else subset
        centers = np.empty(m, np.uint32)
        counts = np.empty(m, np.uint32)
        fps = np.zeros(m, np.uint64)
        kk = min(k, self.n)
        idx = np.empty((m, kk), np.uint32) if collect else None
        dist = np.empty((m, kk), np.float64) if collect else None
        wall = L.ref_knn(self.h, k, mode, subset, seed, th, int(fingerprint), _ptr(centers),
                         _ptr(counts), _ptr(fps), _ptr(idx), _ptr(dist))
        if wall < 0:
            raise ValueError(L.ref_last_error().decode())
        return dict(centers=centers, counts=counts, fps=fps, wall=wall, idx=idx, dist=dist)

    def knn_point(self, c, k):
        c = np.ascontiguousarray(c, np.float64)
        kk = min(k, self.n)
        idx = np.empty(kk, np.uint32)
        dist = np.empty(kk, np.float64)
        cnt = np.zeros(1, np.uint32)
        rc = self.ref.L.ref_knn_point(self.h, _ptr(c), k, _ptr(idx), _ptr(dist), _ptr(cnt))
        if rc != 0:
            raise ValueError(self.ref.L.ref_last_error().decode())
        return idx[: cnt[0]], dist[: cnt[0]]

    def radius_point(self, c, r, shape=0):
        c = np.ascontiguousarray(c, np.float64)
        cnt = self.ref.L.ref_radius_point(self.h, shape, _ptr(c), r, None, 0)
        if cnt < 0:
            raise ValueError(self.ref.L.ref_last_error().decode())
        out = np.empty(cnt, np.uint32)
        self.ref.L.ref_radius_point(self.h, shape, _ptr(c), r, _ptr(out), cnt)
        return out

    def save_tree(self, path):
        """LinearOctree::serialize of this pipeline's tree to a LOC1 file."""
        if self.ref.L.ref_pipeline_save_tree(self.h, os.fsencode(path)) != 0:
            raise RuntimeError(self.ref.L.ref_last_error().decode())

    def radius_struct_point(self, c, r, shape=0):
        """neighbours_struct at centre c: (count, ranges (k, 2) u32, singles u32)."""
        c = np.ascontiguousarray(c, np.float64)
        nr = np.zeros(1, np.uint64)
        ns = np.zeros(1, np.uint64)
        L = self.ref.L
        cnt = L.ref_radius_struct_point(self.h, shape, _ptr(c), r, None, 0, None, 0, _ptr(nr), _ptr(ns))
        if cnt < 0:
            raise ValueError(L.ref_last_error().decode())
        ranges = np.empty((int(nr[0]), 2), np.uint32)
        singles = np.empty(int(ns[0]), np.uint32)
        L.ref_radius_struct_point(self.h, shape, _ptr(c), r, _ptr(ranges), len(ranges), _ptr(singles),
                                  len(singles), _ptr(nr), _ptr(ns))
        return int(cnt), ranges, singles

    def radius_range(self, r, begin, end, shape=0, method=1, threads=None, digests=True):
        """neighbours_lin over the sorted centres [begin, end); returns (wall s, counts, fps)."""
        m = end - begin
        counts = np.empty(m, np.uint32)
        fps = np.empty(m, np.uint64) if digests else None
        wall = self.ref.L.ref_radius_range(self.h, method, shape, r, begin, end,
                                           threads or self.threads, _ptr(counts), _ptr(fps))
        return wall, counts, fps

    def radius_centres(self, r, centres, shape=0, method=1, threads=None):
        """run_batch_loop's radius query over an explicit centre list; (wall s, counts, fps)."""
        centres = np.ascontiguousarray(centres, np.uint32)
        counts = np.empty(len(centres), np.uint32)
        fps = np.empty(len(centres), np.uint64)
        wall = self.ref.L.ref_radius_centres(self.h, method, shape, r, _ptr(centres), len(centres),
                                             threads or self.threads, _ptr(counts), _ptr(fps))
        return wall, counts, fps

    def knn_centres(self, k, centres, threads=None):
        centres = np.ascontiguousarray(centres, np.uint32)
        fps = np.empty(len(centres), np.uint64)
        wall = self.ref.L.ref_knn_centres(self.h, k, _ptr(centres), len(centres),
                                          threads or self.threads, _ptr(fps))
        return wall, fps

    def knn_range(self, k, begin, end, threads=None, digests=True):
        fps = np.empty(end - begin, np.uint64) if digests else None
        wall = self.ref.L.ref_knn_range(self.h, k, begin, end, threads or self.threads, _ptr(fps))
        return wall, fps

    def locality(self, k, use_perm_map=False, threads=None):
        L = self.ref.L
        th = threads or self.threads
        cap = 1 << 22
        d = np.empty(cap, np.uint32)
        c = np.empty(cap, np.uint64)
        nb = L.ref_locality(self.h, k, th, int(use_perm_map), _ptr(d), _ptr(c), cap)
        if nb < 0:
            raise ValueError(L.ref_last_error().decode())
        return d[:nb].copy(), c[:nb].copy()

    def locality_stats(self, k, use_perm_map=False, sample=0, seed=0, threads=None):
        """(bins d, bins count, [mean, stddev, G1, Q1, Q2, Q3]) of locality_histogram(_approx)."""
        L = self.ref.L
        th = threads or self.threads
        out = np.zeros(6)
        nb = L.ref_locality_stats(self.h, k, th, int(use_perm_map), sample, seed, _ptr(out), None, None, 0)
        if nb < 0:
            raise ValueError(L.ref_last_error().decode())
        d = np.empty(nb, np.uint32)
        c = np.empty(nb, np.uint64)
        L.ref_locality_stats(self.h, k, th, int(use_perm_map), sample, seed, _ptr(out), _ptr(d), _ptr(c), nb)
        return d, c, out


class Ref:
    """The unmodified reference library (oracle/_ref/libref_linoct.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    f"{REF_SRC} exists")
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_max_threads.restype = C.c_int
        L.ref_morton_encode.argtypes = [u32, u32, u32, C.c_int]
        L.ref_morton_encode.restype = u64
        L.ref_hilbert_encode.argtypes = [u32, u32, u32, C.c_int]
        L.ref_hilbert_encode.restype = u64
        L.ref_hilbert_decode.argtypes = [u64, C.c_int, P]
        L.ref_octant_bounds.argtypes = [P, u32, u32, u32, C.c_int, C.c_int, P]
        L.ref_gen_uniform.argtypes = [u64, u64, f64, P]
        L.ref_sample_indices.argtypes = [u32, u32, u64, P]
        L.ref_compute_codes.argtypes = [P, u64, C.c_int, P]
        L.ref_pipeline_create.argtypes = [P, u64, C.c_int, C.c_int, u32, C.c_int, P, P]
        L.ref_pipeline_destroy.argtypes = [P]
        L.ref_pipeline_rebuild.argtypes = [P, u32, C.c_int]
        L.ref_pipeline_rebuild.restype = f64
        L.ref_pipeline_sizes.argtypes = [P, P]
        L.ref_pipeline_disc.argtypes = [P, P]
        L.ref_pipeline_coded.argtypes = [P, P, P, P]
        L.ref_pipeline_tree.argtypes = [P, P, P, P]
        L.ref_build_leaves.argtypes = [P, u64, u32, C.c_int, P, P, u64, P]
        L.ref_locality_stats.argtypes = [P, u32, C.c_int, C.c_int, u32, u64, P, P, P, u64]
        L.ref_locality_stats.restype = i64
        L.ref_read_cloud.argtypes = [C.c_char_p, P, u64]
        L.ref_read_cloud.restype = i64
        L.ref_write_cloud.argtypes = [P, u64, C.c_char_p]
        L.ref_pipeline_save_tree.argtypes = [P, C.c_char_p]
        L.ref_link_tree.argtypes = [C.c_char_p, P, P, u64, P, C.c_int, C.c_int, u32, P, P, u64, P, u64,
                                    P, P, P]
        L.ref_radius.argtypes = [P, C.c_int, C.c_int, f64, C.c_int, u32, u64, C.c_int, C.c_int,
                                 P, P, P, P, P, P]
        L.ref_radius.restype = f64
        L.ref_knn.argtypes = [P, u32, C.c_int, u32, u64, C.c_int, C.c_int, P, P, P, P, P]
        L.ref_knn.restype = f64
        L.ref_knn_point.argtypes = [P, P, u32, P, P, P]
        L.ref_radius_point.argtypes = [P, C.c_int, P, f64, P, u64]
        L.ref_radius_point.restype = i64
        L.ref_radius_struct_point.argtypes = [P, C.c_int, P, f64, P, u64, P, u64, P, P]
        L.ref_radius_struct_point.restype = i64
        L.ref_locality.argtypes = [P, u32, C.c_int, C.c_int, P, P, u64]
        L.ref_locality.restype = i64
        L.ref_radius_range.argtypes = [P, C.c_int, C.c_int, f64, u64, u64, C.c_int, P, P]
        L.ref_radius_range.restype = f64
        L.ref_knn_range.argtypes = [P, u32, u64, u64, C.c_int, P]
        L.ref_knn_range.restype = f64
        L.ref_radius_centres.argtypes = [P, C.c_int, C.c_int, f64, P, u64, C.c_int, P, P]
        L.ref_radius_centres.restype = f64
        L.ref_knn_centres.argtypes = [P, u32, P, u64, C.c_int, P]
        L.ref_knn_centres.restype = f64

    def max_threads(self):
        return self.L.ref_max_threads()

    def hilbert(self, x, y, z, level=21):
        return self.L.ref_hilbert_encode(x, y, z, level)

    def morton(self, x, y, z, level=21):
        return self.L.ref_morton_encode(x, y, z, level)

    def hilbert_decode(self, code, level=21):
        out = np.zeros(3, np.uint32)
        self.L.ref_hilbert_decode(code, level, _ptr(out))
        return tuple(int(v) for v in out)

    def octant_bounds(self, box, hx, hy, hz, depth, level=21):
        b = np.ascontiguousarray(box, np.float64)
        out = np.zeros(6)
        if self.L.ref_octant_bounds(_ptr(b), hx, hy, hz, depth, level, _ptr(out)) != 0:
            raise ValueError(self.L.ref_last_error().decode())
        return out

    def gen_uniform(self, n, seed, extent=100.0):
        a = np.empty((n, 3))
        self.L.ref_gen_uniform(n, seed, extent, _ptr(a))
        return a

    def sample_indices(self, n, k, seed):
        out = np.empty(min(n, k), np.uint32)
        self.L.ref_sample_indices(n, k, seed, _ptr(out))
        return out

    def compute_codes(self, xyz, curve):
        xyz = np.ascontiguousarray(xyz, np.float64)
        codes = np.empty(len(xyz), np.uint64)
        if self.L.ref_compute_codes(_ptr(xyz), len(xyz), curve, _ptr(codes)) != 0:
            raise ValueError(self.L.ref_last_error().decode())
        return codes

    def build_leaves(self, codes, n_max, level=21):
        codes = np.ascontiguousarray(codes, np.uint64)
        nl = np.zeros(1, np.uint64)
        rc = self.L.ref_build_leaves(_ptr(codes), len(codes), n_max, level, None, None, 0, _ptr(nl))
        if rc != 0:
            raise ValueError(self.L.ref_last_error().decode())
        L = int(nl[0])
        b = np.empty(L + 1, np.uint64)
        o = np.empty(L + 1, np.uint32)
        self.L.ref_build_leaves(_ptr(codes), len(codes), n_max, level, _ptr(b), _ptr(o), L + 1, _ptr(nl))
        return b, o

    def read_cloud(self, path):
        """read_cloud(path) (io.cpp:83-89): (n, 3) f64, or raises with the reference's text."""
        L = self.L
        n = L.ref_read_cloud(os.fsencode(path), None, 0)
        if n < 0:
            raise RuntimeError(L.ref_last_error().decode())
        out = np.empty((n, 3), np.float64)
        L.ref_read_cloud(os.fsencode(path), _ptr(out), n)
        return out

    def write_cloud(self, xyz, path):
        xyz = np.ascontiguousarray(xyz, np.float64)
        if self.L.ref_write_cloud(_ptr(xyz), len(xyz), os.fsencode(path)) != 0:
            raise RuntimeError(self.L.ref_last_error().decode())

    def link_tree(self, path=None, b=None, o=None, box=None, level=21, curve=0, n_max=32):
        """LinearOctree::deserialize(path), or LinearOctree(LeafArray(b, o), Discretizer(box,
        level), curve, n_max): (boundaries, offsets, nodes, root).  Errors raise ValueError
        (invalid_argument) or RuntimeError with the reference's text."""
        L = self.L
        leaves, internal, root = np.zeros(1, np.uint64), np.zeros(1, np.uint64), np.zeros(1, np.int32)
        bb = None if b is None else np.ascontiguousarray(b, np.uint64)
        oo = None if o is None else np.ascontiguousarray(o, np.uint32)
        box = None if box is None else np.ascontiguousarray(box, np.float64)
        cnt = 0 if bb is None else len(bb)
        pth = None if path is None else os.fsencode(path)
        args = (pth, _ptr(bb), _ptr(oo), cnt, _ptr(box), level, curve, n_max)
        rc = L.ref_link_tree(*args, None, None, 0, None, 0, _ptr(leaves), _ptr(internal), _ptr(root))
        if rc != 0:
            msg = L.ref_last_error().decode()
            raise (ValueError if rc == 1 else RuntimeError)(msg)
        nl, ni = int(leaves[0]), int(internal[0])
        b_out = np.empty(nl + 1, np.uint64)
        o_out = np.empty(nl + 1, np.uint32)
        nodes = np.zeros(ni, NODE_DTYPE)
        L.ref_link_tree(*args, _ptr(b_out), _ptr(o_out), nl + 1, _ptr(nodes), ni, _ptr(leaves), _ptr(internal),
                        _ptr(root))
        return b_out, o_out, nodes, int(root[0])

    def pipeline(self, xyz, curve, n_max, level=21, threads=None):
        return RefPipeline(self, xyz, curve, n_max, level, threads)
