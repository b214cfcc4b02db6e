"""Reference-shaped host API over the C ABI (names, argument meaning and errors of
proj/include/linoct/{sfc,reorder,linear_octree,search}.hpp).

    cloud = PointCloud(xyz)                                   # geometry.hpp:60-99
    coded = reorder_cloud(cloud, Curve.Hilbert)                # reorder.hpp:33
    tree = LinearOctree(coded, n_max=32)                       # linear_octree.hpp:55
    res = run_radius_batch(tree, coded, RadiusMethod.Lin, KernelShape.Sphere, 2.5,
                           BatchOptions())                     # search.hpp:135-137
    knn = run_knn_batch(tree, coded, 16, BatchOptions())       # search.hpp:145-146

Everything runs on the B200 through liblinoct_b200.so; there is no CPU path.  Exceptions
mirror the reference's: InvalidArgument (std::invalid_argument), DomainError
(std::domain_error), LogicError (std::logic_error).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import re
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import (CodedInfo, CsrInfo, DomainError, FileFormatError, InvalidArgument, LogicError, OctreeInfo,
                   check)

__all__ = [
    "Curve", "KernelShape", "RadiusMethod", "BatchMode", "BatchOptions", "BatchResult",
    "PointCloud", "CodedCloud", "LinearOctree", "LeafArray", "SearchKernel", "KnnNeighbor",
    "Context", "default_context", "compute_codes", "reorder_cloud", "build_leaves",
    "invert_permutation", "run_radius_batch", "run_knn_batch", "neighbours_lin",
    "neighbours_prune", "knn_lin_oct", "sample_indices", "generate_uniform",
    "generate_terrain", "generate_mixed", "morton_encode", "hilbert_encode", "sfc_encode",
    "sfc_decode", "InvalidArgument", "DomainError", "LogicError", "kMaxLevel", "INTERNAL_NODE_DTYPE",
]

kMaxLevel = 21


class Curve(enum.IntEnum):  # sfc.hpp:17
    Morton = 0
    Hilbert = 1


class KernelShape(enum.IntEnum):  # geometry.hpp:101
    Sphere = 0
    Circle = 1
    Cube = 2
    Square = 3


class RadiusMethod(enum.IntEnum):  # search.hpp:108
    Ptr = 0
    Lin = 1
    Prune = 2
    Struct = 3


class BatchMode(enum.IntEnum):  # search.hpp:107
    Full = 0
    RandomSubset = 1


# LinearOctree::InternalNode (linear_octree.hpp:46-53), 56 bytes
INTERNAL_NODE_DTYPE = np.dtype(
    [("prefix", "<u8"), ("children", "<i4", (8,)), ("begin", "<u4"), ("end", "<u4"),
     ("depth", "u1"), ("child_mask", "u1"), ("pad_", "u1", (6,))])
assert INTERNAL_NODE_DTYPE.itemsize == 56


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


class Context:
    """One device + one stream (lo_context)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        L = _lib.lib()
        h = C.c_void_p()
        check(L.lo_context_create(device, C.c_void_p(stream) if stream else None, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        """Destroys the context; a no-op while handles created on it are still alive (the C ABI
        refuses with LO_LOGIC_ERROR), retried when this object is collected."""
        if getattr(self, "h", None):
            if _lib.lib().lo_context_destroy(self.h) == _lib.OK:
                self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        check(_lib.lib().lo_context_synchronize(self.h))

    @property
    def stream(self) -> int:
        return _lib.lib().lo_context_stream(self.h) or 0

    def set_timing(self, on: bool):
        check(_lib.lib().lo_context_set_timing(self.h, int(on)))

    def stage_times(self) -> list[tuple[str, float]]:
        cap, nl = 256, 32
        names = C.create_string_buffer(cap * nl)
        ms = np.zeros(cap)
        n = _lib.lib().lo_context_stage_times(self.h, names, nl, _p(ms), cap)
        if n < 0:
            check(-n)
        raw = names.raw
        return [(raw[i * nl:(i + 1) * nl].split(b"\0", 1)[0].decode(), float(ms[i])) for i in range(n)]


_default: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


@dataclass(frozen=True)
class SearchKernel:
    """geometry.hpp:104-125: shape, centre, radius; radius_sq computed once."""
    shape: KernelShape
    center: tuple
    radius: float

    def __post_init__(self):
        r = float(self.radius)
        if not (r > 0.0) or not np.isfinite(r):
            raise InvalidArgument("kernel radius must be positive and finite")
        if not np.all(np.isfinite(np.asarray(self.center, float))):
            raise InvalidArgument("kernel center must be finite")


class PointCloud:
    """Host AoS f64 points (geometry.hpp:60-99): finite check, cached bbox."""

    def __init__(self, points=None):
        a = np.zeros((0, 3)) if points is None else np.ascontiguousarray(points, dtype=np.float64)
        if a.ndim != 2 or a.shape[1] != 3:
            raise InvalidArgument("points must be an (n, 3) array")
        bad = ~np.isfinite(a).all(axis=1)
        if bad.any():
            raise InvalidArgument(f"non-finite coordinate at point {int(np.argmax(bad))}")
        self.points = a

    def size(self) -> int:
        return len(self.points)

    def __len__(self):
        return len(self.points)

    def empty(self) -> bool:
        return len(self.points) == 0

    def __getitem__(self, i):
        return self.points[i]

    def bbox(self):
        if self.empty():
            raise LogicError("bbox of empty cloud")
        return np.concatenate([self.points.min(axis=0), self.points.max(axis=0)])


def _as_points(cloud) -> np.ndarray:
    return cloud.points if isinstance(cloud, PointCloud) else np.ascontiguousarray(cloud, np.float64)


class CodedCloud:
    """reorder.hpp:14-20.  Device resident; host views are downloaded lazily."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx
        info = CodedInfo()
        check(_lib.lib().lo_coded_info_get(self.h, C.byref(info)))
        self.n = int(info.n)
        self.curve = Curve(info.curve)
        self.level = int(info.level)
        self.disc_box = np.array(info.disc_box[:])
        self.cloud_box = np.array(info.cloud_box[:])
        self.scale = np.array(info.scale[:])
        self._cloud = self._codes = self._perm = None

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _lib.lib().lo_coded_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def write_pcb(self, path: str) -> None:
        """write_cloud(coded.cloud, path, BinaryPcb): the reordered cloud as PCB1."""
        check(_lib.lib().lo_coded_write_pcb(self.ctx.h, self.h, os.fsencode(path)))

    def _download(self, xyz=False, codes=False, perm=False):
        a = np.empty((self.n, 3)) if xyz else None
        c = np.empty(self.n, np.uint64) if codes else None
        p = np.empty(self.n, np.uint32) if perm else None
        check(_lib.lib().lo_coded_download(self.ctx.h, self.h, _p(a), _p(c), _p(p)))
        return a, c, p

    @property
    def cloud(self) -> PointCloud:
        if self._cloud is None:
            self._cloud = PointCloud(self._download(xyz=True)[0])
        return self._cloud

    @property
    def codes(self) -> np.ndarray:
        if self._codes is None:
            self._codes = self._download(codes=True)[1]
        return self._codes

    @property
    def permutation(self) -> np.ndarray:
        if self._perm is None:
            self._perm = self._download(perm=True)[2]
        return self._perm

    @property
    def discretizer(self):
        return {"bbox": self.disc_box.copy(), "level": self.level, "scale": self.scale.copy()}


class CloudFormat(enum.IntEnum):  # io.hpp:14
    TextXyz = 0
    BinaryPcb = 1


def format_from_path(path: str) -> CloudFormat:
    """io.cpp:16-23."""
    dot = path.rfind(".")
    ext = "" if dot < 0 else path[dot:]
    if ext == ".pcb":
        return CloudFormat.BinaryPcb
    if ext in (".xyz", ".txt"):
        return CloudFormat.TextXyz
    raise InvalidArgument(f"cannot infer cloud format from '{path}' (expected .pcb, .xyz or .txt)")


_DECIMAL = re.compile(r"^[+-]?(\d+\.?\d*|\.\d+)([eE][+-]?\d+)?$")


def read_cloud(path: str, fmt: CloudFormat | None = None) -> PointCloud:
    """read_cloud (io.cpp:27-85) on the host: PCB1 or text XYZ, the reference's error texts."""
    fmt = format_from_path(path) if fmt is None else fmt
    if fmt == CloudFormat.TextXyz:
        try:
            lines = open(path).read().split("\n")
        except OSError:
            raise FileFormatError(f"cannot open '{path}'") from None
        pts = []
        for no, line in enumerate(lines, 1):
            t = line.strip(" \t\r")
            if not t or t.startswith("#"):
                continue
            f = t.split()
            # what `std::istream >> double` accepts: decimal reals only (no inf/nan/hex), and an
            # out-of-range value is a failed extraction
            if len(f) != 3 or not all(_DECIMAL.match(x) for x in f):
                raise FileFormatError(f"{path}:{no}: expected three reals")
            p = [float(x) for x in f]
            if not all(np.isfinite(p)):
                raise FileFormatError(f"{path}:{no}: expected three reals")
            if not all(np.isfinite(p)):
                raise FileFormatError(f"{path}:{no}: non-finite coordinate")
            pts.append(p)
        return PointCloud(np.array(pts, np.float64).reshape(-1, 3))
    try:
        raw = open(path, "rb").read()
    except OSError:
        raise FileFormatError(f"cannot open '{path}'") from None
    if raw[:4] != b"PCB1":
        raise FileFormatError(f"{path}: bad magic at byte offset 0")
    if len(raw) < 12:
        raise FileFormatError(f"{path}: truncated count at byte offset 4")
    count = int(np.frombuffer(raw, "<u8", 1, 4)[0])
    have = (len(raw) - 12) // 24
    if have < count:
        raise FileFormatError(f"{path}: truncated record at byte offset {12 + 24 * have}")
    a = np.frombuffer(raw, "<f8", 3 * count, 12).reshape(count, 3).astype(np.float64)
    bad = ~np.isfinite(a).all(axis=1)
    if bad.any():
        raise FileFormatError(f"{path}: non-finite coordinate in record {int(np.argmax(bad))}")
    return PointCloud(a)


def write_cloud(cloud, path: str, fmt: CloudFormat | None = None) -> None:
    """write_cloud (io.cpp:94-120): PCB1 little-endian, or '%.17g %.17g %.17g' lines."""
    fmt = format_from_path(path) if fmt is None else fmt
    pts = _as_points(cloud)
    try:
        with open(path, "wb") as f:
            if fmt == CloudFormat.BinaryPcb:
                f.write(b"PCB1" + np.uint64(len(pts)).astype("<u8").tobytes())
                f.write(np.ascontiguousarray(pts, "<f8").tobytes())
            else:
                f.write("".join("%.17g %.17g %.17g\n" % tuple(p) for p in pts).encode())
    except OSError:
        raise FileFormatError(f"cannot open '{path}' for writing") from None


def reorder_pcb(path: str, curve: Curve, level: int = kMaxLevel, ctx: Context | None = None) -> CodedCloud:
    """reorder_cloud(read_cloud(path), curve, level) for a PCB1 file, streamed from disk to the
    device through pinned double buffers (disk reads overlap the H2D copies)."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    check(_lib.lib().lo_reorder_pcb(ctx.h, os.fsencode(path), int(curve), level, C.byref(h)))
    return CodedCloud(h, ctx)


def compute_codes(cloud, curve: Curve, disc_box=None, level: int = kMaxLevel,
                  ctx: Context | None = None) -> np.ndarray:
    """reorder.hpp:23-28: per-point codes in cloud order (cubified bbox by default)."""
    pts = _as_points(cloud)
    if len(pts) == 0:
        raise InvalidArgument("compute_codes: empty cloud")
    ctx = ctx or default_context()
    out = np.empty(len(pts), np.uint64)
    box = None if disc_box is None else np.ascontiguousarray(disc_box, np.float64)
    check(_lib.lib().lo_compute_codes(ctx.h, _p(pts), len(pts), int(curve), level, _p(box), _p(out)))
    return out


def reorder_cloud(cloud, curve: Curve, level: int = kMaxLevel, ctx: Context | None = None) -> CodedCloud:
    """reorder.hpp:33: stable SFC sort, gather, permutation[new] = old."""
    pts = _as_points(cloud)
    ctx = ctx or default_context()
    h = C.c_void_p()
    check(_lib.lib().lo_reorder(ctx.h, _p(pts) if len(pts) else None, len(pts), int(curve), level, C.byref(h)))
    return CodedCloud(h, ctx)


def invert_permutation(perm, ctx: Context | None = None) -> np.ndarray:
    """reorder.hpp:36"""
    perm = np.ascontiguousarray(perm, np.uint32)
    ctx = ctx or default_context()
    out = np.empty_like(perm)
    check(_lib.lib().lo_invert_permutation(ctx.h, _p(perm), len(perm), _p(out)))
    return out


@dataclass
class LeafArray:
    """linear_octree.hpp:20-27"""
    boundaries: np.ndarray
    offsets: np.ndarray

    def leaf_count(self) -> int:
        return len(self.boundaries) - 1


def build_leaves(codes, n_max: int, level: int = kMaxLevel, threads: int = 1,
                 ctx: Context | None = None) -> LeafArray:
    """linear_octree.hpp:33-34 (threads accepted and ignored)."""
    codes = np.ascontiguousarray(codes, np.uint64)
    if n_max < 1:
        raise InvalidArgument("build_leaves: n_max must be >= 1")
    if len(codes) == 0:
        raise InvalidArgument("build_leaves: empty code array")
    ctx = ctx or default_context()
    L = C.c_uint64()
    check(_lib.lib().lo_build_leaves(ctx.h, _p(codes), len(codes), n_max, level, C.byref(L), None, None, 0))
    b = np.empty(L.value + 1, np.uint64)
    o = np.empty(L.value + 1, np.uint32)
    check(_lib.lib().lo_build_leaves(ctx.h, _p(codes), len(codes), n_max, level, C.byref(L), _p(b), _p(o), len(b)))
    return LeafArray(b, o)


class LinearOctree:
    """linear_octree.hpp:40-118, built on the device from a CodedCloud."""

    def __init__(self, coded: CodedCloud, n_max: int = 128, threads: int = 1, _handle=None):
        self.coded = coded
        self.ctx = coded.ctx
        if _handle is None:
            if n_max < 1:
                raise InvalidArgument("build_leaves: n_max must be >= 1")
            h = C.c_void_p()
            check(_lib.lib().lo_octree_build(self.ctx.h, coded.h, n_max, C.byref(h)))
            _handle = h
        self.h = _handle
        info = OctreeInfo()
        check(_lib.lib().lo_octree_info_get(self.h, C.byref(info)))
        self.info = info
        self._leaves = self._nodes = None

    @classmethod
    def from_leaves(cls, coded: CodedCloud, leaf_array: "LeafArray", disc_box, level: int, curve: Curve,
                    n_max: int) -> "LinearOctree":
        """LinearOctree(LeafArray, Discretizer(disc_box, level), curve, n_max)
        (linear_octree.cpp:84-105): validated like the reference, linked on the device."""
        b = np.ascontiguousarray(leaf_array.boundaries, np.uint64)
        o = np.ascontiguousarray(leaf_array.offsets, np.uint32)
        if len(b) != len(o):
            raise InvalidArgument("linear octree: malformed leaf array")
        box = np.ascontiguousarray(disc_box, np.float64)
        h = C.c_void_p()
        check(_lib.lib().lo_octree_from_leaves(coded.ctx.h, coded.h, _p(b), _p(o), len(b), _p(box), int(level),
                                               int(curve), int(n_max), C.byref(h)))
        return cls(coded, _handle=h)

    def serialize(self, path: str) -> None:
        """LinearOctree::serialize (linear_octree.cpp:149-160) to a LOC1 file."""
        check(_lib.lib().lo_octree_save(self.ctx.h, self.h, os.fsencode(path)))

    @classmethod
    def deserialize(cls, path: str, coded: CodedCloud) -> "LinearOctree":
        """LinearOctree::deserialize (linear_octree.cpp:162-190) from a LOC1 file; the tree
        searches `coded` (its leaves must index exactly those points)."""
        h = C.c_void_p()
        check(_lib.lib().lo_octree_load(coded.ctx.h, coded.h, os.fsencode(path), C.byref(h)))
        return cls(coded, _handle=h)

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _lib.lib().lo_octree_destroy(self.h)
            except Exception:
                pass
            self.h = None

    @staticmethod
    def is_leaf(ref: int) -> bool:
        return ref < 0

    @staticmethod
    def leaf_id(ref: int) -> int:
        return ~ref

    @staticmethod
    def leaf_ref(i: int) -> int:
        return ~i

    def root(self) -> int:
        return int(self.info.root)

    def leaf_count(self) -> int:
        return int(self.info.leaves)

    def internal_count(self) -> int:
        return int(self.info.internal)

    def node_count(self) -> int:
        return self.leaf_count() + self.internal_count()

    def point_count(self) -> int:
        return int(self.info.points)

    def n_max(self) -> int:
        return int(self.info.n_max)

    def level(self) -> int:
        return int(self.info.level)

    def curve(self) -> Curve:
        return Curve(self.info.curve)

    def _fetch(self):
        if self._leaves is None:
            L, I = self.leaf_count(), self.internal_count()
            b = np.empty(L + 1, np.uint64)
            o = np.empty(L + 1, np.uint32)
            nodes = np.zeros(I, INTERNAL_NODE_DTYPE)
            check(_lib.lib().lo_octree_download(self.ctx.h, self.h, _p(b), _p(o), _p(nodes) if I else None))
            self._leaves = LeafArray(b, o)
            self._nodes = nodes

    def leaves(self) -> LeafArray:
        self._fetch()
        return self._leaves

    def internal_nodes(self) -> np.ndarray:
        self._fetch()
        return self._nodes

    def internal(self, ref: int):
        return self.internal_nodes()[ref]

    def points_in_node(self, ref: int) -> tuple[int, int]:
        if ref < 0:
            o = self.leaves().offsets
            return int(o[~ref]), int(o[~ref + 1])
        n = self.internal_nodes()[ref]
        return int(n["begin"]), int(n["end"])

    def node_prefix(self, ref: int) -> int:
        return int(self.leaves().boundaries[~ref]) if ref < 0 else int(self.internal_nodes()[ref]["prefix"])

    def node_depth(self, ref: int) -> int:
        if ref >= 0:
            return int(self.internal_nodes()[ref]["depth"])
        b = self.leaves().boundaries
        span = int(b[~ref + 1]) - int(b[~ref])
        return self.level() - ((span & -span).bit_length() - 1) // 3

    def node_bounds(self, refs):
        """linear_octree.cpp:139-147 for one NodeRef or an array of them: (6,) / (m, 6)."""
        scalar = np.isscalar(refs)
        r = np.atleast_1d(np.asarray(refs, np.int32))
        out = np.empty((len(r), 6))
        check(_lib.lib().lo_octree_node_bounds(self.ctx.h, self.h, _p(r), len(r), _p(out)))
        return out[0] if scalar else out


@dataclass
class BatchOptions:
    """search.hpp:110-117"""
    mode: BatchMode = BatchMode.Full
    subset_size: int = 5000
    seed: int = 0
    threads: int = 1
    collect_results: bool = False
    fingerprint: bool = True


@dataclass
class BatchResult:
    """search.hpp:121-131; `results` is kept as CSR (offsets, indices)."""
    centers: np.ndarray
    counts: np.ndarray
    fingerprints: np.ndarray
    offsets: np.ndarray | None = None
    indices: np.ndarray | None = None
    distances: np.ndarray | None = None  # kNN only: row-major (rows, k_eff)
    wall_seconds: float = 0.0
    device_ms: float = 0.0
    mean_count: float = 0.0
    extra: dict = field(default_factory=dict)

    @property
    def results(self):
        if self.offsets is None:
            return []
        return [self.indices[self.offsets[i]:self.offsets[i + 1]] for i in range(len(self.centers))]

    def mean_query_seconds(self) -> float:
        return self.wall_seconds / len(self.centers) if len(self.centers) else 0.0


@dataclass(frozen=True)
class KnnNeighbor:
    index: int
    dist_sq: float


def sample_indices(n: int, k: int, seed: int) -> np.ndarray:
    """rng.hpp:46-58"""
    out = np.empty(min(n, k), np.uint32)
    check(_lib.lib().lo_sample_indices(n, k, seed, _p(out)))
    return out


def _batch_centers(n: int, options: BatchOptions):
    if options.mode == BatchMode.Full:
        return None, np.arange(n, dtype=np.uint32)
    if options.subset_size > n:
        raise InvalidArgument("batch: subset size exceeds cloud size")
    c = sample_indices(n, options.subset_size, options.seed)
    return c, c


def run_radius_batch(tree: LinearOctree, coded: CodedCloud, method: RadiusMethod,
                     shape: KernelShape, radius: float, options: BatchOptions) -> BatchResult:
    """search.hpp:135-137.  Lin, Prune and Struct give the same exact sets.  Lin/Prune
    fingerprints hash the indices (search.cpp:345-347); Struct ones hash the coalesced ranges,
    a separator and the singles (search.cpp:325-336), and the result carries the ranged rows
    in `extra` (range_offsets, ranges, single_offsets, singles)."""
    if method == RadiusMethod.Ptr:
        raise InvalidArgument("run_radius_batch: ptr method needs a pointer octree")
    ctx = coded.ctx
    centres, centers_out = _batch_centers(coded.n, options)
    h = C.c_void_p()
    t0 = time.perf_counter()
    check(_lib.lib().lo_radius(ctx.h, tree.h, coded.h, int(method), int(shape), float(radius),
                               _p(centres), 0 if centres is None else len(centres),
                               int(options.fingerprint), C.byref(h)))
    wall = time.perf_counter() - t0
    try:
        info = CsrInfo()
        check(_lib.lib().lo_csr_info_get(h, C.byref(info)))
        m = int(info.rows)
        counts = np.empty(m, np.uint32)
        fps = np.empty(m, np.uint64) if options.fingerprint else np.zeros(0, np.uint64)
        offs = idx = None
        if options.collect_results:
            offs = np.empty(m + 1, np.uint64)
            idx = np.empty(int(info.total), np.uint32)
        check(_lib.lib().lo_csr_download(ctx.h, h, _p(counts), _p(fps) if options.fingerprint else None,
                                         _p(offs), _p(idx)))
        extra = {}
        if method == RadiusMethod.Struct:
            ro, rg, so, sg = _struct_rows(h, ctx, m)
            extra = dict(range_offsets=ro, ranges=rg, single_offsets=so, singles=sg)
    finally:
        _lib.lib().lo_csr_destroy(h)
    return BatchResult(centers_out, counts, fps, offs, idx, None, wall, float(info.device_ms),
                       float(info.mean_count), extra)


def run_knn_batch(tree: LinearOctree, coded: CodedCloud, k: int, options: BatchOptions,
                  collect_distances: bool = False) -> BatchResult:
    """search.hpp:145-146: per centre the first min(k, N) (index, dist_sq) by (dist, index)."""
    if k < 1:
        raise InvalidArgument("knn: k must be >= 1")
    ctx = coded.ctx
    centres, centers_out = _batch_centers(coded.n, options)
    h = C.c_void_p()
    t0 = time.perf_counter()
    check(_lib.lib().lo_knn(ctx.h, tree.h, coded.h, int(k), _p(centres),
                            0 if centres is None else len(centres), int(options.fingerprint), C.byref(h)))
    wall = time.perf_counter() - t0
    try:
        rows, keff, ms = C.c_uint64(), C.c_uint32(), C.c_double()
        check(_lib.lib().lo_knn_info_get(h, C.byref(rows), C.byref(keff), C.byref(ms)))
        m, ke = int(rows.value), int(keff.value)
        fps = np.empty(m, np.uint64) if options.fingerprint else np.zeros(0, np.uint64)
        idx = dist = None
        if options.collect_results or collect_distances:
            idx = np.empty(m * ke, np.uint32)
            dist = np.empty(m * ke, np.float64)
        check(_lib.lib().lo_knn_download(ctx.h, h, _p(idx), _p(dist), _p(fps) if options.fingerprint else None))
    finally:
        _lib.lib().lo_knn_destroy(h)
    counts = np.full(m, ke, np.uint32)
    offs = np.arange(m + 1, dtype=np.uint64) * ke if idx is not None else None
    return BatchResult(centers_out, counts, fps, offs, idx, dist, wall, ms.value, float(ke))


def neighbours_lin(tree: LinearOctree, coded: CodedCloud, kernel: SearchKernel) -> np.ndarray:
    """search.hpp:61-64: ascending reordered indices strictly inside the kernel."""
    return radius_points(tree, coded, kernel.shape, kernel.radius, np.asarray([kernel.center], float))[0]


neighbours_prune = neighbours_lin


@dataclass
class RangedResult:
    """search.hpp:18-56: disjoint ascending [begin, end) ranges of wholly contained octants
    (adjacent ones coalesced) plus the individually tested survivor indices."""
    ranges: np.ndarray   # (k, 2) u32
    singles: np.ndarray  # u32, ascending

    def count(self) -> int:
        return int(len(self.singles) + (self.ranges[:, 1].astype(np.int64) - self.ranges[:, 0]).sum())

    def expand(self) -> np.ndarray:
        parts = [np.arange(b, e, dtype=np.uint32) for b, e in self.ranges] + [self.singles]
        out = np.concatenate(parts) if parts else np.zeros(0, np.uint32)
        return np.sort(out, kind="stable").astype(np.uint32)


def _struct_rows(h, ctx, m):
    """Download a Struct result: per row a RangedResult (CSR of ranges and singles)."""
    L = _lib.lib()
    tr, ts = C.c_uint64(), C.c_uint64()
    check(L.lo_csr_struct_info(h, C.byref(tr), C.byref(ts)))
    ro = np.empty(m + 1, np.uint64)
    so = np.empty(m + 1, np.uint64)
    rg = np.empty((int(tr.value), 2), np.uint32)
    sg = np.empty(int(ts.value), np.uint32)
    check(L.lo_csr_struct_download(ctx.h, h, _p(ro), _p(rg), _p(so), _p(sg)))
    return ro, rg, so, sg


def neighbours_struct(tree: LinearOctree, coded: CodedCloud, kernel: SearchKernel) -> RangedResult:
    """search.hpp:75-78 at one arbitrary centre."""
    return struct_points(tree, coded, kernel.shape, kernel.radius, np.asarray([kernel.center], float))[0]


def struct_points(tree: LinearOctree, coded: CodedCloud, shape: KernelShape, radius: float,
                  centres_xyz) -> list[RangedResult]:
    """neighbours_struct at arbitrary centres (one RangedResult per centre)."""
    if not (radius > 0.0) or not np.isfinite(radius):
        raise InvalidArgument("kernel radius must be positive and finite")
    q = np.ascontiguousarray(centres_xyz, np.float64).reshape(-1, 3)
    h = C.c_void_p()
    check(_lib.lib().lo_radius_struct_points(coded.ctx.h, tree.h, coded.h, int(shape), float(radius),
                                             _p(q), len(q), C.byref(h)))
    try:
        ro, rg, so, sg = _struct_rows(h, coded.ctx, len(q))
    finally:
        _lib.lib().lo_csr_destroy(h)
    return [RangedResult(rg[ro[i]:ro[i + 1]], sg[so[i]:so[i + 1]]) for i in range(len(q))]


def radius_points(tree: LinearOctree, coded: CodedCloud, shape: KernelShape, radius: float,
                  centres_xyz) -> list[np.ndarray]:
    """neighbours_lin at arbitrary centres (one row per centre)."""
    if not (radius > 0.0) or not np.isfinite(radius):
        raise InvalidArgument("kernel radius must be positive and finite")
    q = np.ascontiguousarray(centres_xyz, np.float64).reshape(-1, 3)
    h = C.c_void_p()
    check(_lib.lib().lo_radius_points(coded.ctx.h, tree.h, coded.h, int(shape), float(radius), _p(q),
                                      len(q), C.byref(h)))
    try:
        info = CsrInfo()
        check(_lib.lib().lo_csr_info_get(h, C.byref(info)))
        offs = np.empty(len(q) + 1, np.uint64)
        idx = np.empty(int(info.total), np.uint32)
        check(_lib.lib().lo_csr_download(coded.ctx.h, h, None, None, _p(offs), _p(idx)))
    finally:
        _lib.lib().lo_csr_destroy(h)
    return [idx[offs[i]:offs[i + 1]] for i in range(len(q))]


def knn_lin_oct(tree: LinearOctree, coded: CodedCloud, center, k: int) -> list[KnnNeighbor]:
    """search.hpp:101-105 at one arbitrary centre."""
    idx, dist = knn_points(tree, coded, np.asarray([center], float), k)
    return [KnnNeighbor(int(i), float(d)) for i, d in zip(idx[0], dist[0])]


def knn_points(tree: LinearOctree, coded: CodedCloud, centres_xyz, k: int):
    """kNN at arbitrary centres -> (idx (m, k_eff), dist (m, k_eff))."""
    if k < 1:
        raise InvalidArgument("knn: k must be >= 1")
    q = np.ascontiguousarray(centres_xyz, np.float64).reshape(-1, 3)
    if not np.isfinite(q).all():
        raise InvalidArgument("kernel center must be finite")
    h = C.c_void_p()
    check(_lib.lib().lo_knn_points(coded.ctx.h, tree.h, coded.h, int(k), _p(q), len(q), C.byref(h)))
    try:
        rows, keff, ms = C.c_uint64(), C.c_uint32(), C.c_double()
        check(_lib.lib().lo_knn_info_get(h, C.byref(rows), C.byref(keff), C.byref(ms)))
        ke = int(keff.value)
        idx = np.empty(len(q) * ke, np.uint32)
        dist = np.empty(len(q) * ke, np.float64)
        check(_lib.lib().lo_knn_download(coded.ctx.h, h, _p(idx), _p(dist), None))
    finally:
        _lib.lib().lo_knn_destroy(h)
    return idx.reshape(len(q), ke), dist.reshape(len(q), ke)


# ---- sfc codecs on grid cells (sfc.hpp:56-83) --------------------------------------------
def sfc_encode(curve: Curve, cells, level: int = kMaxLevel, ctx: Context | None = None) -> np.ndarray:
    c = np.ascontiguousarray(cells, np.uint32).reshape(-1, 3)
    out = np.empty(len(c), np.uint64)
    check(_lib.lib().lo_encode_cells((ctx or default_context()).h, _p(c), len(c), int(curve), level, _p(out)))
    return out


def sfc_decode(curve: Curve, codes, level: int = kMaxLevel, ctx: Context | None = None) -> np.ndarray:
    c = np.ascontiguousarray(codes, np.uint64).reshape(-1)
    out = np.empty((len(c), 3), np.uint32)
    check(_lib.lib().lo_decode_codes((ctx or default_context()).h, _p(c), len(c), int(curve), level, _p(out)))
    return out


def morton_encode(cell, level: int = kMaxLevel) -> int:
    return int(sfc_encode(Curve.Morton, [cell], level)[0])


def hilbert_encode(cell, level: int = kMaxLevel) -> int:
    return int(sfc_encode(Curve.Hilbert, [cell], level)[0])


# ---- synthetic inputs (host) -------------------------------------------------------------
def generate_uniform(n: int, seed: int, extent: float = 100.0) -> np.ndarray:
    a = np.empty((n, 3))
    check(_lib.lib().lo_generate_uniform(n, seed, extent, _p(a)))
    return a


def generate_terrain(n: int, seed: int, extent_xy: float = 1000.0) -> np.ndarray:
    a = np.empty((n, 3))
    check(_lib.lib().lo_generate_terrain(n, seed, extent_xy, _p(a)))
    return a


def generate_mixed(n: int, seed: int) -> np.ndarray:
    a = np.empty((n, 3))
    check(_lib.lib().lo_generate_mixed(n, seed, _p(a)))
    return a


# ---- locality (locality.hpp / locality.cpp) ------------------------------------------------
@dataclass
class LocalityHistogram:
    """locality.hpp:18-40: bins = ascending distinct |i - j| with their counts."""
    k: int
    cloud_size: int
    centres: int
    d: np.ndarray      # u32, ascending
    count: np.ndarray  # u64

    @property
    def bins(self):
        return list(zip(self.d.tolist(), self.count.tolist()))

    def total(self) -> int:
        return int(self.count.sum(dtype=np.uint64))

    def count_at(self, d: int) -> int:
        i = int(np.searchsorted(self.d, d))
        return int(self.count[i]) if i < len(self.d) and self.d[i] == d else 0

    # sequential left-to-right double accumulation, as locality.cpp:19-37 (np.cumsum is
    # sequential; np.sum would be pairwise and round differently)
    def mean(self) -> float:
        t = self.total()
        if t == 0:
            return 0.0
        s = np.cumsum(self.d.astype(np.float64) * self.count.astype(np.float64))[-1]
        return float(s / float(t))

    def stddev(self) -> float:
        t = self.total()
        if t == 0:
            return 0.0
        dd = self.d.astype(np.float64) - self.mean()
        s = np.cumsum(dd * dd * self.count.astype(np.float64))[-1]
        return float(np.sqrt(s / float(t)))


def fisher_pearson_skewness(h: LocalityHistogram) -> float:
    """locality.cpp:112-125."""
    t = h.total()
    if t == 0:
        return 0.0
    mu, sigma = h.mean(), h.stddev()
    if sigma == 0.0:
        return 0.0
    z = (h.d.astype(np.float64) - mu) / sigma
    s = np.cumsum(z * z * z * h.count.astype(np.float64))[-1]
    return float(s / float(t))


def histogram_quantiles(h: LocalityHistogram):
    """locality.cpp:127-140: smallest d whose cumulative count reaches 25 / 50 / 75 % of the mass."""
    t = h.total()
    out = [0.0, 0.0, 0.0]
    if t == 0:
        return out
    cum = np.cumsum(h.count.astype(np.uint64))
    for qi, q in enumerate((0.25, 0.5, 0.75)):
        i = int(np.argmax(cum.astype(np.float64) >= q * float(t)))
        out[qi] = float(h.d[i])
    return out


def _locality(tree: LinearOctree, coded: CodedCloud, k: int, centres, index_map) -> LocalityHistogram:
    n = coded.n
    if k < 1:
        raise InvalidArgument("locality histogram: k must be >= 1")
    if k > n:
        raise InvalidArgument("locality histogram: k exceeds cloud size")
    imap = None
    if index_map is not None:
        imap = np.ascontiguousarray(index_map, np.uint32)
        if len(imap) != n:
            raise InvalidArgument("locality histogram: index map size mismatch")
    L = _lib.lib()
    ctx = coded.ctx
    res = C.c_void_p()
    m = n if centres is None else len(centres)
    check(L.lo_knn(ctx.h, tree.h, coded.h, int(k), _p(centres), 0 if centres is None else m, 0, C.byref(res)))
    try:
        nb = C.c_uint64()
        check(L.lo_locality_histogram(ctx.h, res, coded.h, _p(centres), _p(imap), C.byref(nb), None, None, 0))
        d = np.empty(nb.value, np.uint32)
        c = np.empty(nb.value, np.uint64)
        check(L.lo_locality_histogram(ctx.h, res, coded.h, _p(centres), _p(imap), C.byref(nb), _p(d), _p(c),
                                      len(d)))
    finally:
        L.lo_knn_destroy(res)
    return LocalityHistogram(int(k), n, m, d, c)


def locality_histogram(tree: LinearOctree, coded: CodedCloud, k: int, threads: int = 1,
                       index_map=None) -> LocalityHistogram:
    """locality.hpp:49-51: exact histogram over every centre (index_map: e.g. coded.permutation
    to measure the original storage order)."""
    return _locality(tree, coded, k, None, index_map)


def locality_histogram_approx(tree: LinearOctree, coded: CodedCloud, k: int, sample_size: int, seed: int,
                              threads: int = 1, index_map=None) -> LocalityHistogram:
    """locality.hpp:55-58: over sample_indices(n, sample_size, seed)."""
    if sample_size > coded.n:
        raise InvalidArgument("locality histogram: sample size exceeds cloud size")
    return _locality(tree, coded, k, sample_indices(coded.n, sample_size, seed), index_map)


# ---- memory model (memory_model.hpp / memory_model.cpp) ------------------------------------
@dataclass
class MemoryReport:
    """memory_model.hpp:27-45 for the linear octree; `device_bytes` adds what the B200 path keeps
    resident beyond the reference's arrays (traversal table, FP32 shadow)."""
    bytes_total: int
    node_count: int
    point_count: int
    device_bytes: int = 0

    def rho(self) -> float:
        return 0.0 if self.point_count == 0 else self.node_count / self.point_count

    def overhead(self, point_bytes: float = 32.0) -> float:
        return self.bytes_total / (point_bytes * self.point_count)


def measure_structure(tree: LinearOctree) -> MemoryReport:
    """memory_model.cpp:21-30: boundaries (8 B) + offsets (4 B) per leaf + 1, 56 B per internal node."""
    L = tree.leaf_count()
    b = (L + 1) * 8 + (L + 1) * 4 + tree.internal_count() * 56
    dev = b + int(tree.info.tnodes) * (64 + 48)
    return MemoryReport(b, tree.node_count(), tree.point_count(), dev)


@dataclass
class StructureCostParams:
    """memory_model.hpp:13-24."""
    node_bytes: float = 0.0
    point_extra_bytes: float = 0.0
    nodes_per_point: float = 0.0
    point_bytes: float = 32.0


def expected_overhead(p: StructureCostParams) -> float:
    return (p.point_extra_bytes + p.nodes_per_point * p.node_bytes) / p.point_bytes


def linear_octree_cost_params(rho: float) -> StructureCostParams:
    """memory_model.cpp:39-43: 7 leaves (12 B) per 56 B internal node."""
    return StructureCostParams((7.0 * 12.0 + 56.0) / 8.0, 0.0, rho, 32.0)
