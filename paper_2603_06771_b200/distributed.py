"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL / NVLink).

SURVEY.md §8e: the sorted points and the octree are built once (rank `src`) and broadcast;
queries shard by contiguous SFC-ordered index ranges; each rank's CSR rows are global rows
[begin, end) and are concatenated by offset -- the only other exchange is one all-gather of
the per-rank neighbour totals.  No collective sits on the search path itself.

The tensor-level helpers (`shard_range`, `global_row_base`, `broadcast_buffers`) take plain
torch tensors, so the same code runs with gloo on CPU (tests/test_distributed.py) and NCCL on
device memory views of the library's buffers (`device_view`).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import CodedInfo, OctreeInfo, check


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced split of [0, n): rank r owns [r*n//w, (r+1)*n//w)."""
    return n * rank // world, n * (rank + 1) // world


def weighted_shard_range(prefix: np.ndarray, rank: int, world: int) -> tuple[int, int]:
    """Split rows so each rank gets ~equal work, given an inclusive-prefix-style array of
    per-row cost with prefix[0] = 0 and prefix[-1] = total (e.g. CSR offsets after a count
    pass): the fill pass of cfg3 is balanced by neighbours, not by queries (§8e.3)."""
    total = int(prefix[-1])
    lo = int(np.searchsorted(prefix, total * rank // world, side="left"))
    hi = int(np.searchsorted(prefix, total * (rank + 1) // world, side="left"))
    if rank == world - 1:
        hi = len(prefix) - 1
    return min(lo, len(prefix) - 1), min(hi, len(prefix) - 1)


def global_row_base(local_total: int, group=None, device=None) -> tuple[int, int]:
    """Exclusive prefix of the per-rank totals (u64) -> (this rank's base, grand total)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = torch.tensor([local_total], dtype=torch.int64, device=device)
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t, group=group)
    vals = [int(g.item()) for g in gathered]
    return sum(vals[:rank]), sum(vals)


def broadcast_buffers(buffers: list[torch.Tensor], src: int = 0, group=None) -> None:
    """Broadcast every tensor in place from `src` (uint8 views of device memory under NCCL)."""
    for b in buffers:
        if b.numel():
            dist.broadcast(b, src=src, group=group)


class _CudaArray:
    """Minimal __cuda_array_interface__ wrapper so torch can view library-owned memory."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 2,
            "strides": None,
        }


def device_view(ptr: int, nbytes: int, device: int) -> torch.Tensor:
    """Zero-copy uint8 tensor over `nbytes` of device memory at `ptr`."""
    if nbytes == 0:
        return torch.empty(0, dtype=torch.uint8, device=f"cuda:{device}")
    with torch.cuda.device(device):
        return torch.as_tensor(_CudaArray(ptr, nbytes), device=f"cuda:{device}")


def _coded_views(coded_h, n: int, device: int) -> list[torch.Tensor]:
    L = _lib.lib()
    x, y, z, codes, perm = (C.c_void_p() for _ in range(5))
    check(L.lo_coded_device_ptrs(coded_h, C.byref(x), C.byref(y), C.byref(z), C.byref(codes),
                                 C.byref(perm)))
    return [device_view(x.value, 8 * n, device), device_view(y.value, 8 * n, device),
            device_view(z.value, 8 * n, device), device_view(codes.value, 8 * n, device),
            device_view(perm.value, 4 * n, device)]


def _tree_views(tree_h, info: OctreeInfo, device: int) -> list[torch.Tensor]:
    L = _lib.lib()
    b, o, nodes, tn = (C.c_void_p() for _ in range(4))
    check(L.lo_octree_device_ptrs(tree_h, C.byref(b), C.byref(o), C.byref(nodes), C.byref(tn)))
    return [device_view(b.value, 8 * (info.leaves + 1), device),
            device_view(o.value, 4 * (info.leaves + 1), device),
            device_view(nodes.value, 56 * info.internal, device),
            device_view(tn.value, 64 * info.tnodes, device)]


def broadcast_structure(ctx, coded_h, tree_h, src: int = 0, group=None):
    """Replicate (CodedCloud, LinearOctree) from rank `src` to every rank of `group`.

    Rank src passes its handles; the others pass None and receive new handles.  Returns
    (coded_h, tree_h, coded_info, tree_info) on every rank."""
    rank = dist.get_rank(group)
    L = _lib.lib()
    header = [None]
    if rank == src:
        ci, ti = CodedInfo(), OctreeInfo()
        check(L.lo_coded_info_get(coded_h, C.byref(ci)))
        check(L.lo_octree_info_get(tree_h, C.byref(ti)))
        header = [(bytes(ci), bytes(ti))]
    dist.broadcast_object_list(header, src=src, group=group)
    ci = CodedInfo.from_buffer_copy(header[0][0])
    ti = OctreeInfo.from_buffer_copy(header[0][1])
    if rank != src:
        h = C.c_void_p()
        check(L.lo_coded_create_empty(ctx.h, C.byref(ci), C.byref(h)))
        coded_h = h
        t = C.c_void_p()
        check(L.lo_octree_create_empty(ctx.h, coded_h, C.byref(ti), C.byref(t)))
        tree_h = t
    ctx.synchronize()
    views = _coded_views(coded_h, ci.n, ctx.device) + _tree_views(tree_h, ti, ctx.device)
    broadcast_buffers(views, src=src, group=group)
    torch.cuda.synchronize(ctx.device)
    return coded_h, tree_h, ci, ti


# ---- the C-ABI path: the library's own NCCL communicator (lo_comm) ---------------------------
class Comm:
    """lo_comm (include/linoct_b200.h, csrc/comm.cu): an NCCL communicator owned by the library on
    one context.  torch.distributed only ships the 128-byte NCCL unique id (any process group,
    gloo included); the structure broadcast, the per-rank totals all-gather and the sharded
    searches are C-ABI calls a C++ caller makes the same way."""

    def __init__(self, ctx, rank: int, world: int, group=None, uid: bytes | None = None):
        L = _lib.lib()
        if uid is None:
            box = [None]
            if rank == 0:
                buf = C.create_string_buffer(128)
                check(L.lo_comm_unique_id(buf))
                box = [buf.raw]
            if world > 1:
                dist.broadcast_object_list(box, src=0, group=group)
            uid = box[0]
        h = C.c_void_p()
        check(L.lo_comm_init(ctx.h, C.create_string_buffer(uid, 128), world, rank, C.byref(h)))
        self.h, self.ctx, self.rank, self.world = h, ctx, rank, world

    def close(self):
        if getattr(self, "h", None):
            _lib.lib().lo_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shard(self, n: int) -> tuple[int, int]:
        b, e = C.c_uint64(), C.c_uint64()
        check(_lib.lib().lo_shard_range(n, self.rank, self.world, C.byref(b), C.byref(e)))
        return b.value, e.value

    def broadcast_structure(self, coded_h, tree_h, root: int = 0):
        """Root passes its handles and gets them back; the others get new handles."""
        c, t = C.c_void_p(), C.c_void_p()
        check(_lib.lib().lo_broadcast_structure(self.h, coded_h, tree_h, root, C.byref(c), C.byref(t)))
        return (coded_h, tree_h) if self.rank == root else (c, t)

    def radius(self, tree_h, coded_h, r: float, method: int = 1, shape: int = 0, fingerprint: int = 1,
               bounds: np.ndarray | None = None):
        """-> (csr handle, row_begin, row_base, total neighbours of all ranks); `bounds` (nranks + 1 u64, e.g.
        from work_bounds) replaces the equal slices."""
        csr = C.c_void_p()
        b, base, tot = C.c_uint64(), C.c_uint64(), C.c_uint64()
        if bounds is None:
            check(_lib.lib().lo_radius_sharded(self.h, tree_h, coded_h, method, shape, r, fingerprint, C.byref(csr),
                                               C.byref(b), C.byref(base), C.byref(tot)))
        else:
            bd = np.ascontiguousarray(bounds, dtype=np.uint64)
            check(_lib.lib().lo_radius_sharded_bounds(self.h, tree_h, coded_h, method, shape, r, fingerprint,
                                                      bd.ctypes.data, C.byref(csr), C.byref(b), C.byref(base),
                                                      C.byref(tot)))
        return csr, b.value, base.value, tot.value

    def knn(self, tree_h, coded_h, k: int, fingerprint: int = 1):
        res = C.c_void_p()
        b = C.c_uint64()
        check(_lib.lib().lo_knn_sharded(self.h, tree_h, coded_h, k, fingerprint, C.byref(res), C.byref(b)))
        return res, b.value


def weighted_bounds(sample_counts: np.ndarray, stride: int, n: int, world: int, base_cost: int = 16) -> np.ndarray:
    """lo_weighted_bounds (host arithmetic, no device): bounds[0..world] splitting the sampled radius
    work evenly (sample j covers queries [j*stride, (j+1)*stride), cost count_j + base_cost each)."""
    c = np.ascontiguousarray(sample_counts, dtype=np.uint32)
    out = np.zeros(world + 1, dtype=np.uint64)
    check(_lib.lib().lo_weighted_bounds(c.ctypes.data, len(c), stride, n, base_cost, world, out.ctypes.data))
    return out


def radius_work_bounds(ctx, tree_h, coded_h, r: float, world: int, stride: int = 2048, shape: int = 0) -> np.ndarray:
    """lo_radius_work_bounds: one radius batch over the first query tile (32 centres) of every stride
    block, then weighted_bounds on the tiles' mean counts.
    Deterministic, so every rank computes the same bounds on its own copy of the structure."""
    out = np.zeros(world + 1, dtype=np.uint64)
    check(_lib.lib().lo_radius_work_bounds(ctx.h, tree_h, coded_h, shape, r, stride, world, out.ctypes.data))
    return out


def structure_copy(dst_ctx, coded_h, tree_h):
    """lo_structure_copy: single-process replication onto another context (peer copies)."""
    c, t = C.c_void_p(), C.c_void_p()
    check(_lib.lib().lo_structure_copy(dst_ctx.h, coded_h, tree_h, C.byref(c), C.byref(t)))
    return c, t
