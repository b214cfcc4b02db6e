"""Multi-rank check of the sharded path on real device buffers (launched by
tests/test_gpu_multirank.py under torchrun).  Rank 0 reorders + builds, the structure is
broadcast (distributed.broadcast_structure), every rank searches its contiguous SFC shard
(radius + kNN), and rank 0 compares the concatenated shards with its own single-rank batch.

On a one-GPU box all ranks share cuda:0 and talk over gloo -- the data path (zero-copy views of
library memory, empty-handle replicas, lazily rebuilt FP32 shadows, global row bases) is the
same as with one GPU per rank over NCCL."""
import ctypes as C
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

from oracle.oracle_py import Oracle  # noqa: E402
from paper_2603_06771_b200 import _lib, distributed as D, linoct as lo  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    L = _lib.lib()
    ctx = lo.Context(0)
    n = 300_000
    coded = tree = None
    if rank == 0:
        pts = Oracle().gen_terrain(n, 77, 150.0)
        coded = C.c_void_p()
        _lib.check(L.lo_reorder(ctx.h, pts.ctypes.data, n, 1, 21, C.byref(coded)))
        tree = C.c_void_p()
        _lib.check(L.lo_octree_build(ctx.h, coded, 32, C.byref(tree)))
    coded, tree, ci, ti = D.broadcast_structure(ctx, coded, tree, src=0)
    b0, b1 = D.shard_range(n, rank, world)
    out = {}
    for r in (0.8, 2.0):
        h = C.c_void_p()
        _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, b0, b1, 1, C.byref(h)))
        cnt = np.empty(b1 - b0, np.uint32)
        fps = np.empty(b1 - b0, np.uint64)
        _lib.check(L.lo_csr_download(ctx.h, h, cnt.ctypes.data, fps.ctypes.data, None, None))
        info = _lib.CsrInfo()
        _lib.check(L.lo_csr_info_get(h, C.byref(info)))
        base, total = D.global_row_base(int(info.total), device="cpu")
        L.lo_csr_destroy(h)
        out[r] = (cnt, fps, base, total)
    kh = C.c_void_p()
    _lib.check(L.lo_knn_range(ctx.h, tree, coded, 12, b0, b1, 1, C.byref(kh)))
    kf = np.empty(b1 - b0, np.uint64)
    _lib.check(L.lo_knn_download(ctx.h, kh, None, None, kf.ctypes.data))
    L.lo_knn_destroy(kh)
    gathered = [None] * world
    dist.all_gather_object(gathered, (rank, {r: (c.tobytes(), f.tobytes(), b, t) for r, (c, f, b, t) in out.items()},
                                      kf.tobytes()))
    ok = True
    if rank == 0:
        gathered.sort(key=lambda g: g[0])
        for r in (0.8, 2.0):
            h = C.c_void_p()
            _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, 0, n, 1, C.byref(h)))
            cnt = np.empty(n, np.uint32)
            fps = np.empty(n, np.uint64)
            _lib.check(L.lo_csr_download(ctx.h, h, cnt.ctypes.data, fps.ctypes.data, None, None))
            L.lo_csr_destroy(h)
            c_all = np.concatenate([np.frombuffer(g[1][r][0], np.uint32) for g in gathered])
            f_all = np.concatenate([np.frombuffer(g[1][r][1], np.uint64) for g in gathered])
            bases = [g[1][r][2] for g in gathered]
            ok &= np.array_equal(c_all, cnt) and np.array_equal(f_all, fps)
            ok &= bases[0] == 0 and all(bases[i + 1] - bases[i] == int(np.frombuffer(gathered[i][1][r][0], np.uint32)
                                                                       .astype(np.uint64).sum())
                                        for i in range(world - 1))
        kh = C.c_void_p()
        _lib.check(L.lo_knn_range(ctx.h, tree, coded, 12, 0, n, 1, C.byref(kh)))
        kf = np.empty(n, np.uint64)
        _lib.check(L.lo_knn_download(ctx.h, kh, None, None, kf.ctypes.data))
        L.lo_knn_destroy(kh)
        ok &= np.array_equal(np.concatenate([np.frombuffer(g[2], np.uint64) for g in gathered]), kf)
        print("DIST_CHECK", "PASS" if ok else "FAIL", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
