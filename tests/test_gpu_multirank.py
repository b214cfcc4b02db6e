"""The N > 1 paths on a real device: tests/gpu_dist_check.py (broadcast structure, per-rank
shards, concatenation == single rank) and bench.py's torchrun leg, both with two ranks.  A
one-GPU box runs both ranks on cuda:0 over gloo; with one GPU per rank the same code runs over
NCCL.  These check correctness and that the launch contract holds, not multi-GPU speed."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(args, env_extra, timeout):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    env = dict(os.environ, **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_sharded_search_equals_single_rank():
    r = _torchrun([os.path.join(ROOT, "tests", "gpu_dist_check.py")], {}, 600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "DIST_CHECK PASS" in r.stdout


@pytest.mark.parametrize("replicate", ["0", "1"])  # structure broadcast from rank 0 / built on every rank
def test_bench_two_ranks_contract(replicate):
    r = _torchrun(["bench.py", "--gpus", "2", "--steps", "2", "--warmup", "1", "--no-cpu-baseline",
                   "--config", "cfg0"],
                  {"LO_BENCH_SAME_DEVICE": "1", "LO_BENCH_DIST_BACKEND": "gloo",
                   "LO_BENCH_REPLICATE": replicate}, 900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0


# ---- the C-ABI multi-GPU path (lo_comm / lo_structure_copy, csrc/comm.cu) ------------------------
def _csr_rows(L, ctx_h, csr):
    import ctypes as C
    import numpy as np
    from paper_2603_06771_b200 import _lib
    info = _lib.CsrInfo()
    _lib.check(L.lo_csr_info_get(csr, C.byref(info)))
    counts = np.empty(info.rows, np.uint32)
    fps = np.empty(info.rows, np.uint64)
    offs = np.empty(info.rows + 1, np.uint64)
    idx = np.empty(max(1, info.total), np.uint32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _lib.check(L.lo_csr_download(ctx_h, csr, p(counts), p(fps), p(offs), p(idx)))
    return counts, fps, offs, idx[:info.total]


def test_c_abi_two_contexts_shards_equal_single():
    """Single-process stand-in for G = 2 ranks on one device: the structure is built on context A,
    replicated onto context B with lo_structure_copy (peer copies), each context searches its
    lo_shard_range slice, and the concatenation by offset equals A's single batch bit for bit."""
    import ctypes as C
    import gc

    import numpy as np
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from oracle.oracle_py import Oracle
    from paper_2603_06771_b200 import _lib, distributed as D, linoct as lo
    L = _lib.lib()
    ca, cb = lo.Context(0), lo.Context(0)
    n = 400_000
    pts = Oracle().gen_mixed(n, 5)
    coded, tree = C.c_void_p(), C.c_void_p()
    _lib.check(L.lo_reorder(ca.h, pts.ctypes.data, n, 1, 21, C.byref(coded)))
    _lib.check(L.lo_octree_build(ca.h, coded, 64, C.byref(tree)))
    cb_coded, cb_tree = D.structure_copy(cb, coded, tree)
    # the replica is complete: identical tables
    ta, tb = _lib.OctreeInfo(), _lib.OctreeInfo()
    _lib.check(L.lo_octree_info_get(tree, C.byref(ta)))
    _lib.check(L.lo_octree_info_get(cb_tree, C.byref(tb)))
    assert bytes(ta) == bytes(tb)
    whole = C.c_void_p()
    _lib.check(L.lo_radius_range(ca.h, tree, coded, 1, 0, 1.5, 0, n, 1, C.byref(whole)))
    wc, wf, wo, wi = _csr_rows(L, ca.h, whole)
    parts = []
    for rank, (ctx, c, t) in enumerate([(ca, coded, tree), (cb, cb_coded, cb_tree)]):
        b, e = C.c_uint64(), C.c_uint64()
        _lib.check(L.lo_shard_range(n, rank, 2, C.byref(b), C.byref(e)))
        csr = C.c_void_p()
        _lib.check(L.lo_radius_range(ctx.h, t, c, 1, 0, 1.5, b.value, e.value, 1, C.byref(csr)))
        parts.append((b.value, e.value) + _csr_rows(L, ctx.h, csr))
        L.lo_csr_destroy(csr)
    assert parts[0][1] == parts[1][0] and parts[1][1] == n
    counts = np.concatenate([p[2] for p in parts])
    fps = np.concatenate([p[3] for p in parts])
    idx = np.concatenate([p[5] for p in parts])
    base = int(parts[0][4][-1])
    offs = np.concatenate([parts[0][4][:-1], parts[1][4] + np.uint64(base)])
    assert np.array_equal(counts, wc) and np.array_equal(fps, wf)
    assert np.array_equal(offs, wo) and np.array_equal(idx, wi)
    for h in (whole,):
        L.lo_csr_destroy(h)
    for t, c in ((cb_tree, cb_coded), (tree, coded)):
        L.lo_octree_destroy(t)
        L.lo_coded_destroy(c)
    gc.collect()
    assert L.lo_context_destroy(cb.h) == _lib.OK
    cb.h = None


def test_c_abi_nccl_comm_world_one():
    """lo_comm with one rank (NCCL refuses two ranks on one GPU): unique id, init, the broadcast
    (root keeps its handles), sharded radius / kNN with row base 0 and the global total, timed
    broadcast stage, destroy."""
    import ctypes as C

    import numpy as np
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from oracle.oracle_py import Oracle
    from paper_2603_06771_b200 import _lib, distributed as D, linoct as lo
    L = _lib.lib()
    ctx = lo.Context(0)
    comm = D.Comm(ctx, 0, 1)
    n = 200_000
    pts = Oracle().gen_terrain(n, 8, 150.0)
    coded, tree = C.c_void_p(), C.c_void_p()
    _lib.check(L.lo_reorder(ctx.h, pts.ctypes.data, n, 1, 21, C.byref(coded)))
    _lib.check(L.lo_octree_build(ctx.h, coded, 32, C.byref(tree)))
    ctx.set_timing(True)
    c2, t2 = comm.broadcast_structure(coded, tree, root=0)
    assert c2.value == coded.value and t2.value == tree.value
    assert "broadcast" in [name for name, _ in ctx.stage_times()]
    ctx.set_timing(False)
    csr, b, base, total = comm.radius(tree, coded, 2.0)
    single = C.c_void_p()
    _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, 2.0, 0, n, 1, C.byref(single)))
    a, s = _csr_rows(L, ctx.h, csr), _csr_rows(L, ctx.h, single)
    assert b == 0 and base == 0 and total == int(a[0].astype(np.uint64).sum())
    assert all(np.array_equal(x, y) for x, y in zip(a, s))
    res, kb = comm.knn(tree, coded, 16)
    assert kb == 0
    for h in (csr, single):
        L.lo_csr_destroy(h)
    L.lo_knn_destroy(res)
    L.lo_octree_destroy(tree)
    L.lo_coded_destroy(coded)
    comm.close()


def test_work_weighted_shards():
    """§8e.3: lo_radius_work_bounds (a radius batch over one query tile per stride block) gives bounds that cover the
    cloud, are identical when recomputed (every rank derives them alone), balance the neighbour work
    of a clustered cloud better than equal slices, and whose slices concatenate to the single batch;
    lo_radius_sharded_bounds at world size 1 takes them."""
    import ctypes as C

    import numpy as np
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from oracle.oracle_py import Oracle
    from paper_2603_06771_b200 import _lib, distributed as D, linoct as lo
    L = _lib.lib()
    ctx = lo.Context(0)
    n, r, g = 400_000, 1.0, 8
    pts = Oracle().gen_mixed(n, 11)
    coded, tree = C.c_void_p(), C.c_void_p()
    _lib.check(L.lo_reorder(ctx.h, pts.ctypes.data, n, 1, 21, C.byref(coded)))
    _lib.check(L.lo_octree_build(ctx.h, coded, 64, C.byref(tree)))
    bw = D.radius_work_bounds(ctx, tree, coded, r, g, stride=256)
    assert np.array_equal(bw, D.radius_work_bounds(ctx, tree, coded, r, g, stride=256))
    assert bw[0] == 0 and bw[-1] == n and np.all(np.diff(bw.astype(np.int64)) >= 0)
    full = C.c_void_p()
    _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, 0, n, 1, C.byref(full)))
    fc, ff, _, fi = _csr_rows(L, ctx.h, full)
    parts = []
    for k in range(g):
        s = C.c_void_p()
        _lib.check(L.lo_radius_range(ctx.h, tree, coded, 1, 0, r, int(bw[k]), int(bw[k + 1]), 1, C.byref(s)))
        parts.append(_csr_rows(L, ctx.h, s))
        L.lo_csr_destroy(s)
    assert np.array_equal(np.concatenate([p[0] for p in parts]), fc)
    assert np.array_equal(np.concatenate([p[1] for p in parts]), ff)
    assert np.array_equal(np.concatenate([p[3] for p in parts]), fi)
    cum = np.concatenate([[0], np.cumsum(fc.astype(np.int64) + 16)])
    eq = [D.shard_range(n, k, g) for k in range(g)]
    imb = lambda bb: max(cum[e] - cum[b] for b, e in bb) / (cum[-1] / g)  # noqa: E731
    w = imb([(int(bw[k]), int(bw[k + 1])) for k in range(g)])
    assert w <= 1.05 and w <= imb(eq) + 0.03  # sampled estimate: within a few % of even
    comm = D.Comm(ctx, 0, 1)
    b1 = D.radius_work_bounds(ctx, tree, coded, r, 1, stride=256)
    assert list(b1) == [0, n]
    csr, b, base, total = comm.radius(tree, coded, r, bounds=b1)
    assert b == 0 and base == 0 and total == int(fc.astype(np.uint64).sum())
    for h in (csr, full):
        L.lo_csr_destroy(h)
    L.lo_octree_destroy(tree)
    L.lo_coded_destroy(coded)
    comm.close()
