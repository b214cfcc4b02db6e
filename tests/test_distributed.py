"""Multi-GPU plumbing on CPU (gloo, world_size 2): query sharding, global CSR row bases, the
structure broadcast helpers, and the concatenation-by-offset invariant of SURVEY.md §8e.
The per-rank search itself is the device kernel; here the C oracle stands in for it so the
exchange logic runs without a GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_06771_b200 import distributed as D


def test_shard_range_partitions():
    for n in (0, 1, 7, 1000, 10_000_001):
        for world in range(1, 9):
            spans = [D.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_weighted_shard_range_balances_work():
    rng = np.random.default_rng(0)
    counts = rng.integers(0, 700, 100_000)
    counts[30_000:40_000] *= 10  # a dense cluster run (cfg3)
    prefix = np.concatenate([[0], np.cumsum(counts)])
    for world in (2, 4, 8):
        spans = [D.weighted_shard_range(prefix, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == len(counts)
        for (a, b), (c, d) in zip(spans, spans[1:]):
            assert b == c
        work = [prefix[b] - prefix[a] for a, b in spans]
        assert max(work) <= prefix[-1] / world + counts.max() * 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle_py import Oracle

        o = Oracle()
        pts = o.gen_mixed(3000, 5)
        xs, codes, perm, box = o.reorder(pts, 1)
        # "structure broadcast": rank 0 owns the sorted points + a header, others receive
        header = [("n", len(xs), box.tolist())] if rank == 0 else [None]
        dist.broadcast_object_list(header, src=0)
        buf = torch.from_numpy(xs.copy()) if rank == 0 else torch.zeros(header[0][1], 3, dtype=torch.float64)
        D.broadcast_buffers([buf.view(torch.uint8)], src=0)
        xs_r = buf.numpy()
        assert np.array_equal(xs_r.view(np.uint64), xs.view(np.uint64))
        # each rank answers its contiguous SFC slice of the queries
        b0, b1 = D.shard_range(len(xs_r), rank, world)
        rows = [o.radius_brute(xs_r, xs_r[i], 9.0) for i in range(b0, b1)]
        local_counts = np.array([len(r) for r in rows], np.uint64)
        local_total = int(local_counts.sum())
        base, total = D.global_row_base(local_total)
        offsets = base + np.concatenate([[0], np.cumsum(local_counts)]).astype(np.uint64)
        gathered = [None] * world
        dist.all_gather_object(gathered, (b0, b1, offsets.tolist(),
                                          np.concatenate(rows).tolist() if rows else []))
        if rank == 0:
            # concatenation by offset == the single-rank CSR
            full_rows = [o.radius_brute(xs, xs[i], 9.0) for i in range(len(xs))]
            want_idx = np.concatenate(full_rows)
            want_off = np.concatenate([[0], np.cumsum([len(r) for r in full_rows])])
            got_idx = np.concatenate([np.array(g[3], np.uint32) for g in gathered])
            got_off = np.concatenate([[0]] + [np.array(g[2][1:], np.uint64) for g in gathered])
            assert total == len(want_idx)
            assert np.array_equal(got_idx, want_idx)
            assert np.array_equal(got_off.astype(np.int64), want_off.astype(np.int64))
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shard_and_concatenate():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = dict(q.get(timeout=5) for _ in procs)
    assert results == {0: "ok", 1: "ok"}, results
