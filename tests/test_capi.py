"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol the header
declares, refuses to run without a device (no CPU fallback), and its host-side generators
reproduce the oracle's / reference's inputs."""
import ctypes as C

import numpy as np
import pytest

from paper_2603_06771_b200 import _lib, linoct


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    names = _lib.header_symbols()
    assert len(names) >= 45
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)
    assert L.lo_abi_version() == 1


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = _lib.lib()
    h = C.c_void_p()
    rc = L.lo_context_create(0, None, C.byref(h))
    assert rc == _lib.NO_DEVICE
    assert b"no CUDA device" in L.lo_last_error()
    with pytest.raises(_lib.CudaError):
        linoct.Context(0)


def test_generators_match_oracle(oracle):
    assert np.array_equal(linoct.generate_uniform(3000, 5, 100.0), oracle.gen_uniform(3000, 5, 100.0))
    assert np.array_equal(linoct.generate_terrain(3000, 6, 1000.0), oracle.gen_terrain(3000, 6, 1000.0))
    assert np.array_equal(linoct.generate_mixed(5000, 7), oracle.gen_mixed(5000, 7))
    assert np.array_equal(linoct.sample_indices(9000, 700, 3), oracle.sample_indices(9000, 700, 3))


def test_internal_node_layout():
    assert linoct.INTERNAL_NODE_DTYPE.itemsize == 56
    assert linoct.INTERNAL_NODE_DTYPE.fields["begin"][1] == 40
    assert linoct.INTERNAL_NODE_DTYPE.fields["depth"][1] == 48
    assert linoct.INTERNAL_NODE_DTYPE.fields["child_mask"][1] == 49


def test_host_argument_errors_before_device():
    with pytest.raises(linoct.InvalidArgument):
        linoct.SearchKernel(linoct.KernelShape.Sphere, (0, 0, 0), -1.0)
    with pytest.raises(linoct.InvalidArgument):
        linoct.PointCloud(np.array([[0.0, np.nan, 1.0]]))


def test_octant_bounds_host_matches_reference(ref):
    """lo_octant_bounds (Discretizer::octant_bounds, sfc.cpp:110-127) is host arithmetic in the library:
    bit-equal to the reference's padded boxes on random octants of random boxes."""
    L = _lib.lib()
    rng = np.random.default_rng(3)
    for _ in range(300):
        lo_ = rng.uniform(-1e3, 1e3, 3)
        box = np.concatenate([lo_, lo_ + rng.uniform(0, 500, 3)])
        level = int(rng.integers(1, 22))
        depth = int(rng.integers(0, level + 1))
        h = rng.integers(0, 2 ** depth, 3) if depth else np.zeros(3, np.int64)
        out = np.zeros(6)
        assert L.lo_octant_bounds(box.ctypes.data_as(C.c_void_p), level, int(h[0]), int(h[1]), int(h[2]), depth,
                                  out.ctypes.data_as(C.c_void_p)) == _lib.OK
        want = ref.octant_bounds(box, int(h[0]), int(h[1]), int(h[2]), depth, level)
        assert np.array_equal(out.view(np.uint64), np.asarray(want, np.float64).view(np.uint64))
    out = np.zeros(6)
    assert L.lo_octant_bounds(box.ctypes.data_as(C.c_void_p), 3, 0, 0, 0, 4, out.ctypes.data_as(C.c_void_p)) == \
        _lib.INVALID_ARGUMENT


def test_shard_range_host():
    """lo_shard_range (host arithmetic): contiguous, covering, balanced slices = distributed.shard_range."""
    from paper_2603_06771_b200 import distributed as D
    L = _lib.lib()
    for n in (0, 1, 7, 1000, 100_000_000, 2 ** 32 - 1):
        for g in (1, 2, 3, 8):
            prev = 0
            for r in range(g):
                b, e = C.c_uint64(), C.c_uint64()
                assert L.lo_shard_range(n, r, g, C.byref(b), C.byref(e)) == _lib.OK
                assert (b.value, e.value) == D.shard_range(n, r, g)
                assert b.value == prev and e.value - b.value in (n // g, n // g + 1)
                prev = e.value
            assert prev == n
    b, e = C.c_uint64(), C.c_uint64()
    assert L.lo_shard_range(10, 2, 2, C.byref(b), C.byref(e)) == _lib.INVALID_ARGUMENT


def _weighted_bounds_ref(counts, stride, n, base, g):
    """Restatement of lo_weighted_bounds' rule: cut at the block edge nearest to each total*r/g."""
    import numpy as np
    q = np.minimum(stride, n - np.arange(len(counts), dtype=np.int64) * stride)
    cum = np.cumsum(q.astype(object) * (np.asarray(counts, dtype=object) + base))
    total = int(cum[-1]) if len(cum) else 0
    out, j = [0], 0
    for r in range(1, g):
        t = total * r // g
        while j < len(cum) and cum[j] <= t:
            j += 1
        cut = j
        if j < len(cum):
            before = int(cum[j - 1]) if j else 0
            if t - before > int(cum[j]) - t:
                cut = j + 1
        out.append(max(out[-1], min(n, cut * stride)))
    out.append(n)
    return out


def test_weighted_bounds_host():
    """lo_weighted_bounds (host arithmetic): covering, ordered, stride-aligned cuts that
    split the sampled work evenly; equals the restated rule; uniform work gives ~equal slices."""
    import numpy as np
    from paper_2603_06771_b200 import distributed as D
    rng = np.random.default_rng(3)
    for n, stride in ((1, 64), (1000, 64), (100_000, 64), (1_000_003, 32), (64 * 10, 64)):
        samples = (n + stride - 1) // stride
        for kind in ("uniform", "skewed", "zeros"):
            if kind == "uniform":
                c = np.full(samples, 50, np.uint32)
            elif kind == "zeros":
                c = np.zeros(samples, np.uint32)
            else:  # a dense cluster in the middle: 10x the work
                c = rng.integers(20, 80, samples).astype(np.uint32)
                c[samples // 3: samples // 2] *= 10
            for g in (1, 2, 3, 8):
                b = D.weighted_bounds(c, stride, n, g)
                assert b[0] == 0 and b[-1] == n and np.all(np.diff(b.astype(np.int64)) >= 0)
                assert all(int(x) % stride == 0 for x in b[1:-1] if int(x) != n)
                assert [int(x) for x in b] == _weighted_bounds_ref(c, stride, n, 16, g)
                if samples >= 8 * g:  # each rank within one block's cost of the even share
                    q = np.minimum(stride, n - np.arange(samples) * stride)
                    cost = q * (c.astype(np.int64) + 16)
                    per = [cost[int(b[r]) // stride: (int(b[r + 1]) + stride - 1) // stride].sum() for r in range(g)]
                    assert max(per) - cost.sum() / g <= cost.max() + 1
    L = _lib.lib()
    out = np.zeros(3, np.uint64)
    c = np.zeros(2, np.uint32)
    assert L.lo_weighted_bounds(c.ctypes.data, 3, 64, 100, 16, 2, out.ctypes.data) == _lib.INVALID_ARGUMENT
