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
