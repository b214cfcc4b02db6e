"""ctypes binding of liblinoct_b200.so (the C ABI in include/linoct_b200.h).

There is no CPU fallback: loading fails loudly when the library is missing, and every call
that needs a GPU raises when no CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# LO_LIB_PATH: a side build of a tuning variant (build.py with LO_BUILD_DIR); the product path is the in-tree .so
LIB_PATH = os.environ.get("LO_LIB_PATH") or os.path.join(HERE, "liblinoct_b200.so")
HEADER = os.path.join(HERE, "..", "include", "linoct_b200.h")

P = C.c_void_p
PP = C.POINTER(C.c_void_p)
u32, u64, i32, f64, cint = C.c_uint32, C.c_uint64, C.c_int32, C.c_double, C.c_int

OK, INVALID_ARGUMENT, DOMAIN_ERROR, LOGIC_ERROR, OUT_OF_MEMORY, CUDA_ERROR, NO_DEVICE, RUNTIME_ERROR, NCCL_ERROR = range(9)


class CodedInfo(C.Structure):
    _fields_ = [("n", u64), ("curve", i32), ("level", i32), ("disc_box", f64 * 6),
                ("cloud_box", f64 * 6), ("scale", f64 * 3)]


class OctreeInfo(C.Structure):
    _fields_ = [("leaves", u64), ("internal", u64), ("root", i32), ("n_max", u32),
                ("level", i32), ("curve", i32), ("points", u64), ("tnodes", u64)]


class CsrInfo(C.Structure):
    _fields_ = [("rows", u64), ("total", u64), ("mean_count", f64), ("device_ms", f64)]


# name -> (restype, argtypes)
SIGNATURES = {
    "lo_last_error": (C.c_char_p, []),
    "lo_abi_version": (cint, []),
    "lo_launch_count": (u64, []),
    "lo_device_count": (cint, [P]),
    "lo_context_create": (cint, [cint, P, PP]),
    "lo_context_destroy": (cint, [P]),
    "lo_context_synchronize": (cint, [P]),
    "lo_context_stream": (P, [P]),
    "lo_context_join": (cint, [P]),
    "lo_context_set_option": (cint, [P, cint, C.c_int64]),
    "lo_context_set_timing": (cint, [P, cint]),
    "lo_context_stage_times": (cint, [P, P, cint, P, cint]),
    "lo_device_alloc": (cint, [P, u64, PP]),
    "lo_device_free": (cint, [P, P]),
    "lo_memcpy_h2d": (cint, [P, P, P, u64]),
    "lo_memcpy_d2h": (cint, [P, P, P, u64]),
    "lo_host_alloc_pinned": (cint, [u64, PP]),
    "lo_host_free_pinned": (cint, [P]),
    "lo_flush_l2": (cint, [P, P, u64]),
    "lo_compute_codes": (cint, [P, P, u64, cint, cint, P, P]),
    "lo_encode_cells": (cint, [P, P, u64, cint, cint, P]),
    "lo_decode_codes": (cint, [P, P, u64, cint, cint, P]),
    "lo_reorder": (cint, [P, P, u64, cint, cint, PP]),
    "lo_reorder_device": (cint, [P, P, u64, cint, cint, PP]),
    "lo_coded_info_get": (cint, [P, C.POINTER(CodedInfo)]),
    "lo_coded_download": (cint, [P, P, P, P, P]),
    "lo_coded_device_ptrs": (cint, [P, PP, PP, PP, PP, PP]),
    "lo_coded_destroy": (cint, [P]),
    "lo_coded_create_empty": (cint, [P, C.POINTER(CodedInfo), PP]),
    "lo_invert_permutation": (cint, [P, P, u64, P]),
    "lo_build_leaves": (cint, [P, P, u64, u32, cint, P, P, P, u64]),
    "lo_octree_build": (cint, [P, P, u32, PP]),
    "lo_octree_info_get": (cint, [P, C.POINTER(OctreeInfo)]),
    "lo_octree_download": (cint, [P, P, P, P, P]),
    "lo_octree_node_bounds": (cint, [P, P, P, u64, P]),
    "lo_octree_destroy": (cint, [P]),
    "lo_octree_device_ptrs": (cint, [P, PP, PP, PP, PP]),
    "lo_octree_create_empty": (cint, [P, P, C.POINTER(OctreeInfo), PP]),
    "lo_radius": (cint, [P, P, P, cint, cint, f64, P, u64, cint, PP]),
    "lo_radius_points": (cint, [P, P, P, cint, f64, P, u64, PP]),
    "lo_radius_range": (cint, [P, P, P, cint, cint, f64, u64, u64, cint, PP]),
    "lo_csr_info_get": (cint, [P, C.POINTER(CsrInfo)]),
    "lo_csr_download": (cint, [P, P, P, P, P, P]),
    "lo_csr_device_ptrs": (cint, [P, PP, PP]),
    "lo_csr_download_async": (cint, [P, P, P, P, P, P]),
    "lo_h2d_begin": (cint, [P, P, P, u64, cint]),
    "lo_h2d_wait": (cint, [P, cint]),
    "lo_d2h_fence": (cint, [P, cint]),
    "lo_d2h_wait": (cint, [P, cint]),
    "lo_csr_destroy": (cint, [P]),
    "lo_csr_struct_info": (cint, [P, P, P]),
    "lo_reorder_pcb": (cint, [P, C.c_char_p, cint, cint, PP]),
    "lo_locality_histogram": (cint, [P, P, P, P, P, P, P, P, u64]),
    "lo_coded_write_pcb": (cint, [P, P, C.c_char_p]),
    "lo_octree_from_leaves": (cint, [P, P, P, P, u64, P, cint, cint, u32, PP]),
    "lo_octree_save": (cint, [P, P, C.c_char_p]),
    "lo_octree_load": (cint, [P, P, C.c_char_p, PP]),
    "lo_csr_struct_download": (cint, [P, P, P, P, P, P]),
    "lo_radius_struct_points": (cint, [P, P, P, cint, f64, P, u64, PP]),
    "lo_knn": (cint, [P, P, P, u32, P, u64, cint, PP]),
    "lo_knn_points": (cint, [P, P, P, u32, P, u64, PP]),
    "lo_knn_range": (cint, [P, P, P, u32, u64, u64, cint, PP]),
    "lo_knn_info_get": (cint, [P, P, P, P]),
    "lo_knn_download": (cint, [P, P, P, P, P]),
    "lo_knn_download_async": (cint, [P, P, P, P, P]),
    "lo_link_leaves": (cint, [P, P, P, u64, P, cint, P, P, P, u64]),
    "lo_comm_unique_id": (cint, [P]),
    "lo_comm_init": (cint, [P, P, cint, cint, PP]),
    "lo_comm_info": (cint, [P, P, P]),
    "lo_comm_destroy": (cint, [P]),
    "lo_shard_range": (cint, [u64, cint, cint, P, P]),
    "lo_broadcast_structure": (cint, [P, P, P, cint, PP, PP]),
    "lo_structure_copy": (cint, [P, P, P, PP, PP]),
    "lo_radius_sharded": (cint, [P, P, P, cint, cint, f64, cint, PP, P, P, P]),
    "lo_weighted_bounds": (cint, [P, u64, u32, u64, u32, cint, P]),
    "lo_radius_work_bounds": (cint, [P, P, P, cint, f64, u32, cint, P]),
    "lo_radius_sharded_bounds": (cint, [P, P, P, cint, cint, f64, cint, P, PP, P, P, P]),
    "lo_knn_sharded": (cint, [P, P, P, u32, cint, PP, P]),
    "lo_octant_bounds": (cint, [P, cint, u32, u32, u32, cint, P]),
    "lo_knn_destroy": (cint, [P]),
    "lo_locality_log2": (cint, [P, P, P, P, cint, P]),
    "lo_generate_uniform": (cint, [u64, u64, f64, P]),
    "lo_generate_terrain": (cint, [u64, u64, f64, P]),
    "lo_generate_mixed": (cint, [u64, u64, P]),
    "lo_sample_indices": (cint, [u32, u32, u64, P]),
}

_lib = None


def header_symbols(path: str = HEADER) -> list[str]:
    """Every function the C header declares."""
    import re

    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lo_[a-z0-9_]+)\s*\(", text)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class LinoctError(Exception):
    pass


class InvalidArgument(LinoctError, ValueError):
    """std::invalid_argument"""


class DomainError(LinoctError, ValueError):
    """std::domain_error"""


class LogicError(LinoctError, RuntimeError):
    """std::logic_error"""


class CudaError(LinoctError, RuntimeError):
    """CUDA failure, out of memory, or no device"""


class FileFormatError(LinoctError, RuntimeError):
    """std::runtime_error: unreadable or malformed PCB1 / XYZ / LOC1 files"""


class NcclError(LinoctError, RuntimeError):
    """NCCL missing or a collective failed (multi-GPU entry points)"""


_EXC = {INVALID_ARGUMENT: InvalidArgument, DOMAIN_ERROR: DomainError, LOGIC_ERROR: LogicError,
        RUNTIME_ERROR: FileFormatError, NCCL_ERROR: NcclError}


def check(status: int) -> None:
    if status != OK:
        msg = lib().lo_last_error().decode(errors="replace")
        raise _EXC.get(status, CudaError)(msg)
