"""B200-native SFC reorder -> linear octree -> radius / kNN search (arxiv 2603.06771 hot path).

The product is liblinoct_b200.so (sm_100a CUDA + C ABI, include/linoct_b200.h); this package
is its reference-shaped host API (`linoct`) and the multi-GPU plumbing (`distributed`).
"""
from . import linoct  # noqa: F401
from .linoct import *  # noqa: F401,F403
