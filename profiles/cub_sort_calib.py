"""Calibration only (not a product path): CUB's onesweep radix sort through torch.sort on the
same key counts as the reorder stage (u64 keys + index payload), device-timed with CUDA events.

    python profiles/cub_sort_calib.py
"""
import json

import torch

out = {}
for n in (10_000_000, 100_000_000):
    g = torch.Generator(device="cuda").manual_seed(1)
    k = torch.randint(0, 2**62, (n,), device="cuda", generator=g, dtype=torch.int64)
    for _ in range(3):
        torch.sort(k, stable=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch.sort(k, stable=True)
    e1.record()
    torch.cuda.synchronize()
    out[n] = round(e0.elapsed_time(e1) / 10, 4)
print(json.dumps({"torch_sort_int64_stable_ms": out, "note": "int64 keys + int64 indices (CUB SortPairs)"}))
