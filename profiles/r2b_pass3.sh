#!/bin/bash
# packed (key | index) u64 kNN heap entries (k >= 32) vs split key / index arrays (_var/old)
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fallbacks.py -x -q -k "knn or Knn or kNN" > $OUT/p3_tests.log 2>&1; tail -2 $OUT/p3_tests.log
timeout 600 python profiles/knn_probe.py --config cfg1 --k 16 32 64 --variants heaps >> $OUT/p3_knn.log 2>&1
LO_LIB_PATH=$PWD/_var/old/liblinoct_b200.so timeout 600 python profiles/knn_probe.py --config cfg1 --k 16 32 64 --variants heaps >> $OUT/p3_knn.log 2>&1
grep '^{' $OUT/p3_knn.log
exit 0
