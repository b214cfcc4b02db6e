#!/bin/bash
# kNN (k <= 16) gathered-leaf candidate prefilter (in-tree) vs none (_var/old)
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fallbacks.py tests/test_gpu_scale.py -x -q -k "knn or Knn or kNN" > $OUT/p30_tests.log 2>&1; tail -2 $OUT/p30_tests.log
timeout 600 python profiles/knn_probe.py --config cfg1 --k 8 16 --variants heaps >> $OUT/p30_knn.log 2>&1
LO_LIB_PATH=$PWD/_var/old/liblinoct_b200.so timeout 600 python profiles/knn_probe.py --config cfg1 --k 8 16 --variants heaps >> $OUT/p30_knn.log 2>&1
timeout 900 python profiles/knn_probe.py --config cfg3 --k 16 --reps 2 --variants heaps >> $OUT/p30_knn.log 2>&1
LO_LIB_PATH=$PWD/_var/old/liblinoct_b200.so timeout 900 python profiles/knn_probe.py --config cfg3 --k 16 --reps 2 --variants heaps >> $OUT/p30_knn.log 2>&1
grep '^{' $OUT/p30_knn.log
exit 0
