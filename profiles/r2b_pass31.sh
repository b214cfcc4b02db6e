#!/bin/bash
# kNN prefilter for k >= 16 only: tests and k = 8 / 16 / 32 timings (cfg1), k = 16 (cfg3)
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fallbacks.py -x -q -k "knn or Knn or kNN" > $OUT/p31_tests.log 2>&1; tail -2 $OUT/p31_tests.log
timeout 600 python profiles/knn_probe.py --config cfg1 --k 8 16 32 --variants heaps >> $OUT/p31_knn.log 2>&1
timeout 900 python profiles/knn_probe.py --config cfg3 --k 16 --reps 2 --variants heaps >> $OUT/p31_knn.log 2>&1
grep '^{' $OUT/p31_knn.log
exit 0
