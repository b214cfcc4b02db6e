#!/bin/bash
# L1 prefetch of kept leaf children's FP32 points (in-tree), + FP64 coords (_var/pre2), none (_var/nopre)
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > $OUT/p6_tests.log 2>&1; tail -2 $OUT/p6_tests.log
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p6_radius.log 2>&1
  for v in nopre pre2; do
    LO_LIB_PATH=$PWD/_var/$v/liblinoct_b200.so timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p6_radius.log 2>&1
  done
done
timeout 300 python profiles/sort_probe.py --config cfg3 >> $OUT/p6_sort.log 2>&1
cat $OUT/p6_radius.log $OUT/p6_sort.log
exit 0
