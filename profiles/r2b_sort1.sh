#!/bin/bash
# onesweep v2 (early counts, pipelined match ranking, epoch-tagged look-back) vs the round-2 kernel
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > $OUT/s1_tests.log 2>&1; tail -3 $OUT/s1_tests.log
for c in cfg1 cfg3; do
  timeout 300 python profiles/sort_probe.py --config $c >> $OUT/s1_sort.log 2>&1
  for v in old e0 g2 i16b3 i8b5; do
    LO_LIB_PATH=$PWD/_var/$v/liblinoct_b200.so timeout 300 python profiles/sort_probe.py --config $c >> $OUT/s1_sort.log 2>&1
  done
done
cat $OUT/s1_sort.log
timeout 300 python profiles/cub_sort_calib.py > $OUT/s1_cub.log 2>&1; cat $OUT/s1_cub.log
exit 0
