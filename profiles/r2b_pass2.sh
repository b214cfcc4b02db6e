#!/bin/bash
# look-back width variants (sort) and streamed leaf lists (radius count) vs per-leaf prefilter / none
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fallbacks.py -x -q > $OUT/p2_tests.log 2>&1; tail -2 $OUT/p2_tests.log
for c in cfg1 cfg3; do
  timeout 300 python profiles/sort_probe.py --config $c >> $OUT/p2_sort.log 2>&1
  for v in lb1 lb8; do
    LO_LIB_PATH=$PWD/_var/$v/liblinoct_b200.so timeout 300 python profiles/sort_probe.py --config $c >> $OUT/p2_sort.log 2>&1
  done
done
cat $OUT/p2_sort.log
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p2_radius.log 2>&1
  for v in nostream nopf; do
    LO_LIB_PATH=$PWD/_var/$v/liblinoct_b200.so timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p2_radius.log 2>&1
  done
done
cat $OUT/p2_radius.log
exit 0
