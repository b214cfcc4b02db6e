#!/bin/bash
# persistent onesweep CTAs with the next tile id taken ahead vs one CTA per tile (_var/old)
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_parity.py -x -q > $OUT/p18_tests.log 2>&1; tail -2 $OUT/p18_tests.log
for c in cfg1 cfg3; do
  for i in 1 2; do
    timeout 300 python profiles/sort_probe.py --config $c >> $OUT/p18_sort.log 2>&1
    LO_LIB_PATH=$PWD/_var/old/liblinoct_b200.so timeout 300 python profiles/sort_probe.py --config $c >> $OUT/p18_sort.log 2>&1
  done
done
cat $OUT/p18_sort.log
exit 0
