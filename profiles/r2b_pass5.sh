#!/bin/bash
# digest software pipelining (vs _var/nopipe) and gather ILP 4 (vs _var/ilp1)
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > $OUT/p5_tests.log 2>&1; tail -2 $OUT/p5_tests.log
for c in cfg3 cfg1; do
  timeout 300 python profiles/sort_probe.py --config $c >> $OUT/p5_sort.log 2>&1
  LO_LIB_PATH=$PWD/_var/ilp1/liblinoct_b200.so timeout 300 python profiles/sort_probe.py --config $c >> $OUT/p5_sort.log 2>&1
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p5_radius.log 2>&1
  LO_LIB_PATH=$PWD/_var/nopipe/liblinoct_b200.so timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p5_radius.log 2>&1
done
cat $OUT/p5_sort.log $OUT/p5_radius.log
exit 0
