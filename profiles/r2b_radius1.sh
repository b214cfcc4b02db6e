#!/bin/bash
# per-point tile-box prefilter in the radius walk vs without (side build _var/nopf); full GPU suite
OUT=gpurun_out
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/r1_radius.log 2>&1
  LO_LIB_PATH=$PWD/_var/nopf/liblinoct_b200.so timeout 300 python profiles/radius_probe.py --config $c >> $OUT/r1_radius.log 2>&1
done
cat $OUT/r1_radius.log
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/r1_tests.log 2>&1; tail -3 $OUT/r1_tests.log
exit 0
