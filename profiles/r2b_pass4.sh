#!/bin/bash
# per-group box skip in the radius count (LO_PT_GROUPS) vs without (_var/nogrp)
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fallbacks.py -x -q > $OUT/p4_tests.log 2>&1; tail -2 $OUT/p4_tests.log
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p4_radius.log 2>&1
  LO_LIB_PATH=$PWD/_var/nogrp/liblinoct_b200.so timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p4_radius.log 2>&1
done
cat $OUT/p4_radius.log
exit 0
