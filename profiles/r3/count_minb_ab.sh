#!/bin/bash
# Count-kernel residency: in-tree (__launch_bounds__(128, 10)) vs a side build with 9, then the GPU suite
OUT=gpurun_out
for c in cfg3 cfg1 cfg4; do
  timeout 600 python profiles/radius_probe.py --config $c --reps 3 >> $OUT/minb_ab3.log 2>&1
  LO_LIB_PATH=$PWD/_var/minb9/liblinoct_b200.so timeout 600 python profiles/radius_probe.py --config $c --reps 3 >> $OUT/minb_ab3.log 2>&1
done
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/gputest_minb10.log 2>&1; echo "pytest rc=$?" >> $OUT/gputest_minb10.log
exit 0
