#!/bin/bash
# Struct walk residency: in-tree (__launch_bounds__(128, 8)) vs a side build with 10 (-DLO_STRUCT_MINB=10)
OUT=gpurun_out
for c in cfg1 cfg3; do
  timeout 900 python profiles/struct_probe.py --config $c --reps 3 >> $OUT/struct_minb_ab.log 2>&1
  LO_LIB_PATH=$PWD/_var/structminb10/liblinoct_b200.so timeout 900 python profiles/struct_probe.py --config $c --reps 3 >> $OUT/struct_minb_ab.log 2>&1
done
exit 0
