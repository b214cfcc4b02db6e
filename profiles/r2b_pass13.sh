#!/bin/bash
# leaf-box kernel with 2 (in-tree) / 1 / 4 nodes in flight per 8-lane group
OUT=gpurun_out
for c in cfg3 cfg1; do
  timeout 300 python profiles/build_probe.py --config $c >> $OUT/p13_build.log 2>&1
  for v in lb1 lb4; do LO_LIB_PATH=$PWD/_var/$v/liblinoct_b200.so timeout 300 python profiles/build_probe.py --config $c >> $OUT/p13_build.log 2>&1; done
done
cat $OUT/p13_build.log
exit 0
