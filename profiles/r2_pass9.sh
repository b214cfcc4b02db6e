#!/bin/bash
# GPU pass 9: onesweep occupancy variants (items per thread / blocks per SM), cfg3 + cfg1 sort times
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for c in cfg3 cfg1; do
  timeout 300 python profiles/sort_probe.py --config $c >> $OUT/sort9.log 2>&1
  for v in sort_12_4 sort_8_5 sort_16_4; do
    LO_LIB_PATH=$PWD/_var/$v/liblinoct_b200.so timeout 300 python profiles/sort_probe.py --config $c >> $OUT/sort9.log 2>&1
  done
done
exit 0
