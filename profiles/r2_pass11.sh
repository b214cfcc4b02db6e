#!/bin/bash
# GPU pass 11: radius walk knobs at cfg3 (coarse-node size, compact group-box multiplier)
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
P="python profiles/radius_probe.py --config cfg3 --reps 2"
timeout 200 $P >> $OUT/knobs11.log 2>&1
for c in 0 32 128 256; do LO_COARSE=$c timeout 200 $P >> $OUT/knobs11.log 2>&1; done
for m in 4 16 32; do LO_COMPACT_MUL=$m timeout 200 $P >> $OUT/knobs11.log 2>&1; done
for rm in 20 80; do LO_REPLAY_ROW_MAJOR_MIN=$rm timeout 200 $P >> $OUT/knobs11.log 2>&1; done
exit 0
