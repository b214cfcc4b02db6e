#!/bin/bash
# replay record shape (LO_REPLAY_STATS) at cfg3 r=1 and cfg1 r=3; sort-stage repeatability at cfg3
OUT=gpurun_out
LO_REPLAY_STATS=1 timeout 300 python profiles/radius_probe.py --config cfg3 --reps 0 > $OUT/p7_stats.log 2>&1
LO_REPLAY_STATS=1 timeout 300 python profiles/radius_probe.py --config cfg1 --reps 0 --radius 1.0 3.0 >> $OUT/p7_stats.log 2>&1
grep "replay stats" $OUT/p7_stats.log
for i in 1 2 3; do timeout 300 python profiles/sort_probe.py --config cfg3 >> $OUT/p7_sort.log 2>&1; done
for i in 1 2; do timeout 300 python profiles/sort_probe.py --config cfg1 >> $OUT/p7_sort.log 2>&1; done
cat $OUT/p7_sort.log
exit 0
