#!/bin/bash
# default bench line after the round-2 second-session sort / radius changes, plus the launch list of one step
OUT=gpurun_out
timeout 1500 python bench.py > $OUT/b1.json 2> $OUT/b1.err; echo "bench rc=$?"; tail -3 $OUT/b1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/b1_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn --no-extra > $OUT/b1_ncu.log 2>&1; echo "ncu rc=$?"
exit 0
