#!/bin/bash
# Round-3 evidence pass A: GPU test suite, default bench line, reference arm, launch list of one step
OUT=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $OUT/fa_gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/fa_gputest.log; tail -3 $OUT/fa_gputest.log
timeout 1500 python bench.py > $OUT/fa_bench.json 2> $OUT/fa_bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/fa_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn --no-extra > $OUT/fa_ncu.log 2>&1; echo "ncu rc=$?"
exit 0
