#!/bin/bash
# Round 2 evidence pass A: GPU tests, the default bench line (driver's K/W), the reference arm and the
# launch list of one bench step.
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > $OUT/final_gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/final_gputest.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/final_bench.json 2> $OUT/final_bench.err; echo "bench rc=$?" >> $OUT/final_bench.err
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/final_ref.json 2> $OUT/final_ref.err; echo "ref rc=$?" >> $OUT/final_ref.err
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn --no-extra"
timeout 600 $B > $OUT/final_small.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/final_launches_cfg3.csv $B > $OUT/ncu_l.log 2>&1
du -sh $OUT
exit 0
