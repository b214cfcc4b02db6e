#!/bin/bash
# Final pass (kNN prefilter in): smoke, GPU suite, default bench, launch list, per-stage DRAM traffic
# --set full of the count kernel (cfg3 r = 1 and cfg1 r = 3), per-stage DRAM traffic
source profiles/ncu_cap.sh
OUT=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/fg_smoke.log 2>&1; tail -1 $OUT/fg_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > $OUT/fg_gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/fg_gputest.log; tail -3 $OUT/fg_gputest.log
timeout 1500 python bench.py > $OUT/fg_bench.json 2> $OUT/fg_bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/fg_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn --no-extra > $OUT/fg_ncu.log 2>&1; echo "ncu rc=$?"
P="python profiles/run_profile.py --config cfg3 --reps 1 --radius 1.0 --fingerprint"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/fg_traffic_launches_cfg3.csv $P > $OUT/fg_ncu2.log 2>&1; echo "ncu traffic rc=$?"



exit 0
