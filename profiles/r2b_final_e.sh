#!/bin/bash
# Final pass after the count-pass band / unroll changes: smoke, GPU suite, default bench, launch list,
# --set full of the count kernel (cfg3 r = 1 and cfg1 r = 3), per-stage DRAM traffic
source profiles/ncu_cap.sh
OUT=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/fe_smoke.log 2>&1; tail -1 $OUT/fe_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > $OUT/fe_gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/fe_gputest.log; tail -3 $OUT/fe_gputest.log
timeout 1500 python bench.py > $OUT/fe_bench.json 2> $OUT/fe_bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/fe_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn --no-extra > $OUT/fe_ncu.log 2>&1; echo "ncu rc=$?"
P="python profiles/run_profile.py --config cfg3 --reps 1 --radius 1.0 --fingerprint"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/fe_traffic_launches_cfg3.csv $P > $OUT/fe_ncu2.log 2>&1; echo "ncu traffic rc=$?"
cap g_count radius_pt_kernel "-c 1" python profiles/run_profile.py --config cfg3 --reps 1 --radius 1.0
cap g_c1_count_r3 radius_pt_kernel "-s 3 -c 1" python profiles/run_profile.py --config cfg1 --reps 1 --radius 0.5 1.0 2.0 3.0
cap g_gather gather_soa "-c 1" python profiles/run_profile.py --config cfg3 --reps 1 --radius
exit 0
