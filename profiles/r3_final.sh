#!/bin/bash
# Round 2, third session, final evidence on the committed tree (count kernel at 10 blocks per SM, encode grid 8 per SM):
# smoke, GPU suite, both bench arms, launch list, --set full of the count kernel (cfg3 r = 1)
source profiles/ncu_cap.sh
OUT=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/r3_smoke.log 2>&1; tail -1 $OUT/r3_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > $OUT/r3_gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/r3_gputest.log; tail -3 $OUT/r3_gputest.log
timeout 1500 python bench.py --impl reference > $OUT/r3_ref.json 2> $OUT/r3_ref.err; echo "ref rc=$?"
timeout 1500 python bench.py > $OUT/r3_bench.json 2> $OUT/r3_bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r3_launches_cfg3.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn --no-extra > $OUT/r3_ncu.log 2>&1; echo "ncu rc=$?"
P="python profiles/run_profile.py --config cfg3 --reps 1 --radius 1.0 --fingerprint"
cap r3_count "radius_pt_kernel" "-c 1" $P; echo "cap rc=$?"
exit 0
