#!/bin/bash
# Round capture on one B200: the bench line, the launch list of the same command, and
# --set full captures of the dominant kernels (each only after the plain run exited 0).
set -x
OUT=gpurun_out
timeout 900 python bench.py > $OUT/bench_r1.json 2> $OUT/bench_r1.err || exit 1
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn > $OUT/bench_small.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/launches_r1.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn > $OUT/ncu_launch.log 2>&1
timeout 300 python profiles/run_profile.py --radius 3.0 --k 16 --reps 2 > $OUT/prof_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:radius_pt_kernelILi0ELb0E -s 1 -c 1 \
    -o $OUT/count_r3 python profiles/run_profile.py --radius 3.0 --reps 2 > $OUT/ncu_count.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radius_replay_kernel -s 1 -c 1 \
    -o $OUT/fill_r3 python profiles/run_profile.py --radius 3.0 --reps 2 > $OUT/ncu_fill.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_float_kernel -s 1 -c 1 \
    -o $OUT/knn16 python profiles/run_profile.py --radius --k 16 --reps 2 > $OUT/ncu_knn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radius_digest -s 1 -c 1 \
    -o $OUT/digest_r3 python profiles/run_profile.py --radius 3.0 --reps 2 --fingerprint > $OUT/ncu_digest.log 2>&1
ls -la $OUT
