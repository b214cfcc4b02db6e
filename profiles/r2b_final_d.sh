#!/bin/bash
# per-launch DRAM bytes of every kernel of one cfg3 step (stage traffic for roofline.stages), then the GPU suite
OUT=gpurun_out
P="python profiles/run_profile.py --config cfg3 --reps 1 --radius 1.0 --fingerprint"
timeout 600 $P > $OUT/fd_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/fd_traffic_launches_cfg3.csv $P > $OUT/fd_ncu.log 2>&1; echo "ncu rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > $OUT/fd_gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/fd_gputest.log; tail -3 $OUT/fd_gputest.log
exit 0
