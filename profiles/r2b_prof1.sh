#!/bin/bash
# --set full of the cfg3 radius count and one onesweep pass after the round-2 second-session changes
source profiles/ncu_cap.sh
P="python profiles/run_profile.py --config cfg3 --reps 1"
timeout 600 $P --radius 1.0 > gpurun_out/p1_plain.log 2>&1 || exit 1
cap p1_count radius_pt_kernel "-c 1" $P --radius 1.0
cap p1_sort onesweep_pass "-s 3 -c 1" $P --radius
exit 0
