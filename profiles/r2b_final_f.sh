#!/bin/bash
# --set full of the count kernel (cfg3 r = 1, cfg1 r = 3) and the gather with the final code (reports overwritten)
source profiles/ncu_cap.sh
timeout 600 python profiles/run_profile.py --config cfg3 --reps 1 --radius 1.0 > gpurun_out/ff_plain.log 2>&1 || exit 1
cap g_count radius_pt_kernel "-c 1" python profiles/run_profile.py --config cfg3 --reps 1 --radius 1.0
cap g_c1_count_r3 radius_pt_kernel "-s 3 -c 1" python profiles/run_profile.py --config cfg1 --reps 1 --radius 0.5 1.0 2.0 3.0
cap g_gather gather_soa "-c 1" python profiles/run_profile.py --config cfg3 --reps 1 --radius
tail -2 gpurun_out/ncu_g_count.log
exit 0
