#!/bin/bash
# Round-3 evidence pass B: --set full captures of the changed kernels (after the plain run exited 0)
source profiles/ncu_cap.sh
P="python profiles/run_profile.py --config cfg3 --reps 1"
timeout 600 $P --radius 1.0 --fingerprint > gpurun_out/fb_plain.log 2>&1 || exit 1
cap g_count radius_pt_kernel "-c 1" $P --radius 1.0
cap g_fill radius_replay "-c 1" $P --radius 1.0
cap g_sort onesweep_pass "-s 3 -c 1" $P --radius
cap g_gather gather_soa "-c 1" $P --radius
cap g_c1_count_r3 radius_pt_kernel "-s 3 -c 1" python profiles/run_profile.py --config cfg1 --reps 1 --radius 0.5 1.0 2.0 3.0
cap g_c1_sort onesweep_pass "-s 3 -c 1" python profiles/run_profile.py --config cfg1 --reps 1 --radius
ls gpurun_out | grep "^g_"
exit 0
