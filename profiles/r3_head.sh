#!/bin/bash
# Bench line on the round's last commit (Struct walk at 10 blocks per SM) and a --set full capture of the Struct count walk
source profiles/ncu_cap.sh
OUT=gpurun_out
timeout 600 python bench.py > $OUT/r3_bench_head.json 2> $OUT/r3_bench_head.err; echo "bench rc=$?"
cap r3_struct "struct_pt_kernel" "-c 1" python profiles/struct_probe.py --config cfg3 --reps 1; echo "cap rc=$?"
exit 0
