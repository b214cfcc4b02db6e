#!/bin/bash
# Round 2 evidence pass on one B200: GPU tests, the default bench line (driver's K/W), the reference
# arm, the launch list of one bench step, and --set full captures of the top kernels (each capture
# only after its plain command exited 0).
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > $OUT/final_gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/final_gputest.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/final_bench.json 2> $OUT/final_bench.err; echo "bench rc=$?" >> $OUT/final_bench.err
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/final_ref.json 2> $OUT/final_ref.err; echo "ref rc=$?" >> $OUT/final_ref.err
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn --no-extra"
timeout 600 $B > $OUT/final_small.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/final_launches_cfg3.csv $B > $OUT/ncu_l.log 2>&1
P="python profiles/run_profile.py --config cfg3 --reps 1"
timeout 600 $P --radius 1.0 --k 16 --fingerprint > $OUT/final_prof.log 2>&1 || exit 1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:radius_pt_kernel -c 1 -o $OUT/f_count $P --radius 1.0 > $OUT/n1.log 2>&1
timeout 900 $NCU -k regex:radius_replay -c 1 -o $OUT/f_fill $P --radius 1.0 > $OUT/n2.log 2>&1
timeout 900 $NCU -k regex:radius_digest -c 1 -o $OUT/f_digest $P --radius 1.0 --fingerprint > $OUT/n3.log 2>&1
timeout 900 $NCU -k regex:onesweep_pass -s 3 -c 1 -o $OUT/f_sort $P --radius > $OUT/n4.log 2>&1
timeout 900 $NCU -k regex:"gather_soa|encode_kernel|bbox_kernel" -c 3 -o $OUT/f_reorder $P --radius > $OUT/n5.log 2>&1
timeout 900 $NCU -k regex:"open_count|open_emit|link_nodes|emit_tnodes|tnode" -c 7 -o $OUT/f_build $P --radius > $OUT/n6.log 2>&1
timeout 900 $NCU -k regex:knn_float_kernel -c 1 -o $OUT/f_knn16 $P --radius --k 16 > $OUT/n7.log 2>&1
timeout 900 $NCU -k regex:knn_float_kernel -c 1 -o $OUT/f_c1_knn64 python profiles/run_profile.py --config cfg1 --reps 1 --radius --k 64 > $OUT/n8.log 2>&1
timeout 900 $NCU -k regex:radius_pt_kernel -s 3 -c 1 -o $OUT/f_c1_count_r3 python profiles/run_profile.py --config cfg1 --reps 1 --radius 0.5 1.0 2.0 3.0 > $OUT/n9.log 2>&1
ls -la $OUT | tail -30
exit 0
