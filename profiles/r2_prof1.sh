#!/bin/bash
# round 2 GPU pass 2: new parity tests, compute-sanitizer, cfg3 launch list + --set full captures
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fallbacks.py tests/test_gpu_robustness.py tests/test_gpu_scale.py -x -q --durations=12 > $OUT/newtests.log 2>&1; echo "pytest rc=$?" >> $OUT/newtests.log
for tool in racecheck memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python profiles/san_small.py > $OUT/san_$tool.log 2>&1; echo "rc=$?" >> $OUT/san_$tool.log
done
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn --no-extra > $OUT/b_small.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_cfg3.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn --no-extra > $OUT/ncu_launch.log 2>&1
P="python profiles/run_profile.py --config cfg3 --reps 1"
timeout 600 $P --radius 1.0 --k 16 --fingerprint > $OUT/prof_plain.log 2>&1 || exit 1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:radius_pt_kernel -c 1 -o $OUT/c3_count $P --radius 1.0 > $OUT/ncu1.log 2>&1
timeout 900 $NCU -k regex:radius_replay -c 1 -o $OUT/c3_fill $P --radius 1.0 > $OUT/ncu2.log 2>&1
timeout 900 $NCU -k regex:radius_digest -c 1 -o $OUT/c3_digest $P --radius 1.0 --fingerprint > $OUT/ncu3.log 2>&1
timeout 900 $NCU -k regex:onesweep_pass -c 2 -o $OUT/c3_sort $P --radius > $OUT/ncu4.log 2>&1
timeout 900 $NCU -k regex:"gather_soa|encode_kernel|bbox" -c 3 -o $OUT/c3_reorder $P --radius > $OUT/ncu5.log 2>&1
timeout 900 $NCU -k regex:"open_count|open_emit|link_nodes|emit_tnodes|tnode" -c 8 -o $OUT/c3_build $P --radius > $OUT/ncu6.log 2>&1
timeout 900 $NCU -k regex:knn_float_kernel -c 1 -o $OUT/c3_knn16 $P --radius --k 16 > $OUT/ncu7.log 2>&1
timeout 900 $NCU -k regex:knn_float_kernel -c 1 -o $OUT/c1_knn64 python profiles/run_profile.py --config cfg1 --reps 1 --radius --k 64 > $OUT/ncu8.log 2>&1
ls -la $OUT
