#!/bin/bash
# GPU pass 6: compressed count-pass records (160 B), split tnode boxes: parity + bench + cfg4 ablation
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fallbacks.py tests/test_gpu_struct.py tests/test_gpu_fuzz.py tests/test_gpu_async.py tests/test_cpp_shim.py -q -x > $OUT/t6.log 2>&1; echo "pytest rc=$?" >> $OUT/t6.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/b6.json 2> $OUT/b6.err
timeout 1200 python profiles/cfg4_ablation.py --out $OUT/cfg4_ablation.json > $OUT/cfg4.log 2>&1
timeout 1500 ncu --metrics lts__t_sector_hit_rate.pct,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"radius_pt_kernel|radius_replay|knn_float_kernel" --csv --log-file $OUT/cfg4_l2.csv python profiles/cfg4_ablation.py --searches-only > $OUT/cfg4_ncu.log 2>&1
exit 0
