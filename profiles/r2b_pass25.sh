#!/bin/bash
# L2::64B gather loads: parity subset, per-stage DRAM traffic of one cfg3 step, default bench line
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_sort.py tests/test_gpu_scale.py -x -q > $OUT/p25_tests.log 2>&1; tail -2 $OUT/p25_tests.log
P="python profiles/run_profile.py --config cfg3 --reps 1 --radius 1.0 --fingerprint"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/p25_traffic_launches_cfg3.csv $P > $OUT/p25_ncu.log 2>&1; echo "ncu rc=$?"
timeout 1500 python bench.py > $OUT/p25_bench.json 2> $OUT/p25_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/p25_bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['extra']['cfg1']['ms_per_step'], {k: round(v,2) for k,v in d['stages_ms'].items()})"
exit 0
