#!/bin/bash
# work-weighted shard bounds: GPU tests, then the per-rank critical path of equal vs weighted slices (cfg3, cfg1)
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_sort.py -x -q > $OUT/p14_tests.log 2>&1; tail -2 $OUT/p14_tests.log
timeout 900 python profiles/shard_balance.py --config cfg3 > $OUT/p14_balance_cfg3.json 2> $OUT/p14_balance_cfg3.err; tail -4 $OUT/p14_balance_cfg3.err
timeout 600 python profiles/shard_balance.py --config cfg1 > $OUT/p14_balance_cfg1.json 2> $OUT/p14_balance_cfg1.err; tail -4 $OUT/p14_balance_cfg1.err
exit 0
