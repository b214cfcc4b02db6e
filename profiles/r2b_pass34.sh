#!/bin/bash
# sort: one memset for the passes' tile counters
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_parity.py -x -q > $OUT/p34_tests.log 2>&1; tail -2 $OUT/p34_tests.log
for c in cfg1 cfg3 cfg1; do timeout 300 python profiles/sort_probe.py --config $c >> $OUT/p34_sort.log 2>&1; done
cat $OUT/p34_sort.log
exit 0
