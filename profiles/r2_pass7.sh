#!/bin/bash
# GPU pass 7: 4-ary kNN key heaps (k >= 32): parity + bench
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fallbacks.py tests/test_gpu_fuzz.py -q -x > $OUT/t7.log 2>&1; echo "pytest rc=$?" >> $OUT/t7.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/b7.json 2> $OUT/b7.err
exit 0
