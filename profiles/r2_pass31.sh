#!/bin/bash
# pipelined row digests: stage time + parity
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fallbacks.py -q -x > $OUT/t31.log 2>&1; echo "rc=$?" >> $OUT/t31.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-knn > $OUT/b31.json 2> $OUT/b31.err
exit 0
