#!/bin/bash
# GPU pass 8: keyed kNN as sorted list + pending merges: parity + bench kNN
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fallbacks.py tests/test_gpu_fuzz.py tests/test_gpu_locality.py -q -x > $OUT/t8.log 2>&1; echo "pytest rc=$?" >> $OUT/t8.log
timeout 900 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > $OUT/b8.json 2> $OUT/b8.err
exit 0
