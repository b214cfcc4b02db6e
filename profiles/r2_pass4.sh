#!/bin/bash
# GPU pass 4: warp kNN + tile-local radius point tests: parity tests, scale kNN, bench
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fallbacks.py tests/test_gpu_fuzz.py tests/test_gpu_struct.py tests/test_gpu_locality.py -q -x > $OUT/t4a.log 2>&1; echo "pytest rc=$?" >> $OUT/t4a.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench4.json 2> $OUT/bench4.err; echo "bench rc=$?" >> $OUT/bench4.err
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "cfg1 or knn" > $OUT/t4b.log 2>&1; echo "pytest rc=$?" >> $OUT/t4b.log
tail -3 $OUT/t4a.log $OUT/t4b.log
