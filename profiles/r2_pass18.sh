#!/bin/bash
# big-buffer recycling: step variance + parity + bench main region
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
LO_DEBUG_ALLOC=1 timeout 900 python profiles/step_var_probe.py --config cfg3 --steps 12 > $OUT/var18.log 2> $OUT/var18.err
timeout 900 python profiles/gap_probe.py --config cfg3 --steps 8 > $OUT/gap18.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_struct.py tests/test_gpu_robustness.py tests/test_gpu_multirank.py tests/test_io.py -q -x > $OUT/t18.log 2>&1; echo "pytest rc=$?" >> $OUT/t18.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/b18.json 2> $OUT/b18.err
exit 0
