#!/bin/bash
# GPU pass 10: PACK/VAL sort passes + re-encoding gather: parity, sort probe, bench
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for c in cfg3 cfg1; do timeout 300 python profiles/sort_probe.py --config $c >> $OUT/sort10.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_io.py tests/test_gpu_fuzz.py tests/test_gpu_struct.py tests/test_cpp_shim.py -q -x > $OUT/t10.log 2>&1; echo "pytest rc=$?" >> $OUT/t10.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "cfg1 or structure" > $OUT/t10b.log 2>&1; echo "pytest rc=$?" >> $OUT/t10b.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/b10.json 2> $OUT/b10.err
exit 0
