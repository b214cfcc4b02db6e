#!/bin/bash
# 16-point block boxes in the radius walk: stage times with and without, parity
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
for cfg in cfg3 cfg1 cfg4; do
  for b in 1 0; do
    LO_RADIUS_BLOCKS=$b timeout 900 python profiles/radius_probe.py --config $cfg --reps 2 >> $OUT/rp34.log 2>&1
  done
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fallbacks.py tests/test_gpu_fuzz.py -q -x > $OUT/t34.log 2>&1; echo "rc=$?" >> $OUT/t34.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra --no-knn --no-e2e > $OUT/b34.json 2> $OUT/b34.err
exit 0
