#!/bin/bash
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra --no-knn --no-e2e"
for i in 1 2 3 4; do
  LO_BENCH_STEP_TIMES=1 LO_DEBUG_ALLOC=1 timeout 600 $B > $OUT/b22_$i.json 2> $OUT/b22_$i.err
done
exit 0
