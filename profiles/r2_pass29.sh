#!/bin/bash
# e2e variance: slow host calls and allocations inside the e2e timed regions
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
for i in 1 2 3; do
LO_DEBUG_HOST=1 LO_DEBUG_ALLOC=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra > $OUT/b29_$i.json 2> $OUT/b29_$i.err
done
exit 0
