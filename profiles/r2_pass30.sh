#!/bin/bash
# bench stability after the e2e warm-up change and the copy-guard fix
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
for i in 1 2; do
LO_DEBUG_HOST=1 LO_DEBUG_ALLOC=1 timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/b30_$i.json 2> $OUT/b30_$i.err
done
exit 0
