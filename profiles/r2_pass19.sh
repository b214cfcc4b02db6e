#!/bin/bash
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
LO_DEBUG_ALLOC=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra > $OUT/b19.json 2> $OUT/b19.err
timeout 900 python profiles/gap_probe.py --config cfg3 --steps 8 > $OUT/gap19.log 2>&1
exit 0
