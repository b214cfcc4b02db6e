#!/bin/bash
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
LO_DEBUG_ALLOC=1 timeout 900 python profiles/gap_probe.py --config cfg3 --steps 8 > $OUT/gap15.log 2> $OUT/gap15.err
exit 0
