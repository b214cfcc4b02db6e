#!/bin/bash
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python profiles/pipeline_probe.py --config cfg3 --steps 10 > $OUT/pipe12.log 2>&1
timeout 600 python profiles/pipeline_probe.py --config cfg1 --steps 20 >> $OUT/pipe12.log 2>&1
exit 0
