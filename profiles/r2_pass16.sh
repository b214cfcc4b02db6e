#!/bin/bash
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python profiles/step_var_probe.py --config cfg3 --steps 16 > $OUT/var16.log 2>&1
timeout 900 python profiles/step_var_probe.py --config cfg3 --steps 16 >> $OUT/var16.log 2>&1
exit 0
