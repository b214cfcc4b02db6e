#!/bin/bash
# step-time variance: host segments of lo_radius_range in slow steps
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2 3; do
  LO_DEBUG_HOST=1 timeout 600 python profiles/step_var_probe.py --steps 20 --blocks 3 --timing 0 > $OUT/sv24_$i.json 2> $OUT/sv24_$i.err
done
exit 0
