#!/bin/bash
# step-time variance: per-call device times, stage sums and host times per bench step
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2 3; do
  timeout 600 python profiles/step_var_probe.py --steps 20 --blocks 3 > $OUT/sv23_$i.json 2> $OUT/sv23_$i.err
done
timeout 600 python profiles/step_var_probe.py --steps 20 --blocks 3 --timing 0 > $OUT/sv23_t0.json 2> $OUT/sv23_t0.err
exit 0
