#!/bin/bash
# does nvidia-smi polling during the timed region slow the step?
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra --no-e2e --no-knn"
for ms in 25 0 100 25 0 200; do
  echo "clock_ms=$ms $(LO_BENCH_CLOCK_MS=$ms timeout 600 $B 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), d["clocks"]["samples"])')" >> $OUT/clk20.log
done
exit 0
