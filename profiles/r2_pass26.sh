#!/bin/bash
# step-time variance after removing cudaMemGetInfo from the per-batch record setup
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2; do
  LO_DEBUG_HOST=1 timeout 600 python profiles/step_var_probe.py --steps 20 --blocks 3 --timing 0 > $OUT/sv26_$i.json 2> $OUT/sv26_$i.err
done
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra"
for i in 1 2 3; do
  echo "run $i $(timeout 600 $B 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), round(d["e2e"]["ms_per_step"],2), round(d["e2e_csr"]["ms_per_step"],1), d["e2e_knn"]["ms_per_step"] if "e2e_knn" in d else "")')" >> $OUT/var26.log
done
exit 0
