#!/bin/bash
# spin-waits at the library's host sync points: run-to-run variance of the bench main region
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra --no-knn"
for i in 1 2 3 4 5 6; do
  echo "run $i $(timeout 600 $B 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), round(d["e2e"]["ms_per_step"],2), round(d["e2e_csr"]["ms_per_step"],1))')" >> $OUT/var21.log
done
exit 0
