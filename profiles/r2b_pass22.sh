#!/bin/bash
# Struct radius: leaf-point tile-box prefilter (in-tree) vs none (_var/old)
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_struct.py tests/test_gpu_fuzz.py -x -q > $OUT/p22_tests.log 2>&1; tail -2 $OUT/p22_tests.log
for c in cfg1 cfg3; do
  timeout 600 python profiles/struct_probe.py --config $c --reps 2 2>/dev/null | tail -1 >> $OUT/p22_struct.log
  LO_LIB_PATH=$PWD/_var/old/liblinoct_b200.so timeout 600 python profiles/struct_probe.py --config $c --reps 2 2>/dev/null | tail -1 >> $OUT/p22_struct.log
done
python - <<'PY'
import json
for l in open("gpurun_out/p22_struct.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    print(d["config"], {r: (round(v["struct_ms"], 2), round(v["lin_ms"], 2), v["ranges"], v["singles"]) for r, v in d["struct"].items()})
PY
exit 0
