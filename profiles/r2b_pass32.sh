#!/bin/bash
# count pass: speculative point load at stack pop (in-tree) vs none (_var/old)
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fallbacks.py -x -q > $OUT/p32_tests.log 2>&1; tail -2 $OUT/p32_tests.log
for c in cfg3 cfg1; do
  for i in 1 2; do
    timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p32_radius.log 2>&1
    LO_LIB_PATH=$PWD/_var/old/liblinoct_b200.so timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p32_radius.log 2>&1
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/p32_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    print(d["config"], d["lib"][-28:], d["sha"] if d["config"] == "cfg3" else "", {k: v for k, v in d["ms"].items() if "count" in k})
PY
exit 0
