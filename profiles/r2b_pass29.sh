#!/bin/bash
# count pass: mask zeroing skipped on the all-interested path (in-tree), + no per-query leaf test (_var/nowant), vs HEAD (_var/old)
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > $OUT/p29_tests.log 2>&1; tail -2 $OUT/p29_tests.log
LO_LIB_PATH=$PWD/_var/nowant/liblinoct_b200.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > $OUT/p29_tests_nowant.log 2>&1; tail -2 $OUT/p29_tests_nowant.log
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p29_radius.log 2>&1
  for v in old nowant; do LO_LIB_PATH=$PWD/_var/$v/liblinoct_b200.so timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p29_radius.log 2>&1; done
done
python - <<'PY'
import json
for l in open("gpurun_out/p29_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    print(d["config"], d["lib"][-30:], d["sha"] if d["config"] == "cfg3" else "", {k: v for k, v in d["ms"].items() if "count" in k or "fill" in k})
PY
exit 0
