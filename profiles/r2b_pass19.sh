#!/bin/bash
# FNV byte step in 32-bit halves (mul.wide + 2 mad.lo) vs the 64-bit multiply (_var/old)
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_struct.py tests/test_gpu_fallbacks.py tests/test_gpu_scale.py -x -q > $OUT/p19_tests.log 2>&1; tail -2 $OUT/p19_tests.log
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p19_radius.log 2>&1
  LO_LIB_PATH=$PWD/_var/old/liblinoct_b200.so timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p19_radius.log 2>&1
done
timeout 600 python profiles/knn_probe.py --config cfg1 --k 8 16 --variants heaps >> $OUT/p19_knn.log 2>&1
LO_LIB_PATH=$PWD/_var/old/liblinoct_b200.so timeout 600 python profiles/knn_probe.py --config cfg1 --k 8 16 --variants heaps >> $OUT/p19_knn.log 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/p19_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    print(d["config"], d["lib"][-30:], d["sha"], {k: v for k, v in d["ms"].items() if "digest" in k})
for l in open("gpurun_out/p19_knn.log"):
    if l.startswith("{"): d = json.loads(l); print(d["lib"][-30:], d["ms"], d["fps_xor"])
PY
exit 0
