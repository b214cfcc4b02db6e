#!/bin/bash
# segment replay (shared window + coalesced writeout) vs row-major / buffer-major replay
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fallbacks.py tests/test_gpu_struct.py tests/test_gpu_sort.py -x -q > $OUT/p8_tests.log 2>&1; tail -2 $OUT/p8_tests.log
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p8_radius.log 2>&1
  LO_REPLAY_NO_SEG=1 timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p8_radius.log 2>&1
  for v in seg2k seg4k; do
    LO_LIB_PATH=$PWD/_var/$v/liblinoct_b200.so timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p8_radius.log 2>&1
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/p8_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    print(d["config"], d["lib"].split("/")[-2] if "/" in d["lib"] else d["lib"], d["knobs"].get("LO_REPLAY_NO_SEG", ""), d["sha"],
          {k: v for k, v in d["ms"].items() if "fill" in k or "count" in k})
PY
exit 0
