#!/bin/bash
# row digests fused into the replay fill vs the stand-alone digest pass (LO_DIGEST_SEPARATE=1)
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fallbacks.py tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_struct.py -x -q > $OUT/p15_tests.log 2>&1; tail -2 $OUT/p15_tests.log
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p15_radius.log 2>&1
  LO_DIGEST_SEPARATE=1 timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p15_radius.log 2>&1
done
python - <<'PY'
import json
for l in open("gpurun_out/p15_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    ms = d["ms"]
    tot = {}
    for k, v in ms.items():
        r = k.split("@")[1]
        tot[r] = round(tot.get(r, 0) + v, 3)
    print(d["config"], d["knobs"], d["sha"], "total:", tot, {k: v for k, v in ms.items() if "fill" in k or "digest" in k})
PY
exit 0
