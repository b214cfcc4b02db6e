#!/bin/bash
# digests with two rows per thread (interleaved FNV chains) vs one (LO_DIGEST_ONE_ROW=1)
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fallbacks.py -x -q > $OUT/p20_tests.log 2>&1; tail -2 $OUT/p20_tests.log
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p20_radius.log 2>&1
  LO_DIGEST_ONE_ROW=1 timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p20_radius.log 2>&1
done
python - <<'PY'
import json
for l in open("gpurun_out/p20_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    print(d["config"], d["knobs"], d["sha"], {k: v for k, v in d["ms"].items() if "digest" in k})
PY
exit 0
