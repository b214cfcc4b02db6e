#!/bin/bash
# coarse-node size sweep (continued) with the point prefilter
OUT=gpurun_out
for c in cfg3 cfg1 cfg4; do
  for co in 256 512 1024 2048; do
    LO_COARSE=$co timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p10_radius.log 2>&1
  done
  LO_COARSE=512 LO_COMPACT_MUL=16 timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p10_radius.log 2>&1
done
python - <<'PY'
import json
for l in open("gpurun_out/p10_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    ms = d["ms"]
    print(d["config"], d["knobs"], {k: v for k, v in ms.items() if "count" in k or "fill" in k})
PY
exit 0
