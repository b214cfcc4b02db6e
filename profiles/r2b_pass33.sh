#!/bin/bash
# walk knobs after the band / unroll changes: coarse node size and compact multiplier
OUT=gpurun_out
for c in cfg3 cfg1; do
  for co in 192 256 384; do
    LO_COARSE=$co timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p33_radius.log 2>&1
  done
  LO_COMPACT_MUL=4 timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p33_radius.log 2>&1
  LO_COMPACT_MUL=16 timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p33_radius.log 2>&1
done
python - <<'PY'
import json
for l in open("gpurun_out/p33_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    ms = d["ms"]
    tot = {}
    for k, v in ms.items():
        if "digest" in k: continue
        r = k.split("@")[1]
        tot[r] = round(tot.get(r, 0) + v, 3)
    print(d["config"], d["knobs"], "count+scan+fill:", tot)
PY
exit 0
