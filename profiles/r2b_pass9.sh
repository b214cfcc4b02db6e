#!/bin/bash
# walk knobs re-tuned after the point prefilter: coarse node size, replay row-major threshold
OUT=gpurun_out
for c in cfg3 cfg1; do
  for co in 64 128 256 32; do
    LO_COARSE=$co timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p9_radius.log 2>&1
  done
  LO_REPLAY_ROW_MAJOR_MIN=100 timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p9_radius.log 2>&1
  LO_REPLAY_ROW_MAJOR_MIN=20 timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p9_radius.log 2>&1
done
python - <<'PY'
import json
for l in open("gpurun_out/p9_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    ms = d["ms"]
    tot = {}
    for k, v in ms.items():
        r = k.split("@")[1]
        if "digest" not in k: tot[r] = round(tot.get(r, 0) + v, 3)
    print(d["config"], {k: v for k, v in d["knobs"].items()}, "count+scan+fill:", tot, {k: v for k, v in ms.items() if "count" in k or "fill" in k})
PY
exit 0
