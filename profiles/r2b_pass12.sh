#!/bin/bash
# count kernel occupancy shapes (warps per block x min blocks) and a persistent digest grid (LO_DIGEST_BPS)
OUT=gpurun_out
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p12_radius.log 2>&1
  for v in w8b4 w2b16 b7 b6; do
    LO_LIB_PATH=$PWD/_var/$v/liblinoct_b200.so timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p12_radius.log 2>&1
  done
  for bps in 4 8 16 32; do
    LO_DIGEST_BPS=$bps timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p12_radius.log 2>&1
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/p12_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    print(d["config"], d["lib"].split("/")[-2] if "/" in d["lib"] else d["lib"], d["knobs"].get("LO_DIGEST_BPS", ""), d["sha"] if d["config"] == "cfg3" else "",
          {k: v for k, v in d["ms"].items() if "count" in k or "digest" in k})
PY
exit 0
