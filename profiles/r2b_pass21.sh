#!/bin/bash
# row-major replay: rows per write pass 6 / 8 (vs 4 in-tree)
OUT=gpurun_out
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p21_radius.log 2>&1
  for v in r6 r8 r8b4; do LO_LIB_PATH=$PWD/_var/$v/liblinoct_b200.so timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p21_radius.log 2>&1; done
done
python - <<'PY'
import json
for l in open("gpurun_out/p21_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    print(d["config"], d["lib"][-28:], d["sha"] if d["config"] == "cfg3" else "", {k: v for k, v in d["ms"].items() if "fill" in k})
PY
exit 0
