#!/bin/bash
# Encode blocks per SM A/B (LO_ENCODE_PER_SM), cfg3 and cfg1 stage tables from short bench runs.
OUT=gpurun_out
B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-knn --no-extra"
for c in cfg3 cfg1; do
  for p in 4 5 6 8; do
    LO_ENCODE_PER_SM=$p timeout 600 $B --config $c > $OUT/enc_${c}_${p}.json 2>/dev/null
    python - $c $p <<'PY' >> $OUT/encode_ab.log
import json, sys
c, p = sys.argv[1], sys.argv[2]
d = json.load(open(f"gpurun_out/enc_{c}_{p}.json"))
print(json.dumps({"config": c, "per_sm": int(p), "ms_per_step": round(d["ms_per_step"], 3),
                  "stages_ms": {k: round(v, 3) for k, v in d["stages_ms"].items()}}))
PY
  done
done
exit 0
