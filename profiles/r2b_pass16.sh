#!/bin/bash
# split fill / digest overlap vs fill-then-digest (LO_FILL_NO_SPLIT=1)
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fallbacks.py tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q > $OUT/p16_tests.log 2>&1; tail -2 $OUT/p16_tests.log
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p16_radius.log 2>&1
  LO_FILL_NO_SPLIT=1 timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p16_radius.log 2>&1
done
python - <<'PY'
import json
for l in open("gpurun_out/p16_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    ms = d["ms"]
    tot = {}
    for k, v in ms.items():
        r = k.split("@")[1]
        tot[r] = round(tot.get(r, 0) + v, 3)
    print(d["config"], d["knobs"], d["sha"], "total:", tot, {k: v for k, v in ms.items() if "fill" in k or "digest" in k})
PY
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-knn > $OUT/p16_bench.json 2> $OUT/p16_bench.err; echo bench $?
python -c "import json; d=json.load(open('gpurun_out/p16_bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['extra']['cfg1']['ms_per_step'], {k: round(v,2) for k,v in d['stages_ms'].items()})"
exit 0
