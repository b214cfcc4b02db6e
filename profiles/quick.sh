#!/bin/bash
# quick GPU check: gpu tests + a short bench (radius only), prints the stage table
timeout 700 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${KNN:---no-knn} > gpurun_out/q.json 2> gpurun_out/q.err
tail -3 gpurun_out/q.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/q.json"))
print(round(d["ms_per_step"], 3), {k: round(v, 3) for k, v in d["stages_ms"].items()})
if "knn" in d and d["knn"]:
    print({k: round(v["ms"], 2) for k, v in d["knn"].items()})
PY
