#!/bin/bash
# replay fill: next tile's records prefetched to L2 (in-tree) / L1 (_var/pfl1) / none (_var/nopf); 6 blocks; 2 rows
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_struct.py -x -q > $OUT/p11_tests.log 2>&1; tail -2 $OUT/p11_tests.log
for c in cfg3 cfg1; do
  timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p11_radius.log 2>&1
  for v in nopf pfl1 b6 r2; do
    LO_LIB_PATH=$PWD/_var/$v/liblinoct_b200.so timeout 300 python profiles/radius_probe.py --config $c >> $OUT/p11_radius.log 2>&1
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/p11_radius.log"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    print(d["config"], d["lib"].split("/")[-2] if "/" in d["lib"] else d["lib"], d["sha"], {k: v for k, v in d["ms"].items() if "fill" in k})
PY
exit 0
