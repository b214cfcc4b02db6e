#!/bin/bash
# Parity campaign: 2000 small randomised clouds against the C restatement and 80 mid-size clouds
# (50k-400k points, Full mode) against the reference library itself.
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
LO_FUZZ_CASES=2000 LO_FUZZ_REF_CASES=80 timeout 3000 python -m pytest tests/test_gpu_fuzz.py -q -p no:randomly \
  --durations=5 > $OUT/fuzz_campaign.log 2>&1; echo "rc=$?" >> $OUT/fuzz_campaign.log
exit 0
