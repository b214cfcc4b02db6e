#!/bin/bash
# Parity campaign with the final round-2 kernels: 10,000 small randomised clouds against the C restatement
# and 400 mid-size clouds (50k-400k points, Full mode) against the reference library.
OUT=gpurun_out
LO_FUZZ_CASES=10000 LO_FUZZ_REF_CASES=400 timeout 3000 python -m pytest tests/test_gpu_fuzz.py -q -p no:randomly \
  --durations=5 > $OUT/r2b_fuzz_campaign.log 2>&1; echo "rc=$?" >> $OUT/r2b_fuzz_campaign.log
tail -3 $OUT/r2b_fuzz_campaign.log
exit 0
