#!/bin/bash
# Digest A/B: plain vs skew-gated length ranking (LO_DIGEST_SKEW percent), then the GPU suite with
# ranking forced on every imbalanced block (LO_DIGEST_SKEW=100) and with the default gate.
OUT=gpurun_out
for c in cfg3 cfg1 cfg4; do
  LO_DIGEST_PLAIN=1 timeout 600 python profiles/radius_probe.py --config $c --reps 3 >> $OUT/digest_skew.log 2>&1
  for p in 100 110 125 150; do
    LO_DIGEST_SKEW=$p timeout 600 python profiles/radius_probe.py --config $c --reps 3 >> $OUT/digest_skew.log 2>&1
  done
done
LO_DIGEST_SKEW=100 timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/gputest_skew100.log 2>&1; echo "pytest rc=$?" >> $OUT/gputest_skew100.log
exit 0
