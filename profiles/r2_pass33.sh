#!/bin/bash
# nearest-first seed windows for the kNN heaps: timings + parity
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 900 python profiles/knn_probe.py --config cfg1 --variants heaps near > $OUT/kp33_cfg1.json 2> $OUT/kp33_cfg1.err
timeout 900 python profiles/knn_probe.py --config cfg3 --reps 2 --variants heaps near > $OUT/kp33_cfg3.json 2> $OUT/kp33_cfg3.err
timeout 900 python -m pytest tests/test_gpu_fallbacks.py tests/test_gpu_parity.py -q -x -k "knn" > $OUT/t33.log 2>&1; echo "rc=$?" >> $OUT/t33.log
exit 0
