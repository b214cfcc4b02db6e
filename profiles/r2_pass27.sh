#!/bin/bash
# kNN selection path: GPU tests, timings vs the heaps; step variance after the record-setup fix
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fallbacks.py -q -x -k "knn" > $OUT/t27_knn.log 2>&1; echo "rc=$?" >> $OUT/t27_knn.log
LO_DEBUG=1 timeout 900 python profiles/knn_probe.py --config cfg1 --variants select heaps win2 cap16 > $OUT/kp27_cfg1.json 2> $OUT/kp27_cfg1.err
LO_DEBUG=1 timeout 900 python profiles/knn_probe.py --config cfg3 --reps 2 --variants select heaps > $OUT/kp27_cfg3.json 2> $OUT/kp27_cfg3.err
LO_DEBUG_HOST=1 timeout 600 python profiles/step_var_probe.py --steps 20 --blocks 3 --timing 0 > $OUT/sv27.json 2> $OUT/sv27.err
exit 0
