#!/bin/bash
# kNN heap kernel residency: in-tree (ptxas free, 80 registers at k = 16) vs side builds with
# __launch_bounds__(128, 7) and (128, 8) (-DLO_KNN_MINB=7 / 8)
OUT=gpurun_out
for c in "cfg1 --k 8 16 32 64" "cfg3 --k 16"; do
  timeout 900 python profiles/knn_probe.py --config $c --reps 3 --variants heaps >> $OUT/knn_minb_ab.log 2>&1
  for m in 7 8; do
    LO_LIB_PATH=$PWD/_var/knnminb$m/liblinoct_b200.so timeout 900 python profiles/knn_probe.py --config $c --reps 3 --variants heaps >> $OUT/knn_minb_ab.log 2>&1
  done
done
exit 0
