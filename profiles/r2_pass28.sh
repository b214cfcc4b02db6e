#!/bin/bash
# kNN selection path: per-kernel times (ncu launch list, serialised) at cfg1 k=16 and k=64
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
for k in 16 64; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio --clock-control none -k regex:"knn_" --csv --log-file $OUT/l28_k$k.csv python profiles/knn_probe.py --config cfg1 --k $k --reps 1 --variants select > $OUT/l28_k$k.log 2>&1
done
exit 0
