#!/bin/bash
# gather record-load variants, second set: nc + L2::64B (ld5), L2::64B (ld6), nc + L2::128B (ld7)
OUT=gpurun_out
for v in in-tree ld5 ld6 ld7; do
  if [ $v = in-tree ]; then E=""; else E="LO_LIB_PATH=$PWD/_var/$v/liblinoct_b200.so"; fi
  env $E timeout 300 python profiles/sort_probe.py --config cfg3 >> $OUT/p24_sort.log 2>&1
  env $E timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gather_soa -c 1 --csv \
     python profiles/sort_probe.py --config cfg3 --reps 0 2>/dev/null | grep -E "dram__bytes|gpu__time" | sed "s/^/$v /" >> $OUT/p24_ncu.log
done
exit 0
