#!/bin/bash
# per-launch DRAM bytes of every kernel of one cfg3 step (stage traffic for roofline.stages)
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
P="python profiles/run_profile.py --config cfg3 --reps 1 --radius 1.0 --fingerprint"
timeout 600 $P > $OUT/p32_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/traffic_launches_cfg3.csv $P > $OUT/p32_ncu.log 2>&1
exit 0
