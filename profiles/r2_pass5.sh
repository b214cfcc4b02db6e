#!/bin/bash
# GPU pass 5: digests on the aux stream vs inline at cfg3; ncu of the tile-local count kernel
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
A="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extra --no-knn"
timeout 600 $A > $OUT/b5_inline.json 2> $OUT/b5_inline.err
LO_DIGEST_AUX=1 timeout 600 $A > $OUT/b5_aux.json 2> $OUT/b5_aux.err
P="python profiles/run_profile.py --config cfg3 --reps 1"
timeout 600 $P --radius 1.0 > $OUT/prof5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radius_pt_kernel -c 1 -o $OUT/c3_count_local $P --radius 1.0 > $OUT/ncu5a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tnode_boxes -c 1 -o $OUT/c3_tnode $P --radius > $OUT/ncu5b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:encode_kernel -c 1 -o $OUT/c3_encode $P --radius > $OUT/ncu5c.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fallbacks.py -q -x > $OUT/t5.log 2>&1; echo "pytest rc=$?" >> $OUT/t5.log
exit 0
