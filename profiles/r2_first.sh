#!/bin/bash
# round 2, first GPU pass: host facts, GPU tests, the default bench (cfg3) and the reference arm
OUT=gpurun_out
nproc > $OUT/host.txt; free -g >> $OUT/host.txt; lscpu >> $OUT/host.txt; nvidia-smi >> $OUT/host.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/gputest.log
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/ref.err
tail -2 $OUT/gputest.log; tail -2 $OUT/bench.err; tail -1 $OUT/ref.err
