#!/bin/bash
# round 2 GPU pass 3: all GPU tests (new ones included) + the default bench
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=25 > $OUT/gputest3.log 2>&1; echo "pytest rc=$?" >> $OUT/gputest3.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench3.json 2> $OUT/bench3.err; echo "bench rc=$?" >> $OUT/bench3.err
tail -5 $OUT/gputest3.log
