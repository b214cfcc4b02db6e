#!/bin/bash
# Final pass: smoke(), the whole GPU suite, the default bench line and the reference arm
OUT=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/fc_smoke.log 2>&1; tail -1 $OUT/fc_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $OUT/fc_gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/fc_gputest.log; tail -3 $OUT/fc_gputest.log
timeout 1500 python bench.py > $OUT/fc_bench.json 2> $OUT/fc_bench.err; echo "bench rc=$?"
timeout 1500 python bench.py --impl reference > $OUT/fc_ref.json 2> $OUT/fc_ref.err; echo "ref rc=$?"
exit 0
