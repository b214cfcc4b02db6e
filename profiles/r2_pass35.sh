#!/bin/bash
# e2e phases at cfg3: what the e2e step adds to the device step
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 600 python profiles/e2e_phases.py --config cfg3 --steps 10 > $OUT/ph35_all.log 2>&1
timeout 600 python profiles/e2e_phases.py --config cfg3 --steps 10 --no-dl > $OUT/ph35_nodl.log 2>&1
timeout 600 python profiles/e2e_phases.py --config cfg3 --steps 10 --no-h2d > $OUT/ph35_noh2d.log 2>&1
timeout 600 python profiles/e2e_phases.py --config cfg3 --steps 10 --no-h2d --no-dl > $OUT/ph35_none.log 2>&1
exit 0
