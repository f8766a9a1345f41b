#!/bin/bash
OUT=gpurun_out/r01j
mkdir -p $OUT
timeout 600 python -m pytest tests/test_tc.py -q > $OUT/pytest_tc.log 2>&1; echo "tc rc=$?" >> $OUT/rc.txt
timeout 300 python tools/prof_stencil.py > $OUT/prof.log 2>&1; echo "prof rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
