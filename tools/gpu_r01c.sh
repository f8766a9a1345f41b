#!/bin/bash
OUT=gpurun_out/r01c
mkdir -p $OUT
timeout 300 python -m pytest tests/test_tc.py -x -q -k "energy_grad_parity" > $OUT/pytest_tc1.log 2>&1; echo "tc1 rc=$?" >> $OUT/rc.txt
timeout 900 python -m pytest tests/test_tc.py -q > $OUT/pytest_tc.log 2>&1; echo "tc rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
