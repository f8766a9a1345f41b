#!/bin/bash
OUT=gpurun_out/r01l
mkdir -p $OUT
timeout 900 python -m pytest tests/test_idiv.py -q > $OUT/pytest_idiv.log 2>&1; echo "idiv rc=$?" >> $OUT/rc.txt
timeout 600 python tools/e2e_breakdown.py > $OUT/e2e.log 2>&1; echo "e2e rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
