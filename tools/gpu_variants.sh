#!/bin/bash
OUT=gpurun_out/${1:-var}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_tc.py -q -k "schedule_variants" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
