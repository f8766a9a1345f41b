#!/bin/bash
OUT=gpurun_out/${1:-edge}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_edge_cases.py -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
