#!/bin/bash
OUT=gpurun_out/${1:-p2}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "teacher_forced_P2_every_10" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
