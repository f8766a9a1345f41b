#!/bin/bash
# tall K8 tiles: parity tests, then the A/B of ab_libs on the c4 bench
OUT=gpurun_out/${1:-tall}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_tc.py -m gpu -q -x -k "tall or invalid or c4" > $OUT/pytest_tc.log 2>&1; echo "pytest tc rc=$?" >> $OUT/rc.txt
tail -3 $OUT/pytest_tc.log
bash tools/gpu_ablib.sh ${1:-tall}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c4" > $OUT/pytest_c4.log 2>&1; echo "pytest c4 rc=$?" >> $OUT/rc.txt
tail -3 $OUT/pytest_c4.log; cat $OUT/rc.txt
