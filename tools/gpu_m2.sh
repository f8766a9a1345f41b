#!/bin/bash
OUT=gpurun_out/${1:-m2}; mkdir -p $OUT
timeout 600 python tools/setup_time.py > $OUT/setup_time.log 2>&1; tail -3 $OUT/setup_time.log
timeout 1200 python -m pytest tests/test_tc.py -m gpu -q -x > $OUT/pytest_tc.log 2>&1; echo "pytest tc rc=$?" >> $OUT/rc.txt
tail -3 $OUT/pytest_tc.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c4 or c3 or full_config or P1 or P2" > $OUT/pytest_par.log 2>&1; echo "pytest parity rc=$?" >> $OUT/rc.txt
tail -3 $OUT/pytest_par.log
bash tools/gpu_ablib.sh ${1:-m2}
cat $OUT/rc.txt
