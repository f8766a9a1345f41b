#!/bin/bash
# K8 without row halos: parity (test_tc, c4/c3/c2 P3/P2 in test_gpu_parity), then A/B vs halo tiles
OUT=gpurun_out/${1:-nh}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_tc.py -m gpu -q -x > $OUT/pytest_tc.log 2>&1; echo "pytest tc rc=$?" >> $OUT/rc.txt
tail -3 $OUT/pytest_tc.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c4 or c3 or full_config or P1 or P2" > $OUT/pytest_par.log 2>&1; echo "pytest parity rc=$?" >> $OUT/rc.txt
tail -3 $OUT/pytest_par.log
bash tools/gpu_ablib.sh ${1:-nh}
cat $OUT/rc.txt
