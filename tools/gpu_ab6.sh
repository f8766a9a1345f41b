#!/bin/bash
# K8 v6 (three warp groups) vs v3: parity under FOE_K8_VARIANT=6, then in-process A/B timing
OUT=gpurun_out/${1:-ab6}
mkdir -p $OUT
FOE_K8_VARIANT=6 timeout 600 python -m pytest tests/test_tc.py tests/test_gpu_parity.py -x -q -k "tc or TENSOR or tensor or c4_bench" > $OUT/pytest_v6.log 2>&1; echo "v6 tests rc=$?" >> $OUT/rc.txt
timeout 300 python tools/ab_k8.py 3,6 > $OUT/plain.log 2>&1; echo "ab rc=$?" >> $OUT/rc.txt
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_prior_grad_tc --csv --log-file $OUT/ab.csv python tools/ab_k8.py 3,6 > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt; tail -5 $OUT/plain.log
