#!/bin/bash
OUT=gpurun_out/${1:-ab5v}
mkdir -p $OUT
FOE_K8_VARIANT=5 timeout 180 python -m pytest tests/test_tc.py -x -q -k "energy_grad_parity or slabs or P3 or c4" > $OUT/pytest_v5.log 2>&1; echo "tc5 rc=$?" >> $OUT/rc.txt
timeout 300 python tools/ab_k8.py 4,5 > $OUT/plain.log 2>&1 && \
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_prior_grad_tc --csv --log-file $OUT/ab.csv python tools/ab_k8.py 4,5 > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
