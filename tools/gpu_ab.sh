#!/bin/bash
# In-process A/B of the K8 variants: plain timing, then kernel-only durations under ncu.
OUT=gpurun_out/${1:-ab}
mkdir -p $OUT
timeout 120 python -m pytest tests/test_tc.py -x -q -k "energy_grad_parity or slabs or P3" > $OUT/pytest_tc.log 2>&1; echo "tc rc=$?" >> $OUT/rc.txt
timeout 300 python tools/ab_k8.py > $OUT/plain.log 2>&1 && \
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_prior_grad_tc --csv --log-file $OUT/ab.csv python tools/ab_k8.py > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
