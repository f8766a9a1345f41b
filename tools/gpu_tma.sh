#!/bin/bash
OUT=gpurun_out/${1:-tma}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_tc.py tests/test_slabs.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_prior_grad_tc --csv --log-file $OUT/k8.csv python tools/ab_k8.py 3 > $OUT/k8.log 2>&1; echo "ncu rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
