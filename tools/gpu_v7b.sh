#!/bin/bash
OUT=gpurun_out/${1:-v7b}
mkdir -p $OUT
for r in 64 128 256; do
  FOE_K8_ROWS=$r timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_prior_grad_tc7 --csv --log-file $OUT/ab_$r.csv python tools/ab_k8.py 7 > $OUT/ncu_$r.log 2>&1; echo "rows $r rc=$?" >> $OUT/rc.txt
done
cat $OUT/rc.txt
