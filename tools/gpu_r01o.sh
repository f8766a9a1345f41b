#!/bin/bash
OUT=gpurun_out/r01v
mkdir -p $OUT
timeout 300 python tools/prof_stencil.py --stencil tensor --reps 1 > $OUT/plain.log 2>&1 && \
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_prior_grad_tc -s 1 -c 1 \
  -o $OUT/k8v3 python tools/prof_stencil.py --stencil tensor --reps 1 > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
