#!/bin/bash
# one ncu --set full capture of the default K8 launch (c4 batch) with source-level counters
OUT=gpurun_out/${1:-n01}
mkdir -p $OUT
timeout 300 python tools/prof_stencil.py --stencil tensor --reps 2 > $OUT/prof.log 2>&1; echo "prof rc=$?" >> $OUT/rc.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_prior_grad_tc -c 1 -o $OUT/k8 python tools/prof_stencil.py --stencil tensor --reps 1 > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
