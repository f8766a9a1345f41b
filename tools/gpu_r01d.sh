#!/bin/bash
OUT=gpurun_out/r01f
mkdir -p $OUT
timeout 300 python -m pytest tests/test_tc.py -x -q  > $OUT/pytest_tc1.log 2>&1; echo "tc1 rc=$?" >> $OUT/rc.txt
timeout 300 python tools/prof_stencil.py > $OUT/prof.log 2>&1; echo "prof rc=$?" >> $OUT/rc.txt
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_prior_grad_tc -s 1 -c 1 \
  -o $OUT/k8 python tools/prof_stencil.py --stencil tensor --reps 1 > $OUT/ncu_k8.log 2>&1; echo "ncu rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
