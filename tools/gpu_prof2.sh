#!/bin/bash
# ncu --set full of the current K8 and K2 (c4 bench launch configuration), source-level
OUT=gpurun_out/${1:-prof2}; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_inertial_prox -s 2 -c 1 \
  -o $OUT/k2 python bench.py --steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline > $OUT/ncu_k2.log 2>&1; echo "ncu k2 rc=$?" >> $OUT/rc.txt
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_prior_grad_th -s 5 -c 1 \
  -o $OUT/k8 python bench.py --steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline > $OUT/ncu_k8.log 2>&1; echo "ncu k8 rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
