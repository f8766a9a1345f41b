#!/bin/bash
# Round-2 closing ncu captures (one B200): c4 K8 + K2 (tools/gpu_final.sh TAG k8), c3 K8 and K2
# (BASELINE configs[2] asks for per-kernel counters), each after its plain run exited 0
TAG=${1:-r2ncu}; OUT=gpurun_out/$TAG; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
tools/gpu_final.sh $TAG k8
C3="python bench.py --config c3 --steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 300 $C3 > $OUT/c3_plain.log 2>&1 && \
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_prior_grad_th -s 5 -c 1 \
  -o $OUT/c3_k8 $C3 > $OUT/ncu_c3_k8.log 2>&1; echo "ncu-c3-k8 rc=$?" >> $OUT/rc.txt
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_inertial_prox -s 5 -c 1 \
  -o $OUT/c3_k2 $C3 > $OUT/ncu_c3_k2.log 2>&1; echo "ncu-c3-k2 rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
