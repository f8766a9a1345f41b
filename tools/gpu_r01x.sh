#!/bin/bash
# Final round-1 evidence: launch list of the default bench command, full captures of K8 (v4) and K2.
OUT=gpurun_out/r01x
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 900 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/plain.json 2> $OUT/plain.err && \
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu-launch rc=$?" >> $OUT/rc.txt
timeout 600 python bench.py --steps 1 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > $OUT/plain20.json 2>&1 && \
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_prior_grad_tc4 -s 45 -c 1 \
  -o $OUT/k8 python bench.py --steps 1 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > $OUT/ncu_k8.log 2>&1; echo "ncu-k8 rc=$?" >> $OUT/rc.txt
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_inertial_prox -s 3 -c 1 \
  -o $OUT/k2 python bench.py --steps 1 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > $OUT/ncu_k2.log 2>&1; echo "ncu-k2 rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
