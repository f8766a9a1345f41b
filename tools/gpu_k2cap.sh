#!/bin/bash
OUT=gpurun_out/${1:-k2c}
mkdir -p $OUT
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_inertial_prox -s 2 -c 1 \
  -o $OUT/k2 python bench.py --steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline > $OUT/ncu_k2.log 2>&1; echo "ncu-k2 rc=$?" >> $OUT/rc.txt
timeout 300 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_c1.json 2> $OUT/bench_c1.err; echo "bench c1 rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
