#!/bin/bash
OUT=gpurun_out/r01b
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests/test_slabs.py -x -q > $OUT/pytest_slabs.log 2>&1; echo "slabs rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?" >> $OUT/rc.txt
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_inertial_prox -s 5 -c 1 \
  -o $OUT/k2 python bench.py --steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline > $OUT/ncu_k2.log 2>&1; echo "ncu-k2 rc=$?" >> $OUT/rc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
