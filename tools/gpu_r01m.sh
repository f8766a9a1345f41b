#!/bin/bash
OUT=gpurun_out/r01m
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/rc.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
timeout 600 python tools/e2e_breakdown.py > $OUT/e2e.log 2>&1; echo "e2e rc=$?" >> $OUT/rc.txt
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_inertial_prox -s 3 -c 1 \
  -o $OUT/k2 python bench.py --steps 1 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > $OUT/ncu_k2.log 2>&1; echo "ncu-k2 rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
