#!/bin/bash
OUT=gpurun_out/${1:-kx}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_tc.py -x -q -k fused > $OUT/pytest_fused.log 2>&1; echo "fused test rc=$?" >> $OUT/rc.txt
for px in 16 32; do
  FOE_K2_PXT=$px timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_inertial_prox -c 40 --csv --log-file $OUT/k2_$px.csv python bench.py --steps 1 --warmup 1 --iters 10 --no-e2e --no-cpu-baseline > $OUT/ncu_$px.log 2>&1; echo "pxt $px rc=$?" >> $OUT/rc.txt
done
cat $OUT/rc.txt
