#!/bin/bash
OUT=gpurun_out/${1:-full2}
mkdir -p $OUT
for i in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$i.log 2>&1; echo "pytest $i rc=$?" >> $OUT/rc.txt
done
cat $OUT/rc.txt
