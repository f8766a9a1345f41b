#!/bin/bash
# ncu launch list of the c5 (8192^2 row slab) bench command
OUT=gpurun_out/${1:-c5l}
mkdir -p $OUT
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5.csv \
  python bench.py --config c5 --steps 1 --warmup 1 --iters 10 --no-cpu-baseline > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
