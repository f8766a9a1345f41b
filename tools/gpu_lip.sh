#!/bin/bash
# Lipschitz setup breakdown (c4): plain timing, then the ncu launch list of the same command
OUT=gpurun_out/${1:-lip}; mkdir -p $OUT
timeout 300 python tools/lip_breakdown.py 3 > $OUT/plain.log 2>&1 && \
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python tools/lip_breakdown.py 1 > $OUT/ncu.log 2>&1
echo "rc=$?"; cat $OUT/plain.log | tail -2
