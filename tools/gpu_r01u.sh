#!/bin/bash
OUT=gpurun_out/r01u
mkdir -p $OUT
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -k "c3_P3 or c4_bench_launch" > $OUT/pytest_big.log 2>&1; echo "big rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
