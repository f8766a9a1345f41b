#!/bin/bash
# the FP32-FMA path (K1) on the c4 workload: bench line with --stencil ffma
OUT=gpurun_out/${1:-k1}
mkdir -p $OUT
timeout 900 python bench.py --stencil ffma --no-cpu-baseline --no-e2e > $OUT/bench_ffma.json 2> $OUT/bench_ffma.err; echo "bench ffma rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
