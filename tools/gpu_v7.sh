#!/bin/bash
# K8 v7 (streamed u ring, R per problem): parity under FOE_K8_VARIANT=7, A/B vs v3, c4 bench
OUT=gpurun_out/${1:-v7}
mkdir -p $OUT
FOE_K8_VARIANT=7 timeout 900 python -m pytest tests/test_tc.py tests/test_gpu_parity.py -x -q -k "tc or TENSOR or tensor or c4_bench" > $OUT/pytest_v7.log 2>&1; echo "v7 tests rc=$?" >> $OUT/rc.txt
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_prior_grad_tc --csv --log-file $OUT/ab.csv python tools/ab_k8.py 3,7 > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/rc.txt
FOE_K8_VARIANT=7 timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_v7.json 2> $OUT/bench_v7.err; echo "bench v7 rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
