#!/bin/bash
# fused trial kernel (K2 inside K8, FOE_FUSE_K2=1): parity suites under fusion, then the c4
# bench line with and without fusion
OUT=gpurun_out/${1:-fz}
mkdir -p $OUT
FOE_FUSE_K2=1 timeout 1200 python -m pytest tests/test_tc.py tests/test_gpu_parity.py -x -q -k "tc or TENSOR or tensor or c4_bench or batch or workspace" > $OUT/pytest_fused.log 2>&1; echo "pytest fused rc=$?" >> $OUT/rc.txt
FOE_FUSE_K2=1 timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_fused.json 2> $OUT/bench_fused.err; echo "bench fused rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_plain.json 2> $OUT/bench_plain.err; echo "bench plain rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
