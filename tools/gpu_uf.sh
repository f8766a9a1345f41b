#!/bin/bash
# fp32 u slots (K2 writes u of the candidate, K8 stages from it) vs FOE_K8_UF=0: parity, c4 bench both ways
OUT=gpurun_out/${1:-uf}
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_tc.py tests/test_gpu_parity.py tests/test_idiv.py tests/test_edge_cases.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_uf.json 2> $OUT/bench_uf.err; echo "bench uf rc=$?" >> $OUT/rc.txt
FOE_K8_UF=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_w.json 2> $OUT/bench_w.err; echo "bench w rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
