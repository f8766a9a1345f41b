#!/bin/bash
# K8 fp16 bring-up: parity of the tensor-core stencil, then c4 timing of the new K8 vs the TF32 one
OUT=gpurun_out/${1:-h1}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_tc.py -x -q > $OUT/pytest_tc.log 2>&1; echo "pytest_tc rc=$?" >> $OUT/rc.txt
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_h.json 2> $OUT/bench_h.err; echo "bench h rc=$?" >> $OUT/rc.txt
FOE_K8_TF32=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_t.json 2> $OUT/bench_t.err; echo "bench t rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
