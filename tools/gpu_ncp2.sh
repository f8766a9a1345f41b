#!/bin/bash
OUT=gpurun_out/${1:-ncp2}
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_persistent.py tests/test_gpu_parity.py tests/test_idiv.py tests/test_slabs.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
for c in c1 c2 c3; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?" >> $OUT/rc.txt
done
cat $OUT/rc.txt
