#!/bin/bash
OUT=gpurun_out/r01t
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "P2" > $OUT/pytest_p2.log 2>&1; echo "p2 rc=$?" >> $OUT/rc.txt
for c in c1 c2 c3; do
timeout 600 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?" >> $OUT/rc.txt
done
cat $OUT/rc.txt
