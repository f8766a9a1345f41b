#!/bin/bash
OUT=gpurun_out/${1:-ncp}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
for c in c1 c2; do
  FOE_PERSIST_PHASES=1 timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?" >> $OUT/rc.txt
  grep "foe persistent" $OUT/bench_$c.err | tail -1 >> $OUT/phases.txt
done
cat $OUT/rc.txt $OUT/phases.txt
