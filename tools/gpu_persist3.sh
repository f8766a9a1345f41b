#!/bin/bash
OUT=gpurun_out/${1:-p03}
mkdir -p $OUT
for c in c1 c2 c3; do
  FOE_PERSIST_PHASES=1 timeout 300 python bench.py --config $c --solver persistent --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/phase_${c}.json 2> $OUT/phase_${c}.err; echo "phase $c rc=$?" >> $OUT/rc.txt
  grep "foe persistent" $OUT/phase_${c}.err >> $OUT/phases.txt
done
cat $OUT/phases.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
for c in c1 c2 c3; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_${c}.json 2> $OUT/bench_${c}.err; echo "bench $c rc=$?" >> $OUT/rc.txt
done
cat $OUT/rc.txt
