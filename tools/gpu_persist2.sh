#!/bin/bash
OUT=gpurun_out/${1:-p02}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_persistent.py -x -q > $OUT/pytest_persist.log 2>&1; echo "persist rc=$?" >> $OUT/rc.txt
for c in c1 c2 c3; do
  FOE_PERSIST_PHASES=1 timeout 300 python bench.py --config $c --solver persistent --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/phase_${c}.json 2> $OUT/phase_${c}.err; echo "phase $c rc=$?" >> $OUT/rc.txt
  grep "foe persistent" $OUT/phase_${c}.err >> $OUT/phases.txt
done
cat $OUT/rc.txt $OUT/phases.txt
