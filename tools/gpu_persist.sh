#!/bin/bash
# persistent small-image driver: tests + c1/c2/c3 bench lines, both drivers
OUT=gpurun_out/${1:-p01}
mkdir -p $OUT
python -c "import paper_1404_5344_b200 as P; P.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_persistent.py -x -q > $OUT/pytest_persist.log 2>&1; echo "persist rc=$?" >> $OUT/rc.txt
for c in c1 c2 c3; do
  for s in graph persistent; do
    timeout 300 python bench.py --config $c --solver $s --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_${c}_${s}.json 2> $OUT/bench_${c}_${s}.err; echo "bench $c $s rc=$?" >> $OUT/rc.txt
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_idiv.py -x -q -k "P3 or batch or workspace or host_and_device" > $OUT/pytest_p3.log 2>&1; echo "p3 rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
