#!/bin/bash
OUT=gpurun_out/${1:-s16}
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_slabs.py tests/test_idiv.py tests/test_tc.py -x -q -k "slab" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
