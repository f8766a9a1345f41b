#!/bin/bash
# quick K8 parity subset + default bench line
OUT=gpurun_out/${1:-q}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_tc.py tests/test_slabs.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
