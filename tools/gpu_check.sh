#!/bin/bash
# Tests + default bench of the current tree on one B200: tools/gpu_check.sh TAG
TAG=${1:-chk}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt; tail -3 $OUT/pytest.log; cat $OUT/bench.json
