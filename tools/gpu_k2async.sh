#!/bin/bash
# K2 with cp.async prefetch of its inputs: K2 launch times, parity subset, c4 bench
OUT=gpurun_out/${1:-ka}
mkdir -p $OUT
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_inertial_prox -c 30 --csv --log-file $OUT/k2.csv python bench.py --steps 1 --warmup 1 --iters 10 --no-e2e --no-cpu-baseline > $OUT/ncu.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_slabs.py tests/test_idiv.py tests/test_persistent.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
