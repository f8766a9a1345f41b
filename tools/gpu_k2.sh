#!/bin/bash
OUT=gpurun_out/${1:-k2}
mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "P1 or P2 or (P3 and not c3)" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 300 python bench.py --steps 1 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > $OUT/plain.json 2>&1 && \
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_inertial_prox --csv --log-file $OUT/k2.csv python bench.py --steps 1 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
