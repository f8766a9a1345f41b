#!/bin/bash
OUT=gpurun_out/${1:-pk2}
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_slabs.py tests/test_tc.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu-launch rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
