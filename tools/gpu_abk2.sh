#!/bin/bash
# A/B of ab_libs on the c4 bench with the K2 time: tools/gpu_abk2.sh TAG
OUT=gpurun_out/${1:-abk2}; mkdir -p $OUT
cp paper_1404_5344_b200/libfoe.so $OUT/orig.so.bak
for rep in 1 2; do for f in ab_libs/*.so; do n=$(basename $f .so); cp $f paper_1404_5344_b200/libfoe.so
  timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/$n.$rep.json 2> $OUT/$n.$rep.err
  python -c "import json; d=json.loads(open('$OUT/$n.$rep.json').read().strip().split(chr(10))[-1]); print('$n', $rep, round(d['value']), round(d['roofline']['k_ms_per_launch'],4), round(d['k2']['us_per_launch'],1))" >> $OUT/summary.txt
done; done
cp $OUT/orig.so.bak paper_1404_5344_b200/libfoe.so; cat $OUT/summary.txt
