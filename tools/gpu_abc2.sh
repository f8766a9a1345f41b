#!/bin/bash
# A/B of ab_libs/*.so on a small config (default c2): tools/gpu_abc2.sh TAG CONFIG
OUT=gpurun_out/${1:-abc2}; C=${2:-c2}; mkdir -p $OUT
cp paper_1404_5344_b200/libfoe.so $OUT/orig.so.bak
for rep in 1 2; do for f in ab_libs/*.so; do n=$(basename $f .so); cp $f paper_1404_5344_b200/libfoe.so
  timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/$n.$rep.json 2> $OUT/$n.$rep.err
  python -c "import json; d=json.loads(open('$OUT/$n.$rep.json').read().strip().split(chr(10))[-1]); print('$n', $rep, round(d['value']), round(d['ms_per_step'],3), (d.get('k2') or {}).get('us_per_launch'))" >> $OUT/summary.txt
done; done
cp $OUT/orig.so.bak paper_1404_5344_b200/libfoe.so; cat $OUT/summary.txt
