#!/bin/bash
OUT=gpurun_out/${1:-grp2}
mkdir -p $OUT
for g in 12 16 18 24; do
  timeout 120 python bench.py --config c2 --steps 3 --warmup 2 --filter-groups $g --no-cpu-baseline --no-e2e > $OUT/c2_g$g.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$OUT/c2_g$g.json').read().strip().splitlines()[-1])
print('c2 groups=$g', round(d['ms_per_step'],3))" >> $OUT/summary.txt 2>/dev/null
done
for g in 4 6 8 12; do
  timeout 120 python bench.py --config c3 --steps 3 --warmup 2 --filter-groups $g --no-cpu-baseline --no-e2e > $OUT/c3_g$g.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$OUT/c3_g$g.json').read().strip().splitlines()[-1])
print('c3 groups=$g', round(d['ms_per_step'],3))" >> $OUT/summary.txt 2>/dev/null
done
cat $OUT/summary.txt
