#!/bin/bash
# persistent driver: K1 chunk size x filter groups on c2 and c3 (per-iteration time)
OUT=gpurun_out/${1:-grp}
mkdir -p $OUT
for c in c2 c3; do
  for ncp in 1 2; do
    for g in 0 2 3 4 6 8 9 12; do
      FOE_K1_NCP=$ncp timeout 120 python bench.py --config $c --steps 3 --warmup 2 --filter-groups $g --no-cpu-baseline --no-e2e > $OUT/${c}_n${ncp}_g${g}.json 2>/dev/null
      python -c "
import json
d=json.loads(open('$OUT/${c}_n${ncp}_g${g}.json').read().strip().splitlines()[-1])
print('$c ncp=$ncp groups=$g', round(d['ms_per_step'],3))" >> $OUT/summary.txt 2>/dev/null
    done
  done
done
cat $OUT/summary.txt
