#!/bin/bash
# small-image configs: default (AUTO) vs forced graph + K8 (tensor) for c2 / c3
OUT=gpurun_out/${1:-c3}
mkdir -p $OUT
for c in c3 c2; do
  for v in "auto auto" "graph tensor"; do
    set -- $v
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --solver $1 --stencil $2 > $OUT/$c.$1.json 2> $OUT/$c.$1.err
    python -c "import json; d=json.loads(open('$OUT/$c.$1.json').read().strip().split(chr(10))[-1]); print('$c', '$1 $2', round(d['value']), round(d['ms_per_step'],3), d['roofline'].get('k_ms_per_launch'))" >> $OUT/summary.txt 2>&1
  done
done
cat $OUT/summary.txt
