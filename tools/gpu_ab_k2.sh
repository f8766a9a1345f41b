#!/bin/bash
# A/B of libfoe variants (ab_libs/*.so) on c4: bench value (twice, interleaved) and the K2 launch
# time from an ncu launch list (30 launches after warm-up)
OUT=gpurun_out/${1:-abk2}; CFG=${CFG:-c4}; KRE=${KRE:-k_inertial_prox}
mkdir -p $OUT
cp paper_1404_5344_b200/libfoe.so $OUT/orig.so.bak
for rep in 1 2; do
  for f in ab_libs/*.so; do
    n=$(basename $f .so)
    cp $f paper_1404_5344_b200/libfoe.so
    timeout 300 python bench.py --config $CFG --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/$n.$rep.json 2> $OUT/$n.$rep.err
    python -c "import json,sys; d=json.loads(open('$OUT/$n.$rep.json').read().strip().split(chr(10))[-1]); print('$n', $rep, round(d['value']), round(d['roofline']['k_ms_per_launch'],4), 'k2_us', round((d.get('k2') or {}).get('us_per_launch', 0),1))" >> $OUT/summary.txt
    if [ $rep = 1 ] && [ -n "$NCU_K2" ]; then
      timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$KRE -s 50 -c 30 --csv \
        --log-file $OUT/$n.k.csv python bench.py --config $CFG --steps 1 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > /dev/null 2>&1
      python tools/ncu_avg.py $OUT/$n.k.csv $n >> $OUT/summary.txt 2>&1 || true
    fi
  done
done
cp $OUT/orig.so.bak paper_1404_5344_b200/libfoe.so
cat $OUT/summary.txt
