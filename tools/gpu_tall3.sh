#!/bin/bash
OUT=gpurun_out/${1:-tall3}; mkdir -p $OUT
bash tools/gpu_ablib.sh ${1:-tall3}
cp paper_1404_5344_b200/libfoe.so $OUT/def.so.bak
for v in r256 r64; do
cp ab_libs/$v.so paper_1404_5344_b200/libfoe.so
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_prior_grad_th -s 5 -c 1 \
  -o $OUT/k8_$v python bench.py --steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline > $OUT/ncu_$v.log 2>&1; echo "ncu $v rc=$?" >> $OUT/rc.txt
done
cp $OUT/def.so.bak paper_1404_5344_b200/libfoe.so
cat $OUT/rc.txt
