#!/bin/bash
# Round-1 evidence run: GPU tests, c4 + c5 bench lines, launch list, K8 and K2 full captures.
OUT=gpurun_out/r01k
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/rc.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?" >> $OUT/rc.txt
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu-launch rc=$?" >> $OUT/rc.txt
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_prior_grad_tc -s 45 -c 1 \
  -o $OUT/k8 python bench.py --steps 1 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > $OUT/ncu_k8.log 2>&1; echo "ncu-k8 rc=$?" >> $OUT/rc.txt
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_inertial_prox -s 3 -c 1 \
  -o $OUT/k2 python bench.py --steps 1 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > $OUT/ncu_k2.log 2>&1; echo "ncu-k2 rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
