#!/bin/bash
# One GPU session: parity tests, the bench line, the ncu launch list and full captures of K1/K2.
# Usage (from the repo root, on the GPU box):  bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/rc.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu-launch rc=$?" >> $OUT/rc.txt
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_prior_grad2 -s 40 -c 1 \
  -o $OUT/k1 python bench.py --steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline > $OUT/ncu_k1.log 2>&1; echo "ncu-k1 rc=$?" >> $OUT/rc.txt
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_inertial_prox -s 40 -c 1 \
  -o $OUT/k2 python bench.py --steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline > $OUT/ncu_k2.log 2>&1; echo "ncu-k2 rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
