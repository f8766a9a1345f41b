#!/bin/bash
# Round-end evidence, in parts that each bring back < 64 MiB of gpurun_out:
#   tools/gpu_final.sh TAG bench   smoke, bench lines (c4 default, c5 weak + strong, c1-c3, reference
#                                  arm, the Fig. 2 protocol), ncu launch list of the default bench
#   tools/gpu_final.sh TAG k8      ncu --set full of K8 and K2 (c4)
#   tools/gpu_final.sh TAG aux     ncu --set full of the K8h HVP (c4 setup) and the persistent kernel (c2)
TAG=${1:-final}; PART=${2:-bench}
OUT=gpurun_out/$TAG
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
if [ "$PART" = bench ]; then
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
for sc in weak strong; do
  timeout 900 python bench.py --config c5 --scaling $sc --steps 2 --warmup 3 > $OUT/bench_c5_$sc.json 2> $OUT/bench_c5_$sc.err; echo "bench c5 $sc rc=$?" >> $OUT/rc.txt
done
for c in c1 c2 c3; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?" >> $OUT/rc.txt
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "bench ref rc=$?" >> $OUT/rc.txt
timeout 300 python bench.py --protocol fig2 > $OUT/fig2.json 2> $OUT/fig2.err; echo "fig2 rc=$?" >> $OUT/rc.txt
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu-launch rc=$?" >> $OUT/rc.txt
elif [ "$PART" = k8 ]; then
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_prior_grad_th -s 5 -c 1 \
  -o $OUT/k8 python bench.py --steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline > $OUT/ncu_k8.log 2>&1; echo "ncu-k8 rc=$?" >> $OUT/rc.txt
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_inertial_prox -s 2 -c 1 \
  -o $OUT/k2 python bench.py --steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline > $OUT/ncu_k2.log 2>&1; echo "ncu-k2 rc=$?" >> $OUT/rc.txt
else
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_hvp_th -s 3 -c 1 \
  -o $OUT/hvp python bench.py --steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline > $OUT/ncu_hvp.log 2>&1; echo "ncu-hvp rc=$?" >> $OUT/rc.txt
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_ipiano_persistent -c 1 \
  -o $OUT/kp python bench.py --config c2 --steps 1 --warmup 1 --iters 20 --no-e2e --no-cpu-baseline > $OUT/ncu_kp.log 2>&1; echo "ncu-persistent rc=$?" >> $OUT/rc.txt
fi
cat $OUT/rc.txt
