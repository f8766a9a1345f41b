#!/bin/bash
# K8 column packing + the shared K2 pixel function: K8/K2 parity suites, then the c4 bench line
OUT=gpurun_out/${1:-pk}
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_tc.py tests/test_gpu_parity.py tests/test_slabs.py tests/test_idiv.py tests/test_persistent.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_prior_grad_tc|k_inertial_prox" -c 12 --csv --log-file $OUT/k.csv python tools/prof_stencil.py --stencil tensor --reps 2 > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
