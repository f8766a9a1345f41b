#!/bin/bash
OUT=gpurun_out/r01r
mkdir -p $OUT
timeout 120 python -m pytest tests/test_tc.py -x -q -k "energy_grad_parity or slabs or P3" > $OUT/pytest_tc1.log 2>&1; echo "tc1 rc=$?" >> $OUT/rc.txt
for i in 1 2; do
timeout 300 python tools/prof_stencil.py --stencil tensor > $OUT/prof_v4_$i.log 2>&1; echo "prof4 rc=$?" >> $OUT/rc.txt
FOE_K8_VARIANT=3 timeout 300 python tools/prof_stencil.py --stencil tensor > $OUT/prof_v3_$i.log 2>&1; echo "prof3 rc=$?" >> $OUT/rc.txt
done
cat $OUT/rc.txt
