#!/bin/bash
OUT=gpurun_out/r01n
mkdir -p $OUT
timeout 120 python -m pytest tests/test_tc.py -x -q -k "energy_grad_parity" > $OUT/pytest_tc1.log 2>&1; echo "tc1 rc=$?" >> $OUT/rc.txt
timeout 300 python tools/prof_stencil.py --stencil tensor > $OUT/prof_v4.log 2>&1; echo "prof4 rc=$?" >> $OUT/rc.txt
FOE_K8_VARIANT=3 timeout 300 python tools/prof_stencil.py --stencil tensor > $OUT/prof_v3.log 2>&1; echo "prof3 rc=$?" >> $OUT/rc.txt
timeout 600 python -m pytest tests/test_tc.py tests/test_idiv.py tests/test_slabs.py -q > $OUT/pytest_tc.log 2>&1; echo "tc rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
