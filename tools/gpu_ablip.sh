#!/bin/bash
# A/B of built libfoe variants (ab_libs/*.so) on the c4 Lipschitz setup, then the HVP /
# Lipschitz tests on the in-tree library
OUT=gpurun_out/${1:-ablip}; mkdir -p $OUT
cp paper_1404_5344_b200/libfoe.so $OUT/orig.so.bak
for rep in 1 2; do
  for f in ab_libs/*.so; do
    n=$(basename $f .so); cp $f paper_1404_5344_b200/libfoe.so
    echo "$n $rep $(timeout 300 python tools/lip_breakdown.py 4 2>&1 | tail -1)" >> $OUT/summary.txt
  done
done
cp $OUT/orig.so.bak paper_1404_5344_b200/libfoe.so
timeout 900 python -m pytest tests -m gpu -x -q -k "hvp or lipschitz" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
cat $OUT/summary.txt; tail -3 $OUT/pytest.log
