#!/bin/bash
# concurrency experiment: tools/concur.py with each ab_libs variant
OUT=gpurun_out/${1:-concur}; mkdir -p $OUT
cp paper_1404_5344_b200/libfoe.so $OUT/orig.so.bak
for f in ab_libs/*.so; do n=$(basename $f .so); cp $f paper_1404_5344_b200/libfoe.so
  echo "== $n" >> $OUT/concur.log; timeout 600 python tools/concur.py >> $OUT/concur.log 2>&1
done
cp $OUT/orig.so.bak paper_1404_5344_b200/libfoe.so; cat $OUT/concur.log
