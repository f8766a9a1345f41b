#!/bin/bash
# stored-S HVPs: Lipschitz/HVP parity, smoke, then the setup time of both builds
OUT=gpurun_out/${1:-hvps}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/rc.txt
timeout 1200 python -m pytest tests -m gpu -q -x -k "lipschitz or hvp or idiv_hvp" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
tail -3 $OUT/pytest.log
cp paper_1404_5344_b200/libfoe.so $OUT/orig.so.bak
for f in ab_libs/*.so; do n=$(basename $f .so); cp $f paper_1404_5344_b200/libfoe.so
  echo "== $n" >> $OUT/setup.log; timeout 600 python tools/setup_time.py >> $OUT/setup.log 2>&1
done
cp $OUT/orig.so.bak paper_1404_5344_b200/libfoe.so; cat $OUT/setup.log; cat $OUT/rc.txt
