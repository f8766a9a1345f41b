#!/bin/bash
# one ncu --set full capture of a kernel inside a short bench run (the plain run first, as the
# profiling recipe requires); usage: tools/gpu_prof.sh TAG KERNEL_REGEX [bench args...]
TAG=$1; KRE=$2; SKIP=${SKIP:-5}; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
CMD="python bench.py --steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline $*"
$CMD > $OUT/plain.log 2>&1 && \
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c 1 \
  -o $OUT/prof $CMD > $OUT/ncu.log 2>&1
echo "rc=$?" >> $OUT/ncu.log
