#!/bin/bash
# Build libfoe variants for tools/gpu_ablib.sh: each argument is NAME:"-DFOO=1 -DBAR=2"
set -e
mkdir -p ab_libs; rm -f ab_libs/*.so
P=paper_1404_5344_b200
for spec in "$@"; do
  n=${spec%%:*}; d=${spec#*:}
  /usr/local/cuda/bin/nvcc -gencode=arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -shared -Iinclude -Xptxas -O3 $d -o ab_libs/$n.so $P/csrc/*.cu &
done
wait
ls -la ab_libs
