#!/bin/bash
# Round-2 closing evidence in one call: tools/gpu_final.sh TAG bench (smoke, bench lines, launch
# list), then the whole -m gpu suite
TAG=${1:-r2final}
tools/gpu_final.sh $TAG bench
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/rc.txt
cat gpurun_out/$TAG/rc.txt; tail -2 gpurun_out/$TAG/pytest_gpu.log
