#!/bin/bash
# Dev cycle on the GPU box: parity tests, quick per-config timing, ncu capture of one forward+inverse.
# usage: tools/gpu_cycle.sh TAG [ncu-config]
TAG=${1:-dev}
CFG=${2:-cfg5_3d_512}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python tools/quick_time.py gpurun_out/quick_time_$TAG.json 2>&1 | tail -10
if [ "$CFG" != "none" ]; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:axis_kernel -c 6 \
    -o gpurun_out/prof_$TAG python tools/prof_run.py $CFG > gpurun_out/ncu_$TAG.log 2>&1
  tail -2 gpurun_out/ncu_$TAG.log
fi
