#!/bin/bash
# ncu --set full of the fan-beam projector pair (cfg3 geometry, batch 32) + launch timing.
TAG=${1:-fan}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"forward_kernel|backproject_kernel" -s 2 -c 2 -o gpurun_out/prof_$TAG python tools/prof_step.py fan512 2 32 > gpurun_out/ncu_$TAG.log 2>&1; tail -2 gpurun_out/ncu_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"forward_kernel|backproject_kernel" -s 2 -c 2 -o gpurun_out/prof_${TAG}_par python tools/prof_step.py par512 2 32 > gpurun_out/ncu_${TAG}_par.log 2>&1; tail -2 gpurun_out/ncu_${TAG}_par.log
