#!/bin/bash
# Capture the launch list and one full ncu report of the scenario megakernel.
# Usage (on the GPU box): bash tools/profile.sh <tag> [runs]
set -x
TAG=${1:-r01}; RUNS=${2:-1184}
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --runs $RUNS --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gs_sim_kernel -c 1 \
    -o gpurun_out/prof_${TAG} -f \
    python bench.py --runs $RUNS --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/prof_${TAG}.log 2>&1
ls -la gpurun_out
