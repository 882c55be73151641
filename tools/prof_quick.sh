#!/bin/bash
# quick ncu capture of the megakernel on a reduced C2 batch: bash tools/prof_quick.sh <tag> [runs] [windows]
TAG=${1:-q}; RUNS=${2:-2368}; WIN=${3:-100}
ncu --set full --clock-control none --import-source on -k regex:gs_sim_kernel -c 1 \
    -o gpurun_out/prof_${TAG} -f \
    python bench.py --runs $RUNS --windows $WIN --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/prof_${TAG}.log 2>&1
cp paper_2309_00558_b200/_lib/libgshare_b200.so gpurun_out/prof_${TAG}.so
