#!/bin/bash
# Final-state evidence pass on the GPU box: ncu --set full of the three kernel
# classes (S on one C2 wave, XS on C5's shard, XL on 148 C4 runs x 600 windows),
# the default bench line and the bench's launch list.  usage: bash tools/r2_capture.sh <tag>
TAG=${1:-r2n}
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on -k regex:gs_sim_kernel -c 1"
timeout 900 $NCU -o gpurun_out/full_${TAG}_s -f python tools/launch_config.py C2 --runs 3552 > /dev/null 2>&1; echo "s rc=$?"
timeout 900 $NCU -o gpurun_out/full_${TAG}_xs -f python tools/launch_config.py C5 --runs 12500 > /dev/null 2>&1; echo "xs rc=$?"
timeout 900 $NCU -o gpurun_out/full_${TAG}_xl -f python tools/launch_config.py C4 --runs 148 --windows 600 > /dev/null 2>&1; echo "xl rc=$?"
cp paper_2309_00558_b200/_lib/libgshare_b200.so gpurun_out/full_${TAG}.so
python bench.py > gpurun_out/bench_${TAG}.log 2>&1; tail -1 gpurun_out/bench_${TAG}.log > gpurun_out/bench_${TAG}.json; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-api --no-per-config > /dev/null 2>&1; echo "launches rc=$?"
