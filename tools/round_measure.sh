#!/bin/bash
# Full measurement pass on the GPU box: bench (default config), launch list, one ncu --set full.
TAG=${1:-r1}
python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_${TAG}.log > gpurun_out/bench_${TAG}.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gs_sim_kernel -c 1 \
    -o gpurun_out/full_${TAG} -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
    > gpurun_out/full_${TAG}.log 2>&1
cp paper_2309_00558_b200/_lib/libgshare_b200.so gpurun_out/full_${TAG}.so
nproc > gpurun_out/nproc_${TAG}.txt; lscpu | grep "Model name" >> gpurun_out/nproc_${TAG}.txt
