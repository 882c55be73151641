#!/bin/bash
# GPU pass: tests + smoke + bench (+ optional ncu of the C2 class on one wave)
TAG=${1:-r2b}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_${TAG}.txt 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_${TAG}.log > gpurun_out/bench_${TAG}.json
if [ -n "$NCU_S" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gs_sim_kernel -c 1 \
    -o gpurun_out/full_${TAG}_s -f python tools/launch_config.py C2 --runs 3552 > gpurun_out/full_${TAG}_s.log 2>&1; echo "ncu s rc=$?"
  cp paper_2309_00558_b200/_lib/libgshare_b200.so gpurun_out/full_${TAG}.so
fi
