#!/bin/bash
# Round-2 measurement pass on the GPU box: ncu captures of every kernel class,
# launch lists, compute-sanitizer logs, and the default bench line.
# usage: bash tools/r2_measure.sh <tag> [what...]   what: ncu san bench (default all)
TAG=${1:-r2}; shift
WHAT=${@:-ncu san bench}
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on -k regex:gs_sim_kernel -c 1"
for w in $WHAT; do
case $w in
ncu)
  timeout 600 $NCU -o gpurun_out/full_${TAG}_xl -f python tools/launch_config.py C4 --runs 148 --windows 600 > gpurun_out/full_${TAG}_xl.log 2>&1; echo "ncu xl rc=$?"
  timeout 600 $NCU -o gpurun_out/full_${TAG}_xs -f python tools/launch_config.py C5 --runs 12500 > gpurun_out/full_${TAG}_xs.log 2>&1; echo "ncu xs rc=$?"
  timeout 600 $NCU -o gpurun_out/full_${TAG}_s -f python tools/launch_config.py C2 --runs 21312 > gpurun_out/full_${TAG}_s.log 2>&1; echo "ncu s rc=$?"
  for c in "C4 --runs 148 --windows 600" "C5 --runs 12500" "C1 --runs 2048" "C3 --runs 2048"; do
    n=$(echo $c | cut -d' ' -f1)
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_${n}.csv \
      python tools/launch_config.py $c --launches 2 > gpurun_out/launches_${TAG}_${n}.log 2>&1; echo "launches $n rc=$?"
  done
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-api --no-per-config > gpurun_out/launches_${TAG}.log 2>&1; echo "launches bench rc=$?"
  cp paper_2309_00558_b200/_lib/libgshare_b200.so gpurun_out/full_${TAG}.so
  ;;
san)
  for tool in memcheck racecheck synccheck; do
    for c in "C5 --runs 8" "C2 --runs 4 --windows 20" "MIX --runs 10" "C4 --runs 2 --windows 10"; do
      n=$(echo $c | cut -d' ' -f1)
      timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/launch_config.py $c --check \
        > gpurun_out/san_${TAG}_${tool}_${n}.log 2>&1; echo "san $tool $n rc=$?"
    done
  done
  ;;
bench)
  python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"
  tail -1 gpurun_out/bench_${TAG}.log > gpurun_out/bench_${TAG}.json
  nproc > gpurun_out/nproc_${TAG}.txt; lscpu | grep "Model name" >> gpurun_out/nproc_${TAG}.txt
  ;;
esac
done
