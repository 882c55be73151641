#!/bin/bash
# quick GPU check: all gpu tests, then device timings of C2 / C4 / C5 / C1 / C3
TAG=${1:-q}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_${TAG}.txt 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/tests_${TAG}.txt
for c in "C2 --runs 21312" "C4 --runs 148 --windows 600" "C5 --runs 12500" "C1 --runs 2048" "C3 --runs 2048"; do
  timeout 600 python tools/launch_config.py $c --launches 3 ${CHECK} 2>&1 | tail -1
done
