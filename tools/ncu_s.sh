#!/bin/bash
# ncu --set full capture of the C2 (HotS) kernel on one wave of resident runs
# (3552 = 24 x 148); the bench's 21312-run batch is too large for ncu's
# per-pass save/restore within a call.
TAG=${1:-r2h}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gs_sim_kernel -c 1 \
  -o gpurun_out/full_${TAG}_s -f python tools/launch_config.py C2 --runs 3552 > gpurun_out/full_${TAG}_s.log 2>&1; echo "ncu s rc=$?"
cp paper_2309_00558_b200/_lib/libgshare_b200.so gpurun_out/full_${TAG}.so
