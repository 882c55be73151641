#!/bin/bash
# ncu --set full captures of the C2 (HotS) and C4 (XL) kernels for source-level
# reading here (tools/ncu_lines.py); the .so of the capture is saved beside it.
TAG=${1:-r2d}
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on -k regex:gs_sim_kernel -c 1"
timeout 900 $NCU -o gpurun_out/full_${TAG}_s -f python tools/launch_config.py C2 --runs 3552 > gpurun_out/full_${TAG}_s.log 2>&1; echo "ncu s rc=$?"
timeout 900 $NCU -o gpurun_out/full_${TAG}_xl -f python tools/launch_config.py C4 --runs 148 --windows 300 > gpurun_out/full_${TAG}_xl.log 2>&1; echo "ncu xl rc=$?"
cp paper_2309_00558_b200/_lib/libgshare_b200.so gpurun_out/full_${TAG}.so
