NCU="ncu --set full --clock-control none --import-source on -k regex:gs_sim_kernel -c 1"
timeout 900 $NCU -o gpurun_out/full_r2m_s -f python tools/launch_config.py C2 --runs 3552 > /dev/null 2>&1; echo "s rc=$?"
timeout 900 $NCU -o gpurun_out/full_r2m_xs -f python tools/launch_config.py C5 --runs 12500 > /dev/null 2>&1; echo "xs rc=$?"
cp paper_2309_00558_b200/_lib/libgshare_b200.so gpurun_out/full_r2m.so
python bench.py > gpurun_out/bench_r2m.log 2>&1; tail -1 gpurun_out/bench_r2m.log > gpurun_out/bench_r2m.json; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2m.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-api --no-per-config > /dev/null 2>&1; echo launches rc=$?
