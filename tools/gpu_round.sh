# Round evidence on one B200: parity suite, smoke, bench (both arms), the launch
# list and full ncu captures of the path kernel (c2 bench workload, c4, c5) and
# of the deferred accumulation kernel (c5), all configs GPU vs CPU reference.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:path_kernel -s 1 -c 1 -o gpurun_out/path_full -f python tools/profile_c2.py > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:path_kernel -s 1 -c 1 -o gpurun_out/c4_full -f python tools/profile_isar.py c4 --angles 16 > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:path_kernel -s 1 -c 1 -o gpurun_out/c5_full -f python tools/profile_isar.py c5 --angles 2 > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:path_kernel -s 2 -c 1 -o gpurun_out/c3_full -f python tools/bench_configs.py --configs c3 --out /tmp/c3.json > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:accumulate_kernel -s 1 -c 1 -o gpurun_out/c5_acc -f python tools/profile_isar.py c5 --angles 2 > gpurun_out/ncu_c5acc.log 2>&1; echo "ncu c5acc rc=$?"
timeout 1200 python tools/bench_configs.py --configs c1,c3,c4,c5 --cpu --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; echo "configs rc=$?"
