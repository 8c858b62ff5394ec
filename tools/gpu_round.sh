# Round evidence on one B200: the GPU suite, smoke, the bench (c5 headline +
# c2 secondary) and its reference arm, the bench's ncu launch list, and full
# ncu captures of the c5 path kernel (one 16-azimuth launch group of the bench
# sweep), the c5 accumulation (NUFFT spread) kernel and the c2 path kernel.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/lscpu.txt
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:path_kernel -s 1 -c 1 -o gpurun_out/c5_full -f python tools/profile_isar.py c5 --angles 16 > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spread_kernel -s 1 -c 1 -o gpurun_out/c5_acc -f python tools/profile_isar.py c5 --angles 16 > gpurun_out/ncu_c5acc.log 2>&1; echo "ncu c5acc rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:path_kernel -s 1 -c 1 -o gpurun_out/c2_full -f python tools/profile_c2.py > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
