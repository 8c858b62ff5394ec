set -x
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e.log 2>&1; echo "e2e rc=$?"; cat gpurun_out/e2e.log | tail -8
timeout 300 python tools/profile_isar.py c4 --angles 64 > gpurun_out/c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/c4.log
timeout 300 python tools/profile_isar.py c5 --angles 4 > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"; tail -1 gpurun_out/c5.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:path_kernel -s 1 -c 1 -o gpurun_out/c4_full -f python tools/profile_isar.py c4 --angles 16 > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:path_kernel -s 1 -c 1 -o gpurun_out/c5_full -f python tools/profile_isar.py c5 --angles 2 > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
