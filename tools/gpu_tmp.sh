timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python tools/ab.py --configs c4,c5 --reps 2 new= prev=prev 2>&1 | tail -3
