timeout 1200 python tools/bench_configs.py --configs c1,c3,c4,c5 --cpu --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; echo "configs rc=$?"; tail -3 gpurun_out/configs.log | cut -c1-300
