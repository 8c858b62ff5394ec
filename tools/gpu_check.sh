# quick GPU iteration: parity suite, c2 bench (no CPU leg), the other configs (GPU only)
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-400
timeout 600 python tools/bench_configs.py --configs ${CONFIGS:-c1,c3,c4,c5} --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; echo "configs rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/configs.json'))
for k,v in d.items():
    print(k, {kk: vv for kk, vv in v.items() if 'ms' in kk or 'per_s' in kk})
PY
