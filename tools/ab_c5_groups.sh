for i in 1 2; do
  for e in "X=1" "MCSBR_GROUP_ENTRIES=3000000000 MCSBR_REC_CAP=300000000"; do
    env $e timeout 600 python tools/bench_configs.py --configs c5 --out gpurun_out/ab_c5.json > /dev/null 2>&1
    python -c "import json; d=json.load(open('gpurun_out/ab_c5.json'))['c5']; print('[$e]', {k: (round(v['device_ms'],1), round(v['path_kernel_ms'],1), round(v['accumulate_ms'],1), round(v['e2e_median_ms'],1)) for k,v in d.items() if isinstance(v, dict) and 'device_ms' in v})"
  done
done
