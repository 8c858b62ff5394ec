# Same-box A/B of scheduling knobs on a full config sweep (device and path-kernel ms): CFG=c5|c4 KNOBS="X=1 MCSBR_GSS=32,MCSBR_BAND=16 ..."
for i in 1 2; do
  for e in ${KNOBS:-"X=1" "MCSBR_CHUNK_MAX=1024" "MCSBR_CHUNK_MAX=256" "MCSBR_BAND=16"}; do
    env ${e//,/ } timeout 600 python tools/bench_configs.py --configs ${CFG:-c5} --out gpurun_out/ab_c5.json > /dev/null 2>&1
    python -c "import json; d=json.load(open('gpurun_out/ab_c5.json'))['${CFG:-c5}']['config']; print('[$e]', round(d['device_ms'],1), round(d['path_kernel_ms'],1))"
  done
done
