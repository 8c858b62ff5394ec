# A/B timing of library variants in ONE box session (box-to-box variance is ~5%).
#   LIBS="old s3" CONFIGS=c1,c4,c5 bash tools/ab.sh      ("" = the default in-tree library)
for lib in "" $LIBS; do
  if [ -n "$lib" ]; then export MCSBR_GPU_LIB=$PWD/paper_2511_07586_b200/libmcsbr_gpu_$lib.so; else unset MCSBR_GPU_LIB; fi
  tag=${lib:-default}
  timeout 300 python tools/profile_c2.py > gpurun_out/ab_c2_$tag.log 2>&1
  echo "[$tag] c2: $(tail -1 gpurun_out/ab_c2_$tag.log)"
  timeout 600 python tools/bench_configs.py --configs ${CONFIGS:-c1,c3,c4,c5} --out gpurun_out/ab_$tag.json > gpurun_out/ab_$tag.log 2>&1
  python - "$tag" <<'PY'
import json, sys
d = json.load(open(f'gpurun_out/ab_{sys.argv[1]}.json'))
print(f"[{sys.argv[1]}]", {k: round(v.get('gpu_ms_per_angle', v.get('gpu_ms')), 3) for k, v in d.items()})
PY
done
