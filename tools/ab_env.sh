# A/B timing of library ENV knobs in one box session (box-to-box variance ~5%):
#   ENVS="MCSBR_QNODES_MIN=0" bash tools/ab_env.sh
# each setting (plus the default) times the c2 path kernel and a 16-azimuth
# c5 / 64-azimuth c4 launch group, alternating twice
for rep in 1 2; do
  for e in "" $ENVS; do
    tag=${e:-default}
    c2=$(env $e timeout 300 python tools/profile_c2.py 2>&1 | tail -1 | cut -c1-160)
    c4=$(env $e timeout 300 python tools/profile_isar.py c4 --angles 64 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['path_kernel_ms'],3))")
    c5=$(env $e timeout 600 python tools/profile_isar.py c5 --angles 16 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['path_kernel_ms'],3))")
    echo "[$rep $tag] c2: $c2 | c4 path ms: $c4 | c5 path ms: $c5"
  done
done
