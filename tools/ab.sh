#!/usr/bin/env bash
# A/B the exp/ library variants on the bench step (run under gpurun).
#   tools/ab.sh "bench args" name1 name2 ...
ARGS=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  # spec: variant name, optionally with env assignments: "v3:GRAPE_L2_FETCH_BYTES=32"
  v=${spec%%:*}; envs=""; [ "$spec" != "$v" ] && envs=${spec#*:}
  tag=$(echo "$spec" | tr ':=' '__')
  env $envs GRAPE_WALK_LIB=$PWD/exp/libgrape_walk_$v.so timeout 600 python bench.py $ARGS > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python - "$tag" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
    print(f"{v:12s} {d['value']:.4g} steps/s  {d['ms_per_step']:.2f} ms/step  clocks={d['clocks'].get('sm_mhz')}")
except Exception as e:
    print(v, "FAILED", e, open(f"gpurun_out/ab_{v}.err").read()[-500:])
PY
done
