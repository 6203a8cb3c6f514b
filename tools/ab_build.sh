#!/usr/bin/env bash
# graph_build_ms and the walk launch per library variant (run under gpurun)
#   tools/ab_build.sh "2 3 5" "default cap256"
CFGS=$1; VARS=$2
mkdir -p gpurun_out
for c in $CFGS; do for v in $VARS; do
  lib=""; [ "$v" != default ] && lib="GRAPE_WALK_LIB=$PWD/exp/libgrape_walk_$v.so"
  env $lib timeout 900 python bench.py --config $c --no-cpu --no-e2e --steps 3 > gpurun_out/abb_${c}_$v.json 2> gpurun_out/abb_${c}_$v.err
  python - gpurun_out/abb_${c}_$v.json "cfg$c $v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:16s} build {d['graph_build_ms']:8.1f} ms  walk {d['ms_per_step']:8.2f} ms  {d['value']:.4g} steps/s")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done; done
