#!/usr/bin/env bash
# A/B library variants x GRAPE_LEAN settings on bench configs (run under gpurun)
#   tools/ab_var.sh "2 5" "default b128m7" "0 1"   (GRAPE_LEAN: the round-2 lean-walker switch, since removed; any value runs the kept walker)
CFGS=$1; VARS=$2; LEANS=${3:-"0 1"}; shift 3; EXTRA="$@"
mkdir -p gpurun_out
for c in $CFGS; do for v in $VARS; do for l in $LEANS; do
  lib=""; [ "$v" != default ] && lib="GRAPE_WALK_LIB=$PWD/exp/libgrape_walk_$v.so"
  tag=cfg${c}_${v}_lean$l
  env $lib GRAPE_LEAN=$l timeout 900 python bench.py --config $c --no-cpu --no-e2e --steps 5 $EXTRA > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python - gpurun_out/ab_$tag.json $tag <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:28s} {d['value']:.4g} steps/s {d['ms_per_step']:.2f} ms  clk {d['clocks'].get('sm_mhz')}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done; done; done
