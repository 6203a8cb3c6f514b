#!/usr/bin/env bash
# A/B library variants with the in-run issue counters:  tools/ab_issue.sh "2 5" "default nospot" [bench args]
CFGS=$1; VARS=$2; shift 2; EXTRA="$@"
mkdir -p gpurun_out
for c in $CFGS; do for v in $VARS; do
  lib=""; [ "$v" != default ] && lib="GRAPE_WALK_LIB=$PWD/exp/libgrape_walk_$v.so"
  tag=cfg${c}_${v}
  env $lib timeout 900 python bench.py --config $c --no-cpu --no-e2e --steps 5 $EXTRA > gpurun_out/abi_$tag.json 2> gpurun_out/abi_$tag.err
  python - gpurun_out/abi_$tag.json $tag <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    i = d['roofline'].get('issue') or {}
    print(f"{sys.argv[2]:24s} {d['value']:.4g} steps/s {d['ms_per_step']:.2f} ms  inst/step {i.get('warp_instructions_per_step',0):.1f} thr/inst {i.get('active_threads_per_instruction',0):.1f} issue {i.get('frac',0):.3f}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done; done
