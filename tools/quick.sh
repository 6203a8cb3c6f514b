#!/usr/bin/env bash
# Quick GPU check (run under gpurun): GPU tests (not full size), then bench lines
# for the given configs.   tools/quick.sh TAG "2 3 5" [extra bench args]
TAG=$1; CFGS=${2:-"2 3"}; shift 2; EXTRA="$@"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" --timeout=300 > gpurun_out/t_$TAG.log 2>&1
echo "tests=$?"; tail -3 gpurun_out/t_$TAG.log
for c in $CFGS; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 3 $EXTRA > gpurun_out/b_${TAG}_cfg$c.json 2> gpurun_out/b_${TAG}_cfg$c.err
  echo "bench cfg$c rc=$?"
done
