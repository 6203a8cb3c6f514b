#!/usr/bin/env bash
# bench one config under several forced table layouts (run under gpurun)
#   tools/layout_sweep.sh CFG "layout1" "layout2" ...   (layout: key=val,key=val or "auto")
CFG=$1; shift
for lay in "$@"; do
  arg=""; [ "$lay" != "auto" ] && arg="--layout $lay"
  tag=$(echo "$lay" | tr ',=' '_-')
  timeout 600 python bench.py --config $CFG --no-cpu --no-e2e --steps 3 $arg > gpurun_out/ls_cfg${CFG}_$tag.json 2> gpurun_out/ls_cfg${CFG}_$tag.err
  python tools/show.py gpurun_out/ls_cfg${CFG}_$tag.json | sed "s|^|$lay |" | cut -c1-200
done
