#!/usr/bin/env bash
# DRAM bytes of one timed walk launch (run under gpurun):  tools/traffic_capture.sh TAG [bench args]
# One ncu pass with three metrics (a --set full capture replays ~40 times and saves /
# restores the walk matrix each time: minutes on the large configs).
TAG=$1; shift
KERNEL=${KERNEL:-walk_tab}   # KERNEL=walk_cdf for --sampler cdf
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:$KERNEL -s 1 -c 1 -o gpurun_out/traffic_$TAG python bench.py "$@" > gpurun_out/traffic_$TAG.log 2>&1
echo "traffic capture $TAG rc=$?"
