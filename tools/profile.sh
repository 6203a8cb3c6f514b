#!/usr/bin/env bash
# Profile the bench step on ONE GPU (run under gpurun).  Usage:
#   tools/profile.sh <tag> [bench args...]
# 1) plain run (must exit 0), 2) ncu launch list (gpu__time_duration per launch),
# 3) one `ncu --set full` capture of the timed walk-kernel launch.
set -u
TAG=${1:-r01}; shift || true
ARGS=${@:-"--steps 1 --warmup 1 --no-e2e --no-cpu"}
mkdir -p gpurun_out
CMD="python bench.py $ARGS"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:walk -s 1 -c 1 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full capture rc=$?"
