#!/usr/bin/env bash
# Source-level ncu capture of the walker (run under gpurun, ONE GPU):
#   tools/prof_src.sh TAG "bench args"   -> gpurun_out/TAG_{raw,src}.csv, TAG_sass.csv.gz
set -u
TAG=$1; ARGS=$2; KRE=${3:-walk_}
mkdir -p gpurun_out
B="--steps 3 --warmup 3 --no-cpu --no-e2e"
python bench.py $ARGS $B > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || { echo "plain run failed"; tail gpurun_out/${TAG}_plain.err; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 \
    -o gpurun_out/$TAG python bench.py $ARGS $B > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_src.csv 2>/dev/null
gzip -f gpurun_out/${TAG}_src.csv
sz=$(stat -c %s gpurun_out/$TAG.ncu-rep 2>/dev/null || echo 0)
[ "$sz" -gt 30000000 ] && rm -f gpurun_out/$TAG.ncu-rep
ls -la gpurun_out | grep $TAG
