#!/usr/bin/env bash
# ncu --set full of one timed launch of the final (v7) walker: configs[1], and configs[4] on its
# first 2^22 walks (run under gpurun, ONE GPU, after the plain run exited 0).  tools/profile_v7.sh
set -u
mkdir -p gpurun_out
B="--steps 3 --warmup 3 --no-cpu --no-e2e"
reduce() {
  local r=$1
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_sass.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv > gpurun_out/${r}_src.csv 2>/dev/null
  gzip -f gpurun_out/${r}_sass.csv
  rm -f gpurun_out/$r.ncu-rep
  ls -la gpurun_out/ | grep $r
}
python bench.py --config 2 $B > gpurun_out/v7p2_plain.json 2> gpurun_out/v7p2_plain.err && {
  ncu --set full --clock-control none --import-source on -k regex:walk_tab -s 3 -c 1 \
      -o gpurun_out/prof_v7_cfg2 python bench.py --config 2 $B > gpurun_out/v7p2_full.log 2>&1; echo "cfg2 full rc=$?"
  reduce prof_v7_cfg2; }
python bench.py --config 5 --max-walks 4194304 $B > gpurun_out/v7p5_plain.json 2> gpurun_out/v7p5_plain.err && {
  ncu --set full --clock-control none --import-source on -k regex:walk_tab -s 3 -c 1 \
      -o gpurun_out/prof_v7_cfg5 python bench.py --config 5 --max-walks 4194304 $B > gpurun_out/v7p5_full.log 2>&1
  echo "cfg5 full rc=$?"
  reduce prof_v7_cfg5; }
