#!/usr/bin/env bash
# Round-2 profiles (run under gpurun, ONE GPU): every ncu run follows the same command's
# clean plain run.  Reports are reduced to CSV on the box (gpurun copies back <= 64 MiB).
set -u
mkdir -p gpurun_out
B="--steps 3 --warmup 3 --no-cpu --no-e2e"
KSEL='regex:walk_|build_|check_|row_|skipgram|first_row'
reduce() {   # rep -> raw + source CSV, then drop the report unless it is small
  local r=$1
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_sass.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv > gpurun_out/${r}_src.csv 2>/dev/null
  gzip -f gpurun_out/${r}_sass.csv
  local sz=$(stat -c %s gpurun_out/$r.ncu-rep 2>/dev/null || echo 0)
  [ "$sz" -gt 15000000 ] && rm -f gpurun_out/$r.ncu-rep
  ls -la gpurun_out/ | grep $r
}
# 1) configs[1]: full capture of one timed launch + the launch list of our kernels
python bench.py --config 2 $B > gpurun_out/p2_plain.json 2> gpurun_out/p2_plain.err && {
  ncu --set full --clock-control none --import-source on -k regex:walk_tab -s 3 -c 1 \
      -o gpurun_out/prof_r02_cfg2 python bench.py --config 2 $B > gpurun_out/p2_full.log 2>&1; echo "cfg2 full rc=$?"
  reduce prof_r02_cfg2
  ncu --metrics gpu__time_duration.sum --clock-control none -k "$KSEL" --csv \
      --log-file gpurun_out/launches_r02_cfg2.csv python bench.py --config 2 $B > gpurun_out/p2_launch.log 2>&1
  echo "cfg2 launches rc=$?"; }
# 2) configs[4] node2vec: full capture on the first 2^22 walks (the full graph; the whole
#    walk matrix would make ncu save / restore 34 GB per replay pass)
python bench.py --config 5 --max-walks 4194304 $B > gpurun_out/p5_plain.json 2> gpurun_out/p5_plain.err && {
  ncu --set full --clock-control none --import-source on -k regex:walk_tab -s 3 -c 1 \
      -o gpurun_out/prof_r02_cfg5 python bench.py --config 5 --max-walks 4194304 $B > gpurun_out/p5_full.log 2>&1
  echo "cfg5 full rc=$?"
  reduce prof_r02_cfg5; }
# 3) DRAM traffic of one timed launch, every config (single pass: no replay)
for c in 2 3 4 5; do
  python bench.py --config $c $B > gpurun_out/t${c}_plain.json 2> gpurun_out/t${c}_plain.err && {
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        -k regex:walk_tab -s 3 -c 1 --csv --log-file gpurun_out/traffic_r02_cfg$c.csv python bench.py --config $c $B \
        > gpurun_out/t${c}_ncu.log 2>&1; echo "traffic cfg$c rc=$?"; }
done
du -sh gpurun_out
