#!/usr/bin/env bash
# Round-2 profiles (run under gpurun, ONE GPU): every ncu run follows the same command's
# clean plain run.  Outputs under gpurun_out/ (prof_*.ncu-rep, launches_*.csv, traffic_*).
set -u
mkdir -p gpurun_out
B="--steps 3 --warmup 3 --no-cpu --no-e2e"
KSEL='regex:walk_|build_|check_|row_|skipgram|first_row'
# 1) configs[1]: full capture of one timed launch + the launch list of our kernels
python bench.py --config 2 $B > gpurun_out/p2_plain.json 2> gpurun_out/p2_plain.err && {
  ncu --set full --clock-control none --import-source on -k regex:walk_tab -s 3 -c 1 \
      -o gpurun_out/prof_r02_cfg2 python bench.py --config 2 $B > gpurun_out/p2_full.log 2>&1; echo "cfg2 full rc=$?"
  ncu --metrics gpu__time_duration.sum --clock-control none -k "$KSEL" --csv \
      --log-file gpurun_out/launches_r02_cfg2.csv python bench.py --config 2 $B > gpurun_out/p2_launch.log 2>&1
  echo "cfg2 launches rc=$?"; }
# 2) configs[4] node2vec: full capture on the first 2^22 walks (the full graph; the whole
#    walk matrix would make ncu save / restore 34 GB per replay pass)
python bench.py --config 5 --max-walks 4194304 $B > gpurun_out/p5_plain.json 2> gpurun_out/p5_plain.err && {
  ncu --set full --clock-control none --import-source on -k regex:walk_tab -s 3 -c 1 \
      -o gpurun_out/prof_r02_cfg5 python bench.py --config 5 --max-walks 4194304 $B > gpurun_out/p5_full.log 2>&1
  echo "cfg5 full rc=$?"; }
# 3) DRAM traffic of one timed launch, every config (single pass: no replay)
for c in 2 3 4 5; do
  python bench.py --config $c $B > gpurun_out/t${c}_plain.json 2> gpurun_out/t${c}_plain.err && {
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        -k regex:walk_tab -s 3 -c 1 -o gpurun_out/traffic_r02_cfg$c python bench.py --config $c $B \
        > gpurun_out/t${c}_ncu.log 2>&1; echo "traffic cfg$c rc=$?"; }
done
