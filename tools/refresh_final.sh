#!/usr/bin/env bash
# Final round-2 evidence on the final code (run under gpurun, one GPU):
#   GPU suite, the default bench line + the reference arm, every config / mode line,
#   the SkipGram lines, the launch list of the default command.  tools/refresh_final.sh TAG
TAG=${1:-r02f}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/${TAG}_gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_default.json 2> gpurun_out/${TAG}_default.err; echo "default rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err; echo "reference rc=$?"
tools/refresh_r02.sh $TAG
run() { name=$1; shift; timeout 1500 python bench.py "$@" > gpurun_out/${TAG}_$name.json 2> gpurun_out/${TAG}_$name.err; echo "$name rc=$?"; }
run cfg_5_approx10 --config 5 --approx 10
run cfg2_skipgram --config 2 --skipgram 2000000
run cfg5_skipgram --config 5 --skipgram 2000000
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:walk_|build_|check_|row_|skipgram" --csv \
    --log-file gpurun_out/${TAG}_cfg2_launches_raw.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
echo "launches rc=$?"
python tools/launch_list.py gpurun_out/${TAG}_cfg2_launches_raw.csv > gpurun_out/${TAG}_cfg2_launches.csv 2>/dev/null
tools/prof_src.sh ${TAG}_sg_cfg2 "--config 2 --skipgram 2000000" skipgram_kernel > /dev/null 2>&1; echo "sg prof rc=$?"
rm -f gpurun_out/${TAG}_sg_cfg2.ncu-rep
du -sh gpurun_out
