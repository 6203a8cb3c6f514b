#!/usr/bin/env bash
# Re-run every bench line kept under profiles/ (run under gpurun): tools/refresh_all.sh TAG
TAG=${1:-fin}
mkdir -p gpurun_out
run() { name=$1; shift; python bench.py "$@" > gpurun_out/${TAG}_$name.json 2> gpurun_out/${TAG}_$name.err; echo "$name rc=$?"; }
run cfg_2 --config 2
run cfg_1 --config 1
run cfg_3 --config 3
run cfg_4 --config 4
run cfg_5 --config 5
run cfg_5_first_order --config 5 --mode first_order
run cfg_2_folded --config 2 --sampler folded
run cfg_5_folded --config 5 --sampler folded
run cfg_2_approx10 --config 2 --approx 10
run cfg_3_approx10 --config 3 --approx 10
run cfg_5_approx10 --config 5 --approx 10
run cfg_2_skipgram --config 2 --skipgram 200000
run cfg_5_skipgram --config 5 --skipgram 200000
