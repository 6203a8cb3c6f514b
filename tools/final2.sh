set -u
TAG=r02g
mkdir -p gpurun_out
run() { name=$1; shift; timeout 1500 python bench.py "$@" > gpurun_out/${TAG}_$name.json 2> gpurun_out/${TAG}_$name.err; echo "$name rc=$? $(grep -c 'dram probe' gpurun_out/${TAG}_$name.err)"; }
run default --steps 20 --warmup 5
run cfg_3 --config 3
run cfg_4 --config 4
run cfg_5 --config 5
run cfg_1 --config 1
run cfg2_skipgram --config 2 --skipgram 2000000
run cfg5_skipgram --config 5 --skipgram 2000000
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/${TAG}_gpu_tests.log
