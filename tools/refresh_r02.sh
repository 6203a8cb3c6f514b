#!/usr/bin/env bash
# Round-2 bench lines kept under profiles/ (run under gpurun, one GPU): tools/refresh_r02.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
run() { name=$1; shift; timeout 1500 python bench.py "$@" > gpurun_out/${TAG}_$name.json 2> gpurun_out/${TAG}_$name.err; echo "$name rc=$?"; }
run cfg_2 --config 2 --steps 10 --warmup 5
run cfg_1 --config 1
run cfg_3 --config 3
run cfg_4 --config 4
run cfg_5 --config 5
run cfg_5_first_order --config 5 --mode first_order
run cfg_6 --config 6 --layout table_budget_bytes=100e9
run cfg_2_folded --config 2 --sampler folded
run cfg_5_folded --config 5 --sampler folded
run cfg_2_approx10 --config 2 --approx 10
run cfg_3_approx10 --config 3 --approx 10
run cfg_2_cdf --config 2 --sampler cdf --steps 3 --warmup 3
run cfg_2_parts8 --config 2 --parts 8
# two ranks on this one GPU (gloo): the N > 1 code paths, not a scaling measurement
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29711 \
  bench.py --gpus 2 --config 2 --device 0 --dist-backend gloo --no-e2e > gpurun_out/${TAG}_cfg_2_two_ranks_one_gpu.json \
  2> gpurun_out/${TAG}_cfg_2_two_ranks_one_gpu.err; echo "two ranks rc=$?"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29713 \
  bench.py --gpus 2 --config 2 --device 0 --dist-backend gloo --no-e2e --dist-tables --table-budget 12 \
  > gpurun_out/${TAG}_cfg_2_dist_tables_one_gpu.json 2> gpurun_out/${TAG}_cfg_2_dist_tables_one_gpu.err
echo "dist tables rc=$?"
