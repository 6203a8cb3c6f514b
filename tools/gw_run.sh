# gather_width sweep + DRAM bytes per read (ncu metrics pass), then the GPU suite
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gw_smi.txt
timeout 300 tools/gather_width sweep > gpurun_out/gw_sweep.txt 2>&1; echo "sweep rc=$?"
for S in 1 2 4 8; do
  timeout 120 tools/gather_width one 22 $S 1 > gpurun_out/gw_one_$S.txt 2>&1 &&
  timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum \
      --clock-control none -k regex:chase --csv --log-file gpurun_out/gw_ncu_$S.csv tools/gather_width one 22 $S 1 \
      > gpurun_out/gw_ncu_$S.log 2>&1; echo "S=$S rc=$?"
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gw_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gw_gpu_tests.log
