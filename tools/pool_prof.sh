B="--config 2 --steps 1 --warmup 3 --no-cpu --no-e2e"
export GRAPE_WALK_LIB=$PWD/exp/libgrape_walk_pool.so
python bench.py $B > gpurun_out/pp_plain.json 2> gpurun_out/pp_plain.err && \
ncu --metrics smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_short_scoreboard,smsp__pcsamp_warps_issue_stalled_barrier,smsp__pcsamp_warps_issue_stalled_membar,smsp__pcsamp_warps_issue_stalled_wait,smsp__pcsamp_warps_issue_stalled_mio_throttle,smsp__pcsamp_warps_issue_stalled_lg_throttle,smsp__pcsamp_sample_count --clock-control none -k regex:walk_pool -s 3 -c 1 --csv --log-file gpurun_out/pp_metrics.csv python bench.py $B > gpurun_out/pp_ncu.log 2>&1
echo rc=$?
