set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from __graft_entry__ import smoke; smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
tail -c 600 gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__sass_average_branch_targets_threads_uniform.pct --clock-control none -k regex:"k_ff_near|k_ff_fill|k3_newton|k3_candidates|k3_fallback|k_cull" --csv --log-file gpurun_out/ncu_c5_metrics.csv python tools/profile_run.py 5 1048576 > gpurun_out/ncu_c5.log 2>&1; echo ncu rc $?
tail -3 gpurun_out/ncu_c5.log
