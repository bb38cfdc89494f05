# Round-end evidence run (development aid): bench line, the bench's ncu launch list, and
# ncu --set full captures of the dominant kernels at the bench's chunk size (2^25 queries).
set -x
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; echo ref rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo launches rc $?
timeout 2000 ncu --set full --import-source on --clock-control none -k regex:"^k_ff_near$|k_ff_far_eval|k3_newton_binned|^k_ff_fill$|k3_candidates|k_cull_grid" --profile-from-start off -c 6 -o gpurun_out/c5_32M_full -f python tools/profile_run.py 5 33554432 > gpurun_out/ncu_full.log 2>&1; echo full rc $?
tail -2 gpurun_out/ncu_full.log
