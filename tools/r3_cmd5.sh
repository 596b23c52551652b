# tiled SpMV: tile sizes; C4 bench with the tiled SpMV default; C4 per-kernel ncu metrics (app replay)
python tools/time_cg_large.py 200 two-pass,tile1024,tile1536,tile2048 2>&1 | grep us/it
timeout 900 python bench.py > gpurun_out/bench_c4_tile.log 2>&1; grep '^{' gpurun_out/bench_c4_tile.log | cut -c1-600
timeout 2000 ncu --profile-from-start off --replay-mode application --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum \
  --csv --log-file gpurun_out/r2_c4_step_metrics_v4.csv python tools/profile_step_c4.py > gpurun_out/prof_c4_v4.log 2>&1
tail -2 gpurun_out/prof_c4_v4.log; grep -c k_cg_spmv gpurun_out/r2_c4_step_metrics_v4.csv
