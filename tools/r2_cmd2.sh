set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4_r2a.json 2> gpurun_out/bench_c4_r2a.err
tail -3 gpurun_out/bench_c4_r2a.err
timeout 1500 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,launch__grid_size --csv --log-file gpurun_out/r2_c4_metrics.csv python tools/profile_step_c4.py > gpurun_out/prof_c4.log 2>&1
tail -5 gpurun_out/prof_c4.log
