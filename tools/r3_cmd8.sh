python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 900 > gpurun_out/gputest_v4.log 2>&1; tail -2 gpurun_out/gputest_v4.log
timeout 2000 ncu --profile-from-start off --replay-mode application --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum \
  --csv --log-file gpurun_out/r2_c4_step_metrics_v5.csv python tools/profile_step_c4.py > gpurun_out/prof_c4_v5.log 2>&1
tail -1 gpurun_out/prof_c4_v5.log
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:"k_cg_tile_iter" -s 5 -c 1 -o gpurun_out/r2_tile_iter python tools/time_cg_large.py 200 sptile2048 > /dev/null 2>&1; ls gpurun_out/*.ncu-rep
