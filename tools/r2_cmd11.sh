# colour mode with ordered REDs: tests + timing; SpMV16 vs int32 (same diag form) with ncu; C4 per-kernel metrics (app replay)
python -m pytest tests/test_gpu_colour.py -q -p no:cacheprovider --timeout 900 > gpurun_out/gputest_colour2.log 2>&1
tail -15 gpurun_out/gputest_colour2.log
AB_MODES=pipelined,colour python tools/time_elements.py > gpurun_out/colour_c2b.log 2>&1; cat gpurun_out/colour_c2b.log
timeout 900 python tools/lab/time_spmv16.py 1.0 > gpurun_out/spmv16_c3b.log 2>&1; cat gpurun_out/spmv16_c3b.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cg_spmv16" -s 3 -c 1 -o gpurun_out/r2_spmv16 python tools/lab/time_spmv16.py 1.0 16-scaled-diag > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cg_spmv" -s 3 -c 1 -o gpurun_out/r2_spmv32 python tools/lab/time_spmv16.py 1.0 int32-scaled-diag > /dev/null 2>&1
timeout 1800 ncu --profile-from-start off --replay-mode application --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum \
  --csv --log-file gpurun_out/r2_c4_step_metrics_v3.csv python tools/profile_step_c4.py > gpurun_out/prof_c4h.log 2>&1
tail -3 gpurun_out/prof_c4h.log; grep -c k_cg_spmv gpurun_out/r2_c4_step_metrics_v3.csv; ls -la gpurun_out
