# colour-mode scatter: parity + reproducibility tests, timing vs atomics; SpMV16 diagnosis; C4 per-kernel ncu metrics
python -m pytest tests/test_gpu_colour.py -x -q -p no:cacheprovider --timeout 900 > gpurun_out/gputest_colour.log 2>&1
tail -5 gpurun_out/gputest_colour.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke10.log 2>&1; tail -2 gpurun_out/smoke10.log
AB_MODES=pipelined,colour python tools/time_elements.py > gpurun_out/colour_c2.log 2>&1; cat gpurun_out/colour_c2.log
AB_MODES=pipelined,colour AB_MESH=c3:1.0 python tools/time_elements.py > gpurun_out/colour_c3.log 2>&1; cat gpurun_out/colour_c3.log
timeout 900 python tools/lab/time_spmv16.py 1.0 > gpurun_out/spmv16_c3.log 2>&1; cat gpurun_out/spmv16_c3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cg_spmv16" -s 3 -c 1 -o gpurun_out/r2_spmv16 python tools/lab/time_spmv16.py 1.0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cg_spmv_unit" -s 3 -c 1 -o gpurun_out/r2_spmvunit python tools/lab/time_spmv16.py 1.0 > /dev/null 2>&1
timeout 1500 ncu --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum \
  --csv --log-file gpurun_out/r2_c4_step_metrics_v2.csv python tools/profile_step_c4.py > gpurun_out/prof_c4g.log 2>&1
tail -2 gpurun_out/prof_c4g.log; ls -la gpurun_out
