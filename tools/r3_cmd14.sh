python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 900 > gpurun_out/gputest_v5.log 2>&1; tail -2 gpurun_out/gputest_v5.log
timeout 900 python bench.py > gpurun_out/bench_c4_v6.log 2>&1; grep '^{' gpurun_out/bench_c4_v6.log > gpurun_out/bench_c4_v6.json; python -c "
import json; d=json.load(open('gpurun_out/bench_c4_v6.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline'].get('frac_dram'), d['clocks'], d['kernels']['K5_cg_tile_iter']['avg_us'], d['c2_point']['value'])"
timeout 2000 ncu --profile-from-start off --replay-mode application --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum \
  --csv --log-file gpurun_out/r2_c4_step_metrics_v6.csv python tools/profile_step_c4.py > gpurun_out/prof_c4_v6.log 2>&1
tail -1 gpurun_out/prof_c4_v6.log
