python -m pytest tests -m gpu -q -rf --durations=15 -p no:cacheprovider --timeout 900 > gpurun_out/gputest8.log 2>&1
tail -25 gpurun_out/gputest8.log
AB_MODES=pipelined bash tools/lab/run_variants.sh "python tools/time_elements.py" occ6 occ8 > gpurun_out/k2_occ_lab.log 2>&1
cat gpurun_out/k2_occ_lab.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4_r2e.json 2> gpurun_out/bench_c4_r2e.err
tail -2 gpurun_out/bench_c4_r2e.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_c4_r2e.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']); print(d['roofline']); print({k:(v['avg_us'],v['gbs']) for k,v in d['kernels'].items()}); print(d.get('c2_point')); print(d.get('cpu_baseline'))"
timeout 900 ncu --profile-from-start off --clock-control none --kernel-name regex:"k_cg_init_scaled|k_cg_finish_scaled" --launch-count 2 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r2_c4_initfinish.csv python tools/profile_step_c4.py > gpurun_out/prof_c4e.log 2>&1
cat gpurun_out/r2_c4_initfinish.csv | tail -8
