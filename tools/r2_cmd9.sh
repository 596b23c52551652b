# re-entry check of HEAD: GPU suite, C4 bench, CG kernel ncu
python -m pytest tests -m gpu -q -rf --durations=15 -p no:cacheprovider --timeout 900 > gpurun_out/gputest9.log 2>&1
tail -25 gpurun_out/gputest9.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4_r2f.json 2> gpurun_out/bench_c4_r2f.err
tail -2 gpurun_out/bench_c4_r2f.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_c4_r2f.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']); print(d['roofline']); print({k:(v['avg_us'],v['gbs']) for k,v in d['kernels'].items()}); print(d.get('c2_point')); print(d.get('cpu_baseline'))"
timeout 900 ncu --profile-from-start off --clock-control none --kernel-name regex:"k_cg_spmv|k_cg_update|k_cg_init|k_cg_finish" --launch-count 6 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/r2_c4_cg9.csv python tools/profile_step_c4.py > gpurun_out/prof_c4f.log 2>&1
tail -12 gpurun_out/r2_c4_cg9.csv
