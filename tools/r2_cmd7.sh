python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4_r2d.json 2> gpurun_out/bench_c4_r2d.err
tail -2 gpurun_out/bench_c4_r2d.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_c4_r2d.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']); print(d['roofline']); print({k:(v['avg_us'],v['gbs']) for k,v in d['kernels'].items()})"
timeout 900 ncu --profile-from-start off --clock-control none --kernel-name regex:"k_cg_spmv|k_cg_update_scaled|k_cg_init_scaled" --launch-count 4 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --csv --log-file gpurun_out/r2_c4_cgscaled.csv python tools/profile_step_c4.py > gpurun_out/prof_c4d.log 2>&1
tail -2 gpurun_out/prof_c4d.log
