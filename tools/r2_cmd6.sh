bash tools/lab/run_variants.sh "python tools/lab/time_spmv16.py 1.0" c8 c24 m4 > gpurun_out/spmv16_lab.log 2>&1
cat gpurun_out/spmv16_lab.log
python bench.py --steps 10 --warmup 3 --no-c2 > gpurun_out/bench_c4_r2c.json 2> gpurun_out/bench_c4_r2c.err
tail -2 gpurun_out/bench_c4_r2c.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_c4_r2c.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['clocks']); print({k:(v['avg_us'],v['gbs']) for k,v in d['kernels'].items()})"
