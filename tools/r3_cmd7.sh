timeout 900 python -m pytest tests/test_gpu_flow.py tests/test_gpu_production.py -q -x -p no:cacheprovider --timeout 900 -k "pcg or cg_full" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_c4_sp.log 2>&1; grep '^{' gpurun_out/bench_c4_sp.log | python -c "
import json,sys; d=json.loads(sys.stdin.readline())
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches'], d['clocks'])
print(d['roofline'])
for k,v in d['kernels'].items(): print(k, v)"
