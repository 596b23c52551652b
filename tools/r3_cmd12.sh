timeout 900 python bench.py > gpurun_out/bench_c4_v5.log 2>&1; grep '^{' gpurun_out/bench_c4_v5.log > gpurun_out/bench_c4_v5.json; python -c "
import json; d=json.load(open('gpurun_out/bench_c4_v5.json')); print(d['value'], d['e2e']['value'], d['roofline'], d['clocks'], d.get('cpu_baseline',{}).get('value'))"
timeout 900 python bench.py --workload c3 --no-c2 --no-cpu-baseline > gpurun_out/bench_c3_v9.log 2>&1; grep '^{' gpurun_out/bench_c3_v9.log > gpurun_out/bench_c3_v9.json; python -c "
import json; d=json.load(open('gpurun_out/bench_c3_v9.json')); print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
