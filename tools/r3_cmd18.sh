python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/gputest_v8.log 2>&1; tail -2 gpurun_out/gputest_v8.log
timeout 900 python bench.py > gpurun_out/bench_c4_v8.log 2>&1; grep '^{' gpurun_out/bench_c4_v8.log > gpurun_out/bench_c4_v8.json; python -c "
import json; d=json.load(open('gpurun_out/bench_c4_v8.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline'].get('frac_dram'), d['clocks'], d['c2_point']['value'], d['cpu_baseline']['value'])"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_v8.log 2>&1; grep '^{' gpurun_out/bench_ref_v8.log | cut -c1-200
