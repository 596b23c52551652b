for t in 1024 4096; do AB_CG_TILE=$t timeout 900 python bench.py --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/bench_tile$t.log 2>&1; grep '^{' gpurun_out/bench_tile$t.log | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print($t, d['value'], d['kernels']['K5_cg_tile_iter']['avg_us'], d['clocks']['sm_mhz'])"; done
timeout 900 python bench.py --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/bench_tile2048.log 2>&1; grep '^{' gpurun_out/bench_tile2048.log | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(2048, d['value'], d['kernels']['K5_cg_tile_iter']['avg_us'], d['clocks']['sm_mhz'])"
