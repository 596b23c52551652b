set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 900 --durations=15 > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -c 1500 gpurun_out/bench_ref.log
