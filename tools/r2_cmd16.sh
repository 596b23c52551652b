AB_MODES=pipelined bash tools/lab/run_variants.sh "python tools/time_elements.py" branchy
AB_MODES=pipelined AB_MESH=c3:1.0 bash tools/lab/run_variants.sh "python tools/time_elements.py" branchy
python -m pytest tests/test_gpu_flow.py tests/test_gpu_production.py -q -x -p no:cacheprovider --timeout 900 -k "momentum or multi_block or k2 or divergence or time_steps" 2>&1 | tail -3
