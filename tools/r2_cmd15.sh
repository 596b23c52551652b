AB_MODES=pipelined python tools/time_elements.py 2>&1 | tail -1
AB_MODES=pipelined,colour AB_MESH=c3:1.0 python tools/time_elements.py 2>&1 | tail -2
python -m pytest tests/test_gpu_flow.py tests/test_gpu_colour.py tests/test_gpu_production.py -q -x -p no:cacheprovider --timeout 900 -k "momentum or multi_block or k2 or divergence or colour or time_steps" 2>&1 | tail -3
