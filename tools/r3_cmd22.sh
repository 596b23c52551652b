AB_MODES=pipelined TAIL=1 bash tools/lab/run_variants.sh "python tools/time_elements.py" nodefer 2>&1 | cut -c1-70
AB_MODES=pipelined AB_MESH=c3:1.0 TAIL=1 bash tools/lab/run_variants.sh "python tools/time_elements.py" nodefer 2>&1 | cut -c1-70
timeout 900 python -m pytest tests/test_gpu_flow.py tests/test_gpu_production.py tests/test_gpu_colour.py -q -x -p no:cacheprovider --timeout 900 -k "momentum or multi_block or k2 or time_steps or full_c2_step or mixed_mesh or divergence_gradient or colour" 2>&1 | tail -2
