AB_MODES=pipelined TAIL=1 bash tools/lab/run_variants.sh "python tools/time_elements.py" k2alg1o5 k2alg0
AB_MODES=pipelined AB_MESH=c3:1.0 TAIL=1 bash tools/lab/run_variants.sh "python tools/time_elements.py" k2alg1o5 k2alg0
cp tools/lab/lib_k2alg1o5.so paper_2005_05899_b200/libalyab200.so
timeout 900 python -m pytest tests/test_gpu_flow.py tests/test_gpu_production.py tests/test_gpu_session.py -q -x -p no:cacheprovider --timeout 900 -k "momentum or multi_block or k2 or time_steps or c1_exact or full_c2_step or mixed_mesh or session or tgv" 2>&1 | tail -3
