timeout 900 python -m pytest tests/test_gpu_flow.py tests/test_gpu_production.py -q -x -p no:cacheprovider --timeout 900 -k "pcg or cg_full" 2>&1 | tail -3
bash tools/lab/run_variants.sh "python tools/time_cg_single_pass.py 200" fminb8 fch4 fch16
