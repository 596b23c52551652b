timeout 900 python -m pytest tests/test_gpu_flow.py tests/test_gpu_production.py -q -x -p no:cacheprovider --timeout 900 -k "pcg or cg_full" 2>&1 | tail -2
TAIL=5 bash tools/lab/run_variants.sh "python tools/time_cg_large.py 200 tile2048,sptile1024,sptile2048,sptile4096 2>&1 | grep us/it | cut -c1-110" spminb4 spminb5 spminb6
