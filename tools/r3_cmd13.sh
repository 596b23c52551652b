timeout 900 python -m pytest tests/test_gpu_peer.py -q -x -p no:cacheprovider --timeout 900 2>&1 | tail -2
timeout 900 python tools/time_dd2.py 160 2
