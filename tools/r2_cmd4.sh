python -m pytest tests -m gpu -q -rf --durations=40 -p no:cacheprovider --timeout 900 > gpurun_out/gputest4.log 2>&1
tail -60 gpurun_out/gputest4.log
