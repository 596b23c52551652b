# round 2: the full GPU suite + smoke (new: peer, session, production tests)
python -m pytest tests -m gpu -q -rf --durations=30 -p no:cacheprovider -x --timeout 900 > gpurun_out/gputest3.log 2>&1
tail -45 gpurun_out/gputest3.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.log 2>&1; tail -3 gpurun_out/smoke3.log
