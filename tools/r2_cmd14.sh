python tools/lab/colour_debug.py 2>&1 | tail -4
python -m pytest tests/test_gpu_colour.py -q -p no:cacheprovider --timeout 900 > gpurun_out/gputest_colour4.log 2>&1
tail -8 gpurun_out/gputest_colour4.log
AB_MODES=pipelined,colour python tools/time_elements.py > gpurun_out/colour_c2d.log 2>&1; cat gpurun_out/colour_c2d.log
AB_COLOUR_SPLIT=1 AB_MODES=colour python tools/time_elements.py 2>&1 | tail -1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_pipe<\(int\)1, \(int\)0" -s 1 -c 1 -o gpurun_out/r2_k2 python tools/profile_step.py --steps 1 > gpurun_out/ncu_k2.log 2>&1
tail -3 gpurun_out/ncu_k2.log
