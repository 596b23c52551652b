# colour mode determinism (fenced REDs) + timing; K2 full ncu with source (C2)
python -m pytest tests/test_gpu_colour.py -q -p no:cacheprovider --timeout 900 > gpurun_out/gputest_colour3.log 2>&1
tail -8 gpurun_out/gputest_colour3.log
AB_MODES=pipelined,colour python tools/time_elements.py > gpurun_out/colour_c2c.log 2>&1; cat gpurun_out/colour_c2c.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_pipe<1, 0" -s 1 -c 1 -o gpurun_out/r2_k2 python tools/profile_step.py --steps 1 > gpurun_out/ncu_k2.log 2>&1
tail -3 gpurun_out/ncu_k2.log
