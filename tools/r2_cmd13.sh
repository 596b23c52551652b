python tools/lab/colour_debug.py 2>&1 | tail -15
echo "== split"
AB_COLOUR_SPLIT=1 python tools/lab/colour_debug.py 2>&1 | tail -15
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_pipe<1, 0" -s 1 -c 1 -o gpurun_out/r2_k2 python tools/profile_step.py --steps 1 > gpurun_out/ncu_k2.log 2>&1
tail -3 gpurun_out/ncu_k2.log
