timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_cg_tile_iter|k_pipe" -c 2 -o gpurun_out/r2_c4_full python tools/profile_step_c4.py > gpurun_out/prof_c4_full.log 2>&1
tail -2 gpurun_out/prof_c4_full.log; ls -la gpurun_out/r2_c4_full.ncu-rep
