timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled -k regex:"k_pipe<1, 0" -c 1 -o gpurun_out/r2_c4_k2tet python tools/profile_step_c4.py > gpurun_out/prof_c4_k2.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_cg_tile_iter" -s 3 -c 1 -o gpurun_out/r2_c4_tileiter python tools/profile_step_c4.py > gpurun_out/prof_c4_ti.log 2>&1
ls -la gpurun_out/*.ncu-rep
