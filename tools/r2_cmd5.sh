# C4 bench with the column-compressed SpMV + a targeted ncu of the CG kernels
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4_r2b.json 2> gpurun_out/bench_c4_r2b.err
tail -2 gpurun_out/bench_c4_r2b.err
timeout 1200 ncu --profile-from-start off --clock-control none --kernel-name regex:"k_cg_spmv16|k_cg_update|k_cg_init_perm" --launch-count 4 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed \
  --csv --log-file gpurun_out/r2_c4_cg16.csv python tools/profile_step_c4.py > gpurun_out/prof_c4b.log 2>&1
tail -2 gpurun_out/prof_c4b.log
# the multi-rank bench path (per-rank generation, peer-memory exchanges, fused CG, graphs) with 2 ranks on one GPU
AB_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --workload c3 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_gloo2_c3.json 2> gpurun_out/bench_gloo2_c3.err
tail -5 gpurun_out/bench_gloo2_c3.err; tail -c 1500 gpurun_out/bench_gloo2_c3.json
