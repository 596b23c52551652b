#!/bin/bash
# Profiles committed under profiles/ for one round (run under gpurun, 1 GPU):
#   tools/profile_round.sh r1b
# then: python tools/ncu_summary.py profiles/<R>_ncu_kernels gpurun_out/<R>_*.ncu-rep --launches gpurun_out/<R>_launches_cold.csv
set -x
R=${1:-r1}
# launch list of one eager C2 step (cold cache, serialised: compare shares)
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_cold.csv \
    python tools/profile_step.py --steps 1 > /dev/null 2>&1
# full captures (cold caches = default, like the bench's flushed L2):
# K2 (pipelined element kernel), K4 (gradient-operator product), K6+K7 (fused product), resident CG
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_pipe -s 1 -c 1 -o gpurun_out/${R}_k2 \
    python tools/profile_step.py --steps 1 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_go_div -c 1 -o gpurun_out/${R}_k4 \
    python tools/profile_step.py --steps 1 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_go_grad -s 1 -c 1 -o gpurun_out/${R}_k67 \
    python tools/profile_step.py --steps 1 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_cg_resident -c 1 -o gpurun_out/${R}_cg \
    python tools/profile_step.py --steps 1 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_rk_stage -s 1 -c 1 -o gpurun_out/${R}_k3 \
    python tools/profile_step.py --steps 1 > /dev/null 2>&1
ls -la gpurun_out/
