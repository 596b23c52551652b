#!/bin/bash
# Profiles committed under profiles/ for one round (run under gpurun, 1 GPU).
set -x
R=${1:-r1}
# launch list of one eager C2 step (cold cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_cold.csv \
    python tools/profile_step.py --steps 1 > /dev/null 2>&1
# same with warm caches
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
    --log-file gpurun_out/${R}_launches_warm.csv python tools/profile_step.py --steps 1 > /dev/null 2>&1
# full captures: K2, K4, K6 (pipelined), resident CG (cold caches = default, like bench traffic)
ncu --set full --clock-control none --import-source on -k regex:k_pipe -s 1 -c 1 -o gpurun_out/${R}_k2 \
    python tools/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pipe -s 4 -c 1 -o gpurun_out/${R}_k4 \
    python tools/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pipe -s 5 -c 1 -o gpurun_out/${R}_k6 \
    python tools/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_cg_resident -c 1 -o gpurun_out/${R}_cg_resident \
    python tools/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_cg_spmv|k_cg_update" -s 2 -c 2 \
    -o gpurun_out/${R}_cg_two_kernel python tools/profile_step.py --steps 1 --no-resident > /dev/null 2>&1
ls -la gpurun_out/
