#!/bin/bash
# usage: tools/prof.sh NAME KERNEL_REGEX SKIP [profile_step args...]
# full ncu capture (warm caches) of one launch of an eager C2 step
name=$1; shift; regex=$1; shift; skip=$1; shift
ncu --set full --cache-control none --clock-control none --import-source on -k "regex:$regex" -s "$skip" -c 1 \
    -o "gpurun_out/prof_$name" python tools/profile_step.py --steps 1 "$@" > "gpurun_out/prof_$name.log" 2>&1
