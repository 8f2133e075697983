#!/bin/bash
# ncu launch lists of one virtual-rank slab step: usage tools/slab_prof.sh [workload] [R]
WL=${1:-cfg3}; R=${2:-8}
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/slabprof_${WL}_r${R}.csv python tools/slab_profile.py $WL $R 3 > gpurun_out/slabprof.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/slabprof_${WL}_r1.csv python tools/slab_profile.py $WL 1 3 >> gpurun_out/slabprof.log 2>&1
tail -2 gpurun_out/slabprof.log
